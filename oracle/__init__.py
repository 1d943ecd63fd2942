"""CPU oracle for the LoopServe hot paths -- TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference algorithm
(arxiv 2507.13681, `pkg/src/loopserve/` under the read-only reference mount).
Every function cites the reference file:line it restates.

Who may use it (enforced by review, see DESIGN.md section "Oracle"):
  * tests/ (as the checker of the CUDA path),
  * __graft_entry__.smoke() (as the checker),
  * bench.py's cpu_baseline / --impl reference leg (as the timed CPU baseline).
The product package `paper_2507_13681_b200` never imports this package; its
functions fail loudly when the CUDA library is missing instead of falling
back here.

Parity pinning: tests/test_oracle_golden.py checks this restatement against
golden vectors produced by importing the reference itself
(tests/golden/make_golden.py, committed together with its outputs) and against
the hand-computed known answers of the reference's own tests
(pkg/tests/test_prefill.py, test_tensor_ops.py, test_kvcompress.py).
"""

from . import attention, kvcompress, prefill, seeding, session  # noqa: F401
