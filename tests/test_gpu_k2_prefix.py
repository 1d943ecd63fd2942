"""K2 prefix sort + K3 overflow fallback (select_lines.cu): at alpha = 0.999
the greedy picks more lines of one kind than a sorted prefix holds (PCAP =
4096), so the flagged heads are redone on fully sorted lists; the plans must
still equal the oracle's sparsify_head (prefill.py:363-390) up to documented
near-ties."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import attention as oatt
from oracle import prefill as opf
from parity import check_plan

pytestmark = pytest.mark.gpu


def test_prefix_overflow_falls_back_to_full_sort(cuda_lib):
    from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
    from paper_2507_13681_b200.kvcompress import CompressionConfig

    n_new = 9000
    shape = AttnShape(1, 2, 1, 64)
    store = QKVStore.synthetic(shape, n_new, n_ref=n_new, seed=5)
    eng = SessionEngine(shape, SessionParams(alpha=0.999, comp=CompressionConfig(256, 16, 16), max_new=16, seed=5),
                        n_new, out_dtype=torch.float32)
    res = eng.prefill(store, 0, 0, n_new)
    torch.cuda.synchronize()
    hp = res.plans[0].to_host()
    seqs = res.plans[0].pick_sequences()
    rows = res.rows[0].cpu().numpy()
    K = store.k[0, 0, :n_new].double().cpu().numpy()
    Q = store.q[0].double().cpu().numpy()
    most = 0
    for h in range(shape.n_q):
        Qs = Q[h, rows[h]]
        oplan = opf.sparsify_head(Qs, K, 0.999, rows[h])
        a = opf.line_arrays(oatt.softmax_rows(opf.sampled_logits(Qs, K, rows[h])), rows[h])
        check_plan(oplan, hp[h], seqs[h], dict(enumerate(a["s_w"].tolist())), dict(enumerate(a["v_w"].tolist())))
        most = max(most, len(hp[h].selected_slashes), len(hp[h].selected_verticals))
    assert most > 4096, f"the case no longer exercises the fallback ({most} picks of one kind)"
