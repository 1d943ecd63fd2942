"""Per-head chain / finalize cycle counts of the greedy kernel (C2 turn 3, layer 0)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_13681_b200 import _lib  # noqa: E402
from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams  # noqa: E402
from paper_2507_13681_b200.kvcompress import CompressionConfig  # noqa: E402

shape = AttnShape(1, 32, 8, 128)
cap = 3 * 5128
store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=1)
eng = SessionEngine(shape, SessionParams(alpha=0.955, comp=CompressionConfig(1024, 16, 16), max_new=128), cap)
dbg = torch.zeros(70000, dtype=torch.int32).pin_memory()
for t, (ro, n_new) in enumerate([(0, 5000), (5000, 5128), (10128, 5128), (10128, 5128)]):
    eng.prefill(store, t, ro, n_new)
    torch.cuda.synchronize()
    dbg.zero_()
    dbg[69999] = 1 if t == 3 else 0  # turn "3": turn 2 again without crossing work
    _lib.lib().ls_debug_set_buffer(dbg.data_ptr())
    eng.prefill(store, t, ro, n_new)
    torch.cuda.synchronize()
    _lib.lib().ls_debug_set_buffer(None)
    d = dbg[60000: 60000 + 32 * 8].view(32, 8)
    print(f"turn {t}: chain picks max {int(d[:, 0].max())} mean {float(d[:, 0].float().mean()):.0f}; "
          f"final picks max {int(d[:, 1].max())}; producer cycles max {int(d[:, 2].max())} "
          f"({float(d[:, 2].max()) / max(1, int(d[int(d[:, 2].argmax()), 0])):.0f}/pick); "
          f"finalizer cycles max {int(d[:, 3].max())}; producer ring-full wait max {int(d[:, 4].max())}; "
          f"finalizer wait (slowest head) {int(d[int(d[:, 3].argmax()), 5])}; consumer busy/16 (slowest head) "
          f"{int(d[int(d[:, 3].argmax()), 6])}; producer rounds (slowest head) {int(d[int(d[:, 2].argmax()), 7])}; "
          f"phases head/fold/decide/publish {dbg[61000:61000 + 128].view(32, 4)[int(d[:, 2].argmax())].tolist()}")
