"""Greedy (K3) phase counters at one C5 layer (8 q-heads / 1 kv head, turn 10:
row_offset 91024, n_new 10128, n_total 101152)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_13681_b200 import _lib  # noqa: E402
from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams  # noqa: E402
from paper_2507_13681_b200.kvcompress import CompressionConfig  # noqa: E402

IN, T = int(os.environ.get("INPUT", "10000")), int(os.environ.get("TURNS", "10"))
shape = AttnShape(1, 8, 1, 128)
cap = T * (IN + 128)
store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=1)
eng = SessionEngine(shape, SessionParams(alpha=0.955, comp=CompressionConfig(1024, 16, 16), max_new=128), cap)
ro, n_new = (T - 1) * (IN + 128) - 128, IN + 128
eng.prefill(store, T - 1, ro, n_new)
torch.cuda.synchronize()
H = shape.n_q
for nocross in (0, 1):
    dbg = torch.zeros(70000, dtype=torch.int32).pin_memory()
    dbg[69999] = nocross
    _lib.lib().ls_debug_set_buffer(dbg.data_ptr())
    eng.prefill(store, T - 1, ro, n_new)
    torch.cuda.synchronize()
    _lib.lib().ls_debug_set_buffer(None)
    d = dbg[60000: 60000 + H * 8].view(H, 8)
    ph = dbg[61000:61000 + H * 4].view(H, 4)
    print(f"no_cross={nocross}")
    for h in range(H):
        print(f"  head {h}: picks {int(d[h, 0])} final {int(d[h, 1])} producer_cyc {int(d[h, 2])} "
              f"({int(d[h, 2]) / max(1, int(d[h, 0])):.0f}/pick) finalizer_cyc {int(d[h, 3])} ring_wait {int(d[h, 4])} "
              f"fin_wait {int(d[h, 5])} consumer_busy/16 {int(d[h, 6])} rounds {int(d[h, 7])} phases {ph[h].tolist()}")
