"""Per-CTA phase timeline of the event select kernel (globaltimer records via
ls_debug_set_buffer) at the C2 turn-3 state. Diagnostics only (GPU box)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2507_13681_b200 import _lib
from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
from paper_2507_13681_b200.kvcompress import CompressionConfig

L = 32
shape = AttnShape(L, 32, 8, 128)
cap = 3 * 5128
store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=1)
eng = SessionEngine(shape, SessionParams(alpha=0.955, comp=CompressionConfig(1024, 16, 16), max_new=128), cap)
ro, n_new = 10128, 5128
dbg = torch.zeros(L * 32 * 16, dtype=torch.int32).pin_memory()
_lib.lib().ls_debug_set_buffer(dbg.data_ptr())
eng.prefill(store, 2, ro, n_new)
eng.decode(store, ro + n_new, 128)  # graphs captured with the debug buffer
torch.cuda.synchronize()
g = [v for k, v in eng._graphs.items() if k[0] == "event"][0]
for label, steps in (("first event (dense rows)", 15), ("later event (compressed rows)", 31)):
    eng.prefill(store, 2, ro, n_new)
    eng.decode(store, ro + n_new, steps)
    torch.cuda.synchronize()
    dbg.zero_()
    g.replay()
    torch.cuda.synchronize()
    d = dbg.view(-1, 16).numpy().astype(np.int64)
    t0 = d[:, 0].min()
    rel = lambda c: (d[:, c] - d[:, 0]) / 1e3
    print(f"== {label}: span {(d[:, 6].max() - t0) / 1e3:.1f} us, CTA median: zero {np.median(rel(1)):.2f} "
          f"accumulate {np.median(rel(2)):.2f} list {np.median(rel(3)):.2f} select {np.median(rel(4)):.2f} "
          f"rank {np.median(rel(5)):.2f} end {np.median(rel(6)):.2f} us; max end {rel(6).max():.2f}; "
          f"round0: meta {np.median(rel(8)):.2f} data {np.median(rel(9)):.2f}; "
          f"candidates {d[:, 7].min()}-{d[:, 7].max()}")
_lib.lib().ls_debug_set_buffer(None)
