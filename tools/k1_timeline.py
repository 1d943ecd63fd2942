"""K1 lines phase clocks (CTA 0; threads 0 / 32 / 256) at C2 turn 3, layer 0:
per-tile averages of exp(t+1), reduce(t), the tile barrier, chunk flush / item switch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_13681_b200 import _lib  # noqa: E402
from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams  # noqa: E402
from paper_2507_13681_b200.kvcompress import CompressionConfig  # noqa: E402

shape = AttnShape(1, 32, 8, 128)
cap = 3 * 5128
store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=1)
eng = SessionEngine(shape, SessionParams(alpha=0.955, comp=CompressionConfig(1024, 16, 16), max_new=128), cap)
eng.prefill(store, 2, 10128, 5128)
torch.cuda.synchronize()
dbg = torch.zeros(70000, dtype=torch.int32).pin_memory()
_lib.lib().ls_debug_set_buffer(dbg.data_ptr())
eng.prefill(store, 2, 10128, 5128)
torch.cuda.synchronize()
_lib.lib().ls_debug_set_buffer(None)
names = ["exp(t+1)", "reduce(t)", "barrier", "flush/item"]
for w, who in enumerate(["tid0", "tid32", "tid256"]):
    r12 = dbg[40000 + w * 768: 40000 + (w + 1) * 768].view(64, 12).numpy().astype(np.int64)
    r = r12[:, :5]
    ok = r[:, 0] != 0
    r = r[ok]
    d = np.diff(r, axis=1) & 0xffffffff
    tot = (np.diff(r[:, 0]) & 0xffffffff)
    print(who, "tiles", len(r), " ".join(f"{n}={v:.0f}" for n, v in zip(names, list(d.mean(axis=0)))),
          f"total/tile={tot.mean():.0f} cycles")
    if who in ("tid0", "tid256"):
        for t in range(12):
            print("   tile", t, (d[t]).tolist())
