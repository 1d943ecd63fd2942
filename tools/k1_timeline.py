"""K1 lines phase clocks (CTA 0; threads 0 / 32 / 256) at C2 turn 3, layer 0:
per-tile averages of wait-S, exp+store, barrier 1, vertical, slash, barrier 2, tail."""
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
names = ["waitS", "exp+store", "B1", "issue+vertical", "slash", "B2", "combine+flush", "->next"]
for w, who in enumerate(["tid0", "tid32", "tid256"]):
    r12 = dbg[40000 + w * 768: 40000 + (w + 1) * 768].view(64, 12).numpy().astype(np.int64)
    r = r12[:, :8]
    ok = r[:, 0] != 0
    r = r[ok]
    d = np.diff(r, axis=1) & 0xffffffff
    tail = ((np.roll(r[:, 0], -1) - r[:, 7]) & 0xffffffff)[:-1]
    tot = (np.diff(r[:, 0]) & 0xffffffff)
    print(who, "tiles", len(r), " ".join(f"{n}={v:.0f}" for n, v in zip(names, list(d.mean(axis=0)) + [tail.mean()])),
          f"total/tile={tot.mean():.0f} cycles")
    if who in ("tid0", "tid256"):
        for t in range(12):
            print("   tile", t, (d[t]).tolist())
    if who == "tid0":
        kw = (r12[:, 8] - r12[:, 3]) & 0xffffffff
        iss = (r12[:, 9] - r12[:, 8]) & 0xffffffff
        ready = (np.roll(r12[:, 1], -1) - r12[:, 9]) & 0xffffffff
        lat = (r12[:, 10] - r12[:, 9]) & 0xffffffff
        print(f"   after B1 -> K ready {kw[:-1].mean():.0f}, issue {iss[:-1].mean():.0f}, issue -> S seen ready by tid0 "
              f"{ready[:-1].mean():.0f} cycles; spin-measured MMA latency {lat[:-1].mean():.0f} (LS_K1_MMALAT builds)")
