"""Per-CTA timeline of the tensor-core decode kernel (globaltimer records via
ls_debug_set_buffer) for one dense and one compressed step at the C2 turn-3
state. Diagnostics only (GPU box)."""
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
dbg = torch.zeros(L * 256 * 16, dtype=torch.int32).pin_memory()
_lib.lib().ls_debug_set_buffer(dbg.data_ptr())
eng.prefill(store, 2, ro, n_new)
eng.decode(store, ro + n_new, 128)  # graphs captured with the debug buffer
torch.cuda.synchronize()


def show(kind):
    g = [v for k, v in eng._graphs.items() if k[0] == kind][0]
    eng.prefill(store, 2, ro, n_new)
    eng.decode(store, ro + n_new, 20)
    torch.cuda.synchronize()
    dbg.zero_()
    g.replay()
    torch.cuda.synchronize()
    d = dbg.view(L, -1, 16).numpy().astype(np.int64)
    print(f"== {kind} step")
    t_layer0 = None
    for l in (0, 1, 2, 16, 31):
        r = d[l]
        r = r[r[:, 1] != 0]
        if len(r) == 0:
            continue
        t0 = r[:, 1].min()
        if t_layer0 is None:
            t_layer0 = t0
        rel = lambda c: (r[:, c] - t0) / 1e3
        last = r[r[:, 6] != 0]
        stg = (last[:, 7] - t0) / 1e3 if len(last) else np.array([np.nan])
        sms = np.bincount(r[:, 0], minlength=148)
        print(f"layer {l:2d}: ctas {len(r)} start+{(t0 - t_layer0) / 1e3:7.2f}us | start spread {rel(1).max():5.2f} | "
              f"first data {np.median(rel(2)):5.2f} (max {rel(2).max():5.2f}) | loop end {np.median(rel(3)):5.2f} "
              f"(max {rel(3).max():5.2f}) | partial {np.median(rel(4)):5.2f} (max {rel(4).max():5.2f}) | "
              f"fence1 {np.median(rel(8)):5.2f} (max {rel(8).max():5.2f}) | ticket {np.median(rel(9)):5.2f} (max {rel(9).max():5.2f}) | "
              f"fence2 {((last[:, 10] - t0) / 1e3).max() if len(last) else float('nan'):5.2f} | "
              f"tiles@ {' '.join(f'{np.median((r[r[:, 11 + k] != 0][:, 11 + k] - t0) / 1e3):5.2f}' for k in range(3))} | "
              f"staged {stg.max():5.2f} | combined {((last[:, 6] - t0) / 1e3).max() if len(last) else float('nan'):5.2f} | tiles {r[:, 5].min()}-{r[:, 5].max()} "
              f"| SMs used {int((sms > 0).sum())}, max CTAs/SM {int(sms.max())}")


show("dense")
show("comp")
_lib.lib().ls_debug_set_buffer(None)
