"""Diagnostic: K5 error distribution at C2 turn 3 vs the oracle (per row)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import attention as oatt  # noqa: E402
from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams  # noqa: E402
from paper_2507_13681_b200.kvcompress import CompressionConfig  # noqa: E402

RO, N_NEW = 10128, 5128
N = RO + N_NEW
shape = AttnShape(1, 32, 8, 128)
store = QKVStore.synthetic(shape, N + 128, n_ref=N + 128, seed=21)
eng = SessionEngine(shape, SessionParams(alpha=0.955, comp=CompressionConfig(1024, 16, 16), max_new=128, seed=21),
                    N + 128, out_dtype=torch.float32 if "f32" in sys.argv else torch.bfloat16)
res = eng.prefill(store, 2, RO, N_NEW)
torch.cuda.synchronize()
hp = res.plans[0].to_host()
out = res.out[0].float().cpu().numpy()
rep = {}
for h in [int(x) for x in sys.argv[1].split(",")]:
    Qb = store.q[0, h, RO:N].double().cpu().numpy()
    Kd = store.k[0, h // 4, :N].double().cpu().numpy()
    Vd = store.v[0, h // 4, :N].double().cpu().numpy()
    Zo, Wt, co = oatt.masked_sparse_attention(Qb, Kd, Vd, hp[h].selected_slashes, hp[h].selected_verticals, RO,
                                              return_weights=True)
    e = np.abs(out[:, h] - Zo)
    er = e.max(axis=1)
    worst = np.argsort(-er)[:8]
    rep[h] = {"max": float(er.max()), "p999": float(np.quantile(er, 0.999)), "n_gt_1e2": int((er > 1e-2).sum()),
              "cells_dev": int(res.cells[0][h].item()), "cells_oracle": int(co),
              "worst": [{"row": int(r), "err": float(er[r]), "ncell": int((Wt[r] > 0).sum()),
                         "wmax": float(Wt[r].max()), "zmax": float(np.abs(Zo[r]).max()),
                         "dim": int(np.argmax(e[r]))} for r in worst]}
print(json.dumps(rep, indent=1))
