"""Plan and K5 tile-kind statistics of the C2 synthetic layers (GPU box).
Replicates the K5 tile lists on the host from the device plans."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams  # noqa: E402
from paper_2507_13681_b200.kvcompress import CompressionConfig  # noqa: E402

BM = BN = 128
L = 2
shape = AttnShape(L, 32, 8, 128)
cap = 3 * 5128
store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=1)
eng = SessionEngine(shape, SessionParams(alpha=0.955, comp=CompressionConfig(1024, 16, 16), max_new=128), cap)
for t, (ro, n_new) in enumerate([(0, 5000), (5000, 5128), (10128, 5128)]):
    res = eng.prefill(store, t, ro, n_new)
    torch.cuda.synchronize()
    n_total = ro + n_new
    for l in range(L):
        p = res.plans[l]
        cn = p.counts.cpu().numpy()
        sl = p.slash_ids.cpu().numpy()
        vt = p.vert_ids.cpu().numpy()
        cells = res.cells[l].cpu().numpy()
        dense_cells = n_new * ro + n_new * (n_new + 1) // 2
        nd, ng, ndi = [], [], []
        for h in range(shape.n_q):
            S = sl[h, :cn[h, 0]]
            V = vt[h, :cn[h, 1]]
            for qt in range((n_new + BM - 1) // BM):
                g0 = ro + qt * BM
                g_hi = min(g0 + BM, n_total) - 1
                cnt = np.zeros(g_hi // BN + 1, int)
                for d in S[S <= g_hi]:
                    lo, hi = max(0, g0 - d), g_hi - d
                    cnt[lo // BN: hi // BN + 1] += 1
                dense = cnt >= 3
                diag = 0
                for d in S[S <= g_hi]:
                    lo, hi = max(0, g0 - d), g_hi - d
                    if (~dense[lo // BN: hi // BN + 1]).any():
                        diag += 1
                nd.append(int(dense.sum()))
                ng.append((int((V <= g_hi).sum()) + BN - 1) // BN)
                ndi.append(diag)
        print(f"turn {t} layer {l}: |S| mean {cn[:, 0].mean():.1f} max {cn[:, 0].max()}, |V| mean {cn[:, 1].mean():.1f}"
              f" max {cn[:, 1].max()}, density {cells.sum() / (dense_cells * shape.n_q):.4f};"
              f" per q-tile: dense {np.mean(nd):.2f}, gathered {np.mean(ng):.2f}, diagonal {np.mean(ndi):.2f}"
              f" (max {max(ndi)})")
