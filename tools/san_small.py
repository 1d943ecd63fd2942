"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
one 2-turn session through every kernel family -- K0-K5, seeds, decode
graphs off (plain launches), events (K7/K8) -- plus the reference-API
drop-in kernels and the obswindow baseline."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2507_13681_b200 import kvcompress as kv
from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
from paper_2507_13681_b200.kvcompress import CompressionConfig

shape = AttnShape(1, 4, 2, 128)
IN, MAX_NEW = 700, 20
cap = 2 * (IN + MAX_NEW)
store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=4)
for mode in ("loopserve", "obswindow"):
    eng = SessionEngine(shape, SessionParams(mode=mode, alpha=0.9, comp=CompressionConfig(64, 8, 8), max_new=MAX_NEW),
                        cap)
    for t, (ro, n_new) in enumerate(eng.turn_blocks(IN, 2, MAX_NEW)):
        eng.prefill(store, t, ro, n_new)
        eng.decode(store, ro + n_new, MAX_NEW, use_graphs=False)
    torch.cuda.synchronize()
rows = [(np.arange(50), np.full(50, 0.02)), (np.array([3, 7, 60]), np.array([0.5, 0.25, 0.25]))]
ids, sc = kv.accumulate_scores(rows)
kv._top_by_score(ids, sc, 5)
kv.retained_union([1, 5, 9], 4, 20)
torch.cuda.synchronize()
print("san_small ok")
