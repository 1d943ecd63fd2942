"""cProfile of SessionEngine.prefill's host path (C2 turn 1, 32 layers): where the
Python enqueue time goes (the prefill is host-bound when the GPU work per layer is
short)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
from paper_2507_13681_b200.kvcompress import CompressionConfig

shape = AttnShape(32, 32, 8, 128)
cap = 3 * 5128
store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=1)
eng = SessionEngine(shape, SessionParams(alpha=0.955, comp=CompressionConfig(1024, 16, 16), max_new=128), cap)
for _ in range(2):
    eng.prefill(store, 0, 0, 5000)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
eng.prefill(store, 0, 0, 5000)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
