"""Host vs device time of one C2 turn-3 prefill (diagnostics, GPU box)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
from paper_2507_13681_b200.kvcompress import CompressionConfig

L = int(os.environ.get("LAYERS", "32"))
shape = AttnShape(L, 32, 8, 128)
cap = 3 * 5128
store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=1)
eng = SessionEngine(shape, SessionParams(alpha=0.955, comp=CompressionConfig(1024, 16, 16), max_new=128), cap)
ro, n_new = 10128, 5128
for _ in range(2):
    eng.prefill(store, 2, ro, n_new)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
eng.prefill(store, 2, ro, n_new)
t1 = time.perf_counter()
e1.record()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e3*(t1-t0):.2f} ms, device {e0.elapsed_time(e1):.2f} ms, wall {1e3*(t2-t0):.2f} ms")
pr = cProfile.Profile()
pr.enable()
eng.prefill(store, 2, ro, n_new)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
