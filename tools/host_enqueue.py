import os, sys, time
sys.path.insert(0, '/root/repo')
import torch
from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
from paper_2507_13681_b200.kvcompress import CompressionConfig
shape = AttnShape(32, 32, 8, 128)
cap = 3 * 5128
store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=1)
eng = SessionEngine(shape, SessionParams(alpha=0.955, comp=CompressionConfig(1024, 16, 16), max_new=128), cap)
for t, (ro, n) in enumerate([(0, 5000), (5000, 5128), (10128, 5128)]):
    eng.prefill(store, t, ro, n)
torch.cuda.synchronize()
for t, (ro, n) in enumerate([(0, 5000), (5000, 5128), (10128, 5128)]):
    t0 = time.perf_counter(); eng.prefill(store, t, ro, n); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"turn {t}: host enqueue {1e3*(t1-t0):.2f} ms, total {1e3*(t2-t0):.2f} ms")
