"""Decode step time by kind (dense / compressed / event) at the C2 turn-3 state:
CUDA-graph replays timed with events, so PDL overlap between layers counts
as it does in bench.py. Diagnostics for the GPU box (launch-shape sweeps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
from paper_2507_13681_b200.kvcompress import CompressionConfig

L = int(os.environ.get("LAYERS", "32"))
IN = int(os.environ.get("INPUT", "5000"))
N = int(os.environ.get("REPS", "50"))
shape = AttnShape(L, 32, 8, 128)
cap = 3 * (IN + 128)
store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=1)
eng = SessionEngine(shape, SessionParams(alpha=0.955, comp=CompressionConfig(1024, 16, 16), max_new=128), cap)
ro, n_new = 2 * (IN + 128) - 128, IN + 128
eng.prefill(store, 2, ro, n_new)
eng.decode(store, ro + n_new, 128)  # captures the graphs
torch.cuda.synchronize()
res = {}
for kind, g in sorted(eng._graphs.items(), key=lambda kv: str(kv[0])):
    name = kind[0]
    eng.prefill(store, 2, ro, n_new)
    eng.decode(store, ro + n_new, 20)  # past the first event: compressed state valid
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        g.replay()
    e0.record()
    for _ in range(N):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    res[name] = e0.elapsed_time(e1) / N
eng.prefill(store, 2, ro, n_new)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
eng.decode(store, ro + n_new, 128)
e1.record()
torch.cuda.synchronize()
print(" ".join(f"{k}={v * 1e3:.1f}us/step" for k, v in res.items()), f"turn={e0.elapsed_time(e1):.2f}ms",
      f"per_layer: " + " ".join(f"{k}={v * 1e3 / L:.2f}us" for k, v in res.items() if k != "event"))
