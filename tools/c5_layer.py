"""Diagnostics: one C5 layer (8 q-heads / 1 kv head, turn 10: row_offset 91024, n_new 10128) -- plan sizes and
per-kernel device times (torch.profiler / CUPTI)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
from paper_2507_13681_b200.kvcompress import CompressionConfig

IN, T = int(os.environ.get("INPUT", "10000")), int(os.environ.get("TURNS", "10"))
shape = AttnShape(1, 8, 1, 128)
cap = T * (IN + 128)
store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=1)
eng = SessionEngine(shape, SessionParams(alpha=0.955, comp=CompressionConfig(1024, 16, 16), max_new=128), cap)
ro, n_new = (T - 1) * (IN + 128) - 128, IN + 128
for _ in range(2):
    res = eng.prefill(store, T - 1, ro, n_new)
torch.cuda.synchronize()
cn = res.plans[0].counts.cpu().numpy()
print("plans (slashes, verticals):", cn.tolist(), "n_picks", res.plans[0].n_picks.cpu().numpy().tolist())
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    eng.prefill(store, T - 1, ro, n_new)
    torch.cuda.synchronize()
agg = {}
for e in prof.events():
    if e.device_type.name == "CUDA":
        agg.setdefault(e.name[:70], []).append(e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total)
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[:14]:
    print(f"{sum(v)/1e3:9.3f} ms {len(v):4d} x  {k}")
