"""Per-kernel device time of one C2 turn-3 prefill and one decode turn, from
CUPTI activity records (torch.profiler): warm caches, real overlap, no replay.
Diagnostics for the GPU box; bench numbers come from bench.py only."""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
from paper_2507_13681_b200.kvcompress import CompressionConfig

L = int(os.environ.get("LAYERS", "32"))
IN = int(os.environ.get("INPUT", "5000"))
shape = AttnShape(L, 32, 8, 128)
cap = 3 * (IN + 128)
store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=1)
eng = SessionEngine(shape, SessionParams(alpha=0.955, comp=CompressionConfig(1024, 16, 16), max_new=128), cap)
ro, n_new = 2 * (IN + 128) - 128, IN + 128


def turn():
    eng.prefill(store, 2, ro, n_new)
    eng.decode(store, ro + n_new, 128)


for _ in range(2):
    turn()
torch.cuda.synchronize()


def table(prof, title):
    agg = defaultdict(lambda: [0, 0.0])
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            name = e.name.split("(")[0][:60]
            agg[name][0] += 1
            agg[name][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    tot = sum(v[1] for v in agg.values())
    print(f"## {title}: {tot / 1e3:.3f} ms summed kernel time")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
        print(f"{us / 1e3:9.3f} ms {n:6d} x {us / max(n, 1):8.2f} us  {k}")


ONLY = os.environ.get("ONLY", "")
for name, fn in (("prefill turn 3", lambda: eng.prefill(store, 2, ro, n_new)),
                 ("decode turn 3", lambda: eng.decode(store, ro + n_new, 128))):
    if ONLY and not name.startswith(ONLY):
        continue
    if name.startswith("decode"):
        eng.prefill(store, 2, ro, n_new)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1):.3f} ms (events, unprofiled)")
    if name.startswith("decode"):
        eng.prefill(store, 2, ro, n_new)
        torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    table(prof, name)
