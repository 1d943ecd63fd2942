"""K2/K3 device times at C2 turn 3 (4 layers) plus a
plan digest so variants can be checked for identical output."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
from paper_2507_13681_b200.kvcompress import CompressionConfig

CFG = os.environ.get("CFG", "c2")
if CFG == "c2":
    shape, cap, ro, n_new, t = AttnShape(4, 32, 8, 128), 3 * 5128, 10128, 5128, 2
elif CFG == "c2t1":
    shape, cap, ro, n_new, t = AttnShape(4, 32, 8, 128), 3 * 5128, 0, 5000, 0
else:  # c3 turn 4
    shape, cap, ro, n_new, t = AttnShape(4, 32, 8, 128), 4 * 8448, 25088, 8448, 3
store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=1)
mode = "dense" if os.environ.get("DENSE") else "loopserve"
eng = SessionEngine(shape, SessionParams(mode=mode, alpha=0.955, comp=CompressionConfig(1024, 16, 16), max_new=128), cap)
for _ in range(2):
    res = eng.prefill(store, t, ro, n_new)
torch.cuda.synchronize()
h = hashlib.sha1()
for p in (x for x in res.plans if x is not None):
    h.update(p.counts.cpu().numpy().tobytes())
    h.update(p.slash_ids.cpu().numpy().tobytes())
    h.update(p.vert_ids.cpu().numpy().tobytes())
ho = hashlib.sha1()
for o in res.out:
    ho.update(o.float().cpu().numpy().tobytes())
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    eng.prefill(store, t, ro, n_new)
    torch.cuda.synchronize()
agg = {}
for e in prof.events():
    if e.device_type.name == "CUDA":
        agg.setdefault(e.name[:60], []).append(e.device_time_total)
print(f"{os.environ.get('LS_LIB_PATH', 'lib')} {CFG} {mode} plans sha1 {h.hexdigest()[:16]} out sha1 {ho.hexdigest()[:16]}")
tot = 0.0
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[:int(os.environ.get('TOP', '16'))]:
    print(f"  {sum(v) / 1e3 / shape.n_layers:8.3f} ms/layer {len(v):4d} x  {k}")
