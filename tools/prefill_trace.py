"""Kernel timeline (stream, start, duration) of one C2 turn-3 prefill layer from a
torch.profiler chrome trace: shows how the head-group streams overlap.
Diagnostics for the GPU box. env: LS_HEAD_GROUPS, LAYER (default 16)."""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

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
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    eng.prefill(store, 2, ro, n_new)
    torch.cuda.synchronize()
path = os.path.join(tempfile.mkdtemp(), "t.json")
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0, t1 = ev[0]["ts"], ev[-1]["ts"] + ev[-1]["dur"]
print(f"prefill kernels {len(ev)}, span {(t1 - t0) / 1e3:.2f} ms, busy-sum {sum(e['dur'] for e in ev) / 1e3:.2f} ms")
# one layer: split by the k1_stats launches (one per group per layer)
starts = [i for i, e in enumerate(ev) if "k1_stats" in e["name"]]
G = eng.head_groups
lay = int(os.environ.get("LAYER", "16"))
a = starts[lay * G]
b = starts[(lay + 1) * G] if (lay + 1) * G < len(starts) else len(ev)
base = ev[a]["ts"]
for e in ev[a:b]:
    nm = e["name"].split("(")[0].replace("void ", "")[:48]
    print(f"  s{e['tid']!s:>4} {(e['ts'] - base):8.1f} +{e['dur']:7.1f}  {nm}")
