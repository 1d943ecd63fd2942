"""torch.profiler timeline of one C2 turn-3 prefill (+ a few decode steps):
reports GPU idle gaps and the host ops that were running during them."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams  # noqa: E402
from paper_2507_13681_b200.kvcompress import CompressionConfig  # noqa: E402

L = int(os.environ.get("LAYERS", "32"))
shape = AttnShape(L, 32, 8, 128)
RO = int(os.environ.get("RO", "10128"))
NNEW = int(os.environ.get("NNEW", "5128"))
cap = RO + NNEW + 256
store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=1)
eng = SessionEngine(shape, SessionParams(alpha=0.955, comp=CompressionConfig(2048 if RO > 20000 else 1024, 16, 16),
                                         max_new=128), cap)
ro, n_new = RO, NNEW
for _ in range(2):
    eng.prefill(store, 2, ro, n_new)
    eng.decode(store, ro + n_new, 40)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    eng.prefill(store, 2, ro, n_new)
    torch.cuda.synchronize()
    eng.decode(store, ro + n_new, 40)
    torch.cuda.synchronize()
path = "gpurun_out/trace_turn.json"
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
gpu = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy") and "dur" in e],
             key=lambda e: e["ts"])
cpu = [e for e in ev if e.get("cat") in ("cpu_op", "cuda_runtime", "python_function", "cuda_driver") and "dur" in e]
print(f"{len(gpu)} GPU events, span {(gpu[-1]['ts'] + gpu[-1]['dur'] - gpu[0]['ts']) / 1e3:.2f} ms, "
      f"busy {sum(e['dur'] for e in gpu) / 1e3:.2f} ms")
gaps = []
for a, b in zip(gpu, gpu[1:]):
    g = b["ts"] - (a["ts"] + a["dur"])
    if g > 20:
        gaps.append((g, a, b))
print(f"gaps > 20 us: {len(gaps)}, total {sum(g for g, _, _ in gaps) / 1e3:.2f} ms")
agg = {}
for g, a, b in gaps:
    t0, t1 = a["ts"] + a["dur"], b["ts"]
    over = [c for c in cpu if c["ts"] < t1 and c["ts"] + c["dur"] > t0 and c.get("cat") in ("cuda_runtime", "cuda_driver")]
    key = (a["name"][:40], b["name"][:40], ",".join(sorted({c["name"] for c in over}))[:120])
    s = agg.setdefault(key, [0, 0.0])
    s[0] += 1
    s[1] += g
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{t / 1e3:8.2f} ms  n={n:4d}  after {k[0]} -> before {k[1]} | host: {k[2]}")
