"""TTFT per turn of the C2 dialogue (32 layers, sparse prefill only; CUDA events,
after a warm-up dialogue). Env: LS_HEAD_GROUPS, CFG=c2|c3, LAYERS."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
from paper_2507_13681_b200.kvcompress import CompressionConfig

CFG = os.environ.get("CFG", "c2")
L = int(os.environ.get("LAYERS", "32"))
n_q, n_kv = 32, 8
if CFG == "c2":
    blocks, budget = [(0, 5000), (5000, 5128), (10128, 5128)], 1024
elif CFG == "c5":  # one KV-head group of Llama-70B (8 q-heads / 1 KV head), 10 turns x 10K
    blocks = [(0, 10000)] + [(10000 + (t - 1) * 10128, 10128) for t in range(1, 10)]
    budget, n_q, n_kv = 1024, 8, 1
else:
    blocks, budget = [(0, 8192), (8192, 8448), (16640, 8448), (25088, 8448)], 2048
cap = blocks[-1][0] + blocks[-1][1]
shape = AttnShape(L, n_q, n_kv, 128)
store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=1)
mode = "dense" if os.environ.get("DENSE") else "loopserve"
eng = SessionEngine(shape, SessionParams(mode=mode, alpha=0.955, comp=CompressionConfig(budget, 16, 16), max_new=128),
                    cap)
for t, (ro, n) in enumerate(blocks):
    eng.prefill(store, t, ro, n)
torch.cuda.synchronize()
ms = []
for rep in range(2):
    for t, (ro, n) in enumerate(blocks):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.prefill(store, t, ro, n)
        e1.record()
        torch.cuda.synchronize()
        if rep == 1:
            ms.append(e0.elapsed_time(e1))
print(f"{CFG} {mode} groups={os.environ.get('LS_HEAD_GROUPS', '1')} layers={L} TTFT per turn "
      f"{[round(x, 2) for x in ms]} mean {sum(ms) / len(ms):.2f} ms")
