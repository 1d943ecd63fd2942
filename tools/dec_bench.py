"""Decode time of one C2 turn-3 decode (128 tokens, all 32 layers; CUDA events
around SessionEngine.decode after an untimed re-prefill, best of REPS) --
diagnostics for launch-shape sweeps (tools/sweep_dec.sh)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
from paper_2507_13681_b200.kvcompress import CompressionConfig

L = int(os.environ.get("LAYERS", "32"))
IN = int(os.environ.get("INPUT", "5000"))
N = int(os.environ.get("REPS", "5"))
shape = AttnShape(L, 32, 8, 128)
cap = 3 * (IN + 128)
store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=1)
eng = SessionEngine(shape, SessionParams(alpha=0.955, comp=CompressionConfig(1024, 16, 16), max_new=128), cap)
ro, n_new = 2 * (IN + 128) - 128, IN + 128
best = None
for rep in range(N + 1):
    eng.prefill(store, 2, ro, n_new)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.decode(store, ro + n_new, 128)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if rep > 0:
        best = ms if best is None else min(best, ms)
print(f"decode turn (128 tokens, {L} layers): {best:.3f} ms = {128 / best * 1e3:.0f} tokens/s")
