"""Compressed decode step (C2 turn-3 state, or SHAPE=c4: 8 batched C4 sessions): CUDA events
over graph replays of the per-layer K6 launches. Diagnostics for launch-shape sweeps."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
from paper_2507_13681_b200.kvcompress import CompressionConfig
C4 = os.environ.get("SHAPE") == "c4"  # 8 Qwen2.5-7B sessions batched (28 layers, 8 x 28 q / 8 x 4 kv heads)
L, NQ, NKV = (28, 224, 32) if C4 else (32, 32, 8)
shape = AttnShape(L, NQ, NKV, 128)
cap = 3 * 5128
store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=1)
eng = SessionEngine(shape, SessionParams(alpha=0.955, comp=CompressionConfig(1024, 16, 16), max_new=128), cap,
                    session_seeds=list(range(8)) if C4 else None)
eng.prefill(store, 2, 10128, 5128)
eng.decode(store, 15256, 20)
torch.cuda.synchronize()
st = eng.stack
cols = 1024 + eng.window + 1
out = torch.empty((L, NQ, 128), dtype=torch.bfloat16, device="cuda")
na = st.n_a.cpu()
lo = max(0, st.length - eng.window)
bytes_step = sum((int(na[hr]) + st.length - lo + 1) * 128 * 4 for hr in range(L * NQ))
def per_layer():
    for l in range(L):
        st.step_archive(l, store.q[l], store.k[l], store.v[l], True, cols, out[l], pdl=l > 0)
for _ in range(5): per_layer()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    g.capture_begin()
    for _ in range(10): per_layer()
    g.capture_end()
torch.cuda.current_stream().wait_stream(s); g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): g.replay()
e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / 50
print(f"{os.environ.get('LS_LIB_PATH', 'default'):40s} {us:7.1f} us/step {us / L:5.2f} us/layer "
      f"{bytes_step / us / 1e3:7.1f} GB/s ({bytes_step / 1e6:.1f} MB/step)")
