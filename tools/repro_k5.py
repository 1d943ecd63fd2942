"""Run one K5 configuration (tensor-core path + CUDA-core cross-check) for
debugging under compute-sanitizer:
  compute-sanitizer --tool memcheck python tools/repro_k5.py 128 8 2 2048 2048
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2507_13681_b200 import _lib  # noqa: E402
from paper_2507_13681_b200 import prefill as pf  # noqa: E402
from paper_2507_13681_b200 import tensor_ops as tops  # noqa: E402
from paper_2507_13681_b200.synth import SynthSpec, layer_qkv_torch  # noqa: E402

d, n_q, n_kv, ro, n_new = (int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (128, 8, 2, 2048, 2048)))
n_total = ro + n_new
spec = SynthSpec(n_q, n_kv, d, n_total, seed=7)
Q, K, V = layer_qkv_torch(spec, 0)
qb = Q[:, ro:n_total].contiguous()
rows = pf.sample_rows_device(n_new, 0.1, 32, 3, 1, 0, 0, n_q)
plans = pf.sparsify_layer(qb, K, rows, 0.955, n_new, n_total, n_kv)
torch.cuda.synchronize()
print("plans ok", plans.counts.cpu().tolist())
n_cta = ((n_new + 127) // 128) * n_q
dbg = torch.full((n_cta * 16,), -7, dtype=torch.int32).pin_memory()
if os.environ.get("LS_DEBUG"):
    _lib.lib().ls_debug_set_buffer(dbg.data_ptr())
try:
    out_tc, cells_tc = tops.attention_layer(qb, K, V, plans.slash_ids, plans.vert_ids, plans.counts, n_new,
                                            n_total, n_kv, out_dtype=torch.float32)
    torch.cuda.synchronize()
except Exception as e:  # noqa: BLE001
    print("FAILED:", e)
    d = dbg.view(n_cta, 4, 4).tolist()
    names = ["producer", "mma", "softmax", "counts"]
    for i, rec in enumerate(d):
        print("cta", i, {names[r]: rec[r][:2] if r < 3 else rec[r] for r in range(4)})
    sys.exit(1)
_lib.lib().ls_debug_set_buffer(None)
L = pf.layer_desc(n_q, n_kv, d, n_new, n_total, qb.stride(0), K.stride(0))
out_s = torch.empty_like(out_tc)
cells_s = torch.empty_like(cells_tc)
n = _lib.lib().ls_vs_attention_workspace(ctypes.byref(L))
ws = torch.empty(n, dtype=torch.uint8, device="cuda")
_lib.call("ls_vs_attention_simt", ctypes.byref(L), qb.data_ptr(), K.data_ptr(), V.data_ptr(),
          plans.slash_ids.data_ptr(), plans.vert_ids.data_ptr(), plans.counts.data_ptr(), out_s.data_ptr(), 0,
          cells_s.data_ptr(), ws.data_ptr(), n, _lib.stream_ptr())
torch.cuda.synchronize()
print("cells tc", cells_tc.tolist())
print("cells simt", cells_s.tolist())
print("max abs diff", (out_tc - out_s).abs().max().item())
