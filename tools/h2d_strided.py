import torch, time
H, n, d, cap = 32, 5128, 128, 15384
src = torch.randn(H, n, d).to(torch.bfloat16).pin_memory()
dst = torch.empty(H, cap, d, dtype=torch.bfloat16, device="cuda")
stg = torch.empty(H, n, d, dtype=torch.bfloat16, device="cuda")
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
b = src.numel() * 2 / 1e9
ms = t(lambda: dst[:, 5000:5000 + n].copy_(src, non_blocking=True)); print(f"strided dst copy_: {ms:.3f} ms {b/ms*1e3:.1f} GB/s")
ms = t(lambda: stg.copy_(src, non_blocking=True)); print(f"contiguous staging: {ms:.3f} ms {b/ms*1e3:.1f} GB/s")
from cuda.bindings import runtime as cudart
def m2d():
    err, = cudart.cudaMemcpy2DAsync(dst[:, 5000:].data_ptr(), cap * d * 2, src.data_ptr(), n * d * 2, n * d * 2, H,
                                    cudart.cudaMemcpyKind.cudaMemcpyHostToDevice, torch.cuda.current_stream().cuda_stream)
ms = t(m2d); print(f"cudaMemcpy2DAsync: {ms:.3f} ms {b/ms*1e3:.1f} GB/s")
