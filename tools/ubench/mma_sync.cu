// mma.sync.m16n8k16 bf16 latency / throughput on this GPU (one warp per SMSP,
// dependent chain vs 8 independent accumulators). Diagnostics only.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void mma(float *d, uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
__global__ void k(int n, long long *out, float *sink) {
  uint32_t a = threadIdx.x * 0x3f803f80u, b = 0x3f803f80u;
  float c[8][4] = {};
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) mma(c[0], a, a, b, b);  // dependent chain
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) mma(c[j], a, a, b, b);  // 8 independent chains
  }
  long long t2 = clock64();
  if (threadIdx.x == 0) { out[blockIdx.x * 2] = t1 - t0; out[blockIdx.x * 2 + 1] = t2 - t1; }
  float s = 0; for (int j = 0; j < 8; ++j) s += c[j][0];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  long long *o; float *s; cudaMalloc(&o, 16 * 4); cudaMalloc(&s, 4 * 128 * 4);
  const int n = 1024;
  for (int warps = 1; warps <= 4; warps *= 4) {
    k<<<1, 32 * warps>>>(n, o, s);
    long long h[2]; cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
    printf("warps/CTA %d: dependent %.1f cycles/mma, 8 independent chains %.1f cycles/mma (per warp)\n", warps,
           (double)h[0] / n, (double)h[1] / (8.0 * n));
  }
  return 0;
}
