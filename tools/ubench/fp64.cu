// fp64 add latency on this GPU (dependent chain, one warp). Diagnostics only.
#include <cstdio>
__global__ void k(int n, double x, long long *out, double *sink) {
  double a = x, b = x * 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { a += b; b += 1e-9; }
  long long t1 = clock64();
  float f = static_cast<float>(x), g = 0.5f;
  for (int i = 0; i < n; ++i) { f += g; g += 1e-9f; }
  long long t2 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; }
  sink[threadIdx.x] = a + f;
}
int main() {
  long long *o; double *s; cudaMalloc(&o, 16); cudaMalloc(&s, 256);
  k<<<1, 32>>>(4096, 1.0, o, s);
  long long h[2]; cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
  printf("dependent DADD: %.1f cycles, dependent FADD: %.1f cycles\n", h[0] / 4096.0, h[1] / 4096.0);
  return 0;
}
