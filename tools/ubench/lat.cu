// dependent-chain latency microbenchmarks (cycles per op) on the current GPU
#include <cstdio>
__global__ void k_dadd(double *out, double x, int n, long long *cyc) {
  double a = x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = a + 1e-9 * a;  // DFMA chain
  cyc[0] = clock64() - t0;
  out[0] = a;
}
__global__ void k_dadd2(double *out, double x, int n, long long *cyc) {
  double a = x, b = 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { a = a + b; b = b - a * 1e-12; }
  cyc[0] = clock64() - t0;
  out[0] = a + b;
}
__global__ void k_fadd(float *out, float x, int n, long long *cyc) {
  float a = x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = a + 1e-9f * a;
  cyc[0] = clock64() - t0;
  out[0] = a;
}
__global__ void k_membar(int *out, int n, long long *cyc) {
  __shared__ volatile int s[32];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { s[i & 31] = i; __threadfence_block(); }
  cyc[0] = clock64() - t0;
  out[0] = s[3];
}
__global__ void k_lds(int *out, int n, long long *cyc) {
  __shared__ int s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  int j = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) j = s[j];
  cyc[0] = clock64() - t0;
  out[0] = j;
}
int main() {
  double *dd; float *fd; int *id; long long *c, h;
  cudaMalloc(&dd, 8); cudaMalloc(&fd, 4); cudaMalloc(&id, 4); cudaMalloc(&c, 8);
  const int n = 100000;
  k_dadd<<<1, 1>>>(dd, 1.0, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("DFMA dep chain: %.1f cyc\n", (double)h / n);
  k_dadd2<<<1, 1>>>(dd, 1.0, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("DADD+DFMA pair chain: %.1f cyc/iter\n", (double)h / n);
  k_fadd<<<1, 1>>>(fd, 1.0f, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("FFMA dep chain: %.1f cyc\n", (double)h / n);
  k_membar<<<1, 1>>>(id, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("STS+membar.cta: %.1f cyc\n", (double)h / n);
  k_lds<<<1, 32>>>(id, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("LDS dep chain: %.1f cyc\n", (double)h / n);
  return 0;
}
