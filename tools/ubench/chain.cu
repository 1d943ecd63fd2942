// producer-chain microbenchmark: cycles per greedy pick (smem lists, fp64 decisions)
#include <cstdio>
constexpr int N = 800;
__device__ __forceinline__ bool dec(double a, int ds, double b, int dv) {
  const double x = a * static_cast<double>(dv), y = b * static_cast<double>(ds);
  const double diff = x - y, mag = fmax(fabs(x), fabs(y));
  if (fabs(diff) > 1e-13 * mag) return diff > 0.0;
  return a / ds >= b / dv;
}
template <int MODE>
__global__ void chain(long long *cyc, int *out) {
  __shared__ double w[2][N], mx[2][N];
  __shared__ int len[2][N], idx[2][N];
  __shared__ double rw[256], ra[256];
  __shared__ int rc[256], ro[256];
  __shared__ volatile int nprod;
  for (int i = threadIdx.x; i < N; i += blockDim.x)
    for (int k = 0; k < 2; ++k) {
      w[k][i] = 100.0 / (i + 1 + k);
      mx[k][i] = 0.5 / (i + 2);
      len[k][i] = 5000 - i;
      idx[k][i] = i;
    }
  __syncthreads();
  if (threadIdx.x) return;
  long long t0 = clock64();
  int s = 0, v = 0, n = 0;
  double ols = 0, olv = 0, ap = 0;
  double ws = w[0][0], mxs = mx[0][0], wv = w[1][0], mxv = mx[1][0];
  int ls = len[0][0], lv = len[1][0], is = 0, iv = 0;
  while (s < N - 1 && v < N - 1) {
    const bool ts = dec(ws - olv, max(1, ls - v), wv - ols, max(1, lv - s));
    int code, other;
    double wl;
    if (ts) {
      wl = ws; ap += ws - olv; ols += mxs; code = is; other = v; ++s;
      ws = w[0][s]; mxs = mx[0][s]; ls = len[0][s]; is = idx[0][s];
    } else {
      wl = wv; ap += wv - ols; olv += mxv; code = iv; other = s; ++v;
      wv = w[1][v]; mxv = mx[1][v]; lv = len[1][v]; iv = idx[1][v];
    }
    if (MODE >= 1) {
      const int sl = n & 255;
      rc[sl] = code; ro[sl] = other; rw[sl] = wl; ra[sl] = ap;
    }
    if (MODE >= 2) __threadfence_block();
    if (MODE >= 1) nprod = n + 1;
    ++n;
  }
  cyc[0] = clock64() - t0;
  out[0] = n + (int)ap + rc[3] + ro[5] + (int)rw[7] + (int)ra[9];
  out[1] = n;
}
int main() {
  long long *c, h; int *o, ho[2];
  cudaMalloc(&c, 8); cudaMalloc(&o, 8);
  chain<0><<<1, 128>>>(c, o); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); cudaMemcpy(ho, o, 8, cudaMemcpyDeviceToHost);
  printf("chain only: %.1f cyc/pick (%d picks)\n", (double)h / ho[1], ho[1]);
  chain<1><<<1, 128>>>(c, o); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); cudaMemcpy(ho, o, 8, cudaMemcpyDeviceToHost);
  printf("+ ring stores: %.1f cyc/pick\n", (double)h / ho[1]);
  chain<2><<<1, 128>>>(c, o); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); cudaMemcpy(ho, o, 8, cudaMemcpyDeviceToHost);
  printf("+ membar: %.1f cyc/pick\n", (double)h / ho[1]);
  return 0;
}
