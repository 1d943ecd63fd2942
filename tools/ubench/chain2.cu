// optimized producer chain: speculative head prefetch, branchless select
#include <cstdio>
constexpr int N = 800;
__device__ __forceinline__ bool dec(double a, int ds, double b, int dv) {
  const double x = a * static_cast<double>(dv), y = b * static_cast<double>(ds);
  const double diff = x - y, mag = fmax(fabs(x), fabs(y));
  if (__builtin_expect(fabs(diff) > 1e-13 * mag, 1)) return diff > 0.0;
  return a / ds >= b / dv;
}
struct Head { double w, mx; int len, idx; };
__global__ void chain(long long *cyc, int *out, int mode) {
  __shared__ double w[2][N + 2], mx[2][N + 2];
  __shared__ int len[2][N + 2], idx[2][N + 2];
  __shared__ double rw[256], ra[256];
  __shared__ int rc[256], ro[256];
  __shared__ volatile int nprod;
  for (int i = threadIdx.x; i < N + 2; i += blockDim.x)
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
  Head hs{w[0][0], mx[0][0], len[0][0], idx[0][0]}, hv{w[1][0], mx[1][0], len[1][0], idx[1][0]};
  Head ns{w[0][1], mx[0][1], len[0][1], idx[0][1]}, nv{w[1][1], mx[1][1], len[1][1], idx[1][1]};
  while (s < N - 2 && v < N - 2) {
    const bool ts = dec(hs.w - olv, max(1, hs.len - v), hv.w - ols, max(1, hv.len - s));
    const double wl = ts ? hs.w : hv.w;
    ap += wl - (ts ? olv : ols);
    ols += ts ? hs.mx : 0.0;
    olv += ts ? 0.0 : hv.mx;
    const int code = ts ? hs.idx : (hv.idx | 0x80000000);
    const int other = ts ? v : s;
    s += ts; v += !ts;
    // advance the taken list's head to its prefetched successor, prefetch the next
    if (ts) { hs = ns; ns = Head{w[0][s + 1], mx[0][s + 1], len[0][s + 1], idx[0][s + 1]}; }
    else { hv = nv; nv = Head{w[1][v + 1], mx[1][v + 1], len[1][v + 1], idx[1][v + 1]}; }
    const int sl = n & 255;
    rc[sl] = code; ro[sl] = other; rw[sl] = wl; ra[sl] = ap;
    ++n;
    if (mode == 1 || (n & 7) == 0) { __threadfence_block(); nprod = n; }
  }
  cyc[0] = clock64() - t0;
  out[0] = n + (int)ap + rc[3] + ro[5] + (int)rw[7] + (int)ra[9];
  out[1] = n;
}
int main() {
  long long *c, h; int *o, ho[2];
  cudaMalloc(&c, 8); cudaMalloc(&o, 8);
  for (int mode = 1; mode <= 2; ++mode) {
    chain<<<1, 128>>>(c, o, mode); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); cudaMemcpy(ho, o, 8, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): %.1f cyc/pick (%d picks)\n", mode, mode == 1 ? "fence every pick" : "fence every 8", (double)h / ho[1], ho[1]);
  }
  return 0;
}
