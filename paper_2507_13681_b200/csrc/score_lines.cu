// K1 -- sampled-row scoring and vertical / slash line sums.
//
// Replaces the scoring part of sparsify_head (reference prefill.py:377-390),
// softmax_rows (tensor_ops.py:24-40) and _line_sums (prefill.py:138-169).
//
// One CTA per (head, tile of K1_BM sampled rows) sweeps the causal key range
// twice: pass 1 keeps an online (max, sum) per row; pass 2 recomputes the
// scores, forms P = exp2(s - m) / l in fp32 and reduces it into
//   * vertical partials: per column, rows ascending, fp64;
//   * slash partials: per diagonal d = g - c, rows ascending, fp64, by a
//     thread-owns-d gather over the P tile in shared memory (deterministic,
//     no float atomics; "reductions in ascending index order").
// Partials are per row tile ([head][row_tile][n_total]); k1_reduce sums them
// in row-tile order. Every reduction is deterministic; a given (d or c) sum
// differs from the reference only through fp32 P values.
//
// This is the CUDA-core path (scores by FFMA from shared memory); the
// tcgen05 path replaces the tile product, the reductions are shared.

#include "ls_common.cuh"

namespace ls {
namespace k1 {

constexpr int BM = 32;        // sampled rows per CTA
constexpr int BN = 64;        // keys per tile
constexpr int THREADS = 256;  // 8 threads per row, 8 columns each

struct Params {
  const uint16_t *q;
  const uint16_t *k;
  const int32_t *rows;  // [H][n_s] local block rows, sorted
  int n_heads, group, d, n_s, n_total, row_offset, n_rt;
  int64_t q_head_stride, kv_head_stride;
  float scale_log2;  // log2(e) / sqrt(d)
  double *vpart;     // [H][n_rt][n_total]
  float *vmaxp;
  double *spart;
  float *smaxp;
  float *row_stats;  // [H][n_s][2]: (m2, 1/l)
};

__device__ __forceinline__ void load_rows_f32(float *dst, int ld, const uint16_t *src, int64_t row_stride,
                                              const int *row_ids, int n_rows, int n_valid, int d) {
  // dst[r][0..d) = bf16 src row row_ids[r]; rows >= n_valid are zero.
  const int vec_per_row = d / 8;
  for (int i = threadIdx.x; i < n_rows * vec_per_row; i += blockDim.x) {
    int r = i / vec_per_row, v = i % vec_per_row;
    float f[8];
    if (r < n_valid) {
      uint4 u = *reinterpret_cast<const uint4 *>(src + static_cast<int64_t>(row_ids[r]) * row_stride + v * 8);
      bf16x8_to_f32(u, f);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) dst[r * ld + v * 8 + j] = f[j];
  }
}

__device__ __forceinline__ void load_krows(float *Ks, int ld, const uint16_t *kbase, int c0, int n_total, int d) {
  const int vec_per_row = d / 8;
  for (int i = threadIdx.x; i < BN * vec_per_row; i += blockDim.x) {
    int j = i / vec_per_row, v = i % vec_per_row;
    int c = c0 + j;
    float f[8];
    if (c < n_total) {
      uint4 u = *reinterpret_cast<const uint4 *>(kbase + static_cast<int64_t>(c) * d + v * 8);
      bf16x8_to_f32(u, f);
    } else {
#pragma unroll
      for (int t = 0; t < 8; ++t) f[t] = 0.f;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) Ks[j * ld + v * 8 + t] = f[t];
  }
}

// scores of row `row` against tile columns (cq + 8*i), i < 8
__device__ __forceinline__ void tile_scores(const float *Qs, const float *Ks, int ld, int d, int row, int cq,
                                            float *acc) {
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;
  const float *qr = Qs + row * ld;
  for (int kk = 0; kk < d; ++kk) {
    float qv = qr[kk];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fmaf(qv, Ks[(cq + 8 * i) * ld + kk], acc[i]);
  }
}

__global__ void __launch_bounds__(THREADS) score_lines_kernel(Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int h = blockIdx.y, rt = blockIdx.x;
  const int d = p.d, ld = d + 1;
  float *Qs = reinterpret_cast<float *>(smem_raw);  // [BM][ld]
  float *Ks = Qs + BM * ld;                          // [BN][ld]
  float *Ps = Ks + BN * ld;                          // [BM][BN+1]
  int *gs = reinterpret_cast<int *>(Ps + BM * (BN + 1));
  int *rid = gs + BM;
  float *m2s = reinterpret_cast<float *>(rid + BM);
  float *lis = m2s + BM;

  const int r_begin = rt * BM;
  const int nr = min(BM, p.n_s - r_begin);
  const int32_t *rows_h = p.rows + static_cast<int64_t>(h) * p.n_s;
  if (threadIdx.x < BM) {
    int r = threadIdx.x;
    int lr = r < nr ? rows_h[r_begin + r] : rows_h[r_begin + nr - 1];
    rid[r] = lr;
    gs[r] = r < nr ? p.row_offset + lr : 0x7fffffff;  // padded rows never match
  }
  __syncthreads();
  const int g_first = gs[0];
  const int g_last = gs[nr - 1];  // <= n_total - 1
  const uint16_t *qbase = p.q + static_cast<int64_t>(h) * p.q_head_stride;
  const uint16_t *kbase = p.k + static_cast<int64_t>(h / p.group) * p.kv_head_stride;
  load_rows_f32(Qs, ld, qbase, d, rid, BM, nr, d);

  const int64_t part_off = (static_cast<int64_t>(h) * p.n_rt + rt) * p.n_total;
  double *vpart = p.vpart + part_off;
  float *vmaxp = p.vmaxp + part_off;
  double *spart = p.spart + part_off;
  float *smaxp = p.smaxp + part_off;
  // this CTA exclusively owns spart[0..g_last]; zero it (RMW accumulator)
  for (int i = threadIdx.x; i <= g_last; i += blockDim.x) {
    spart[i] = 0.0;
    smaxp[i] = 0.f;
  }

  const int row = threadIdx.x / 8, cq = threadIdx.x % 8;
  const int my_g = gs[row];
  const int n_tiles = g_last / BN + 1;

  // ---- pass 1: online max / sum per row (log2 domain)
  float m = -INFINITY, l = 0.f;
  for (int t = 0; t < n_tiles; ++t) {
    const int c0 = t * BN;
    __syncthreads();
    load_krows(Ks, ld, kbase, c0, p.n_total, d);
    __syncthreads();
    float acc[8];
    tile_scores(Qs, Ks, ld, d, row, cq, acc);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int c = c0 + cq + 8 * i;
      if (row < nr && c <= my_g) {
        float s = acc[i] * p.scale_log2;
        if (s > m) {
          l = l * fast_exp2(m - s) + 1.f;
          m = s;
        } else {
          l += fast_exp2(s - m);
        }
      }
    }
  }
  // combine the 8 threads of a row (consecutive lanes)
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    float mo = __shfl_xor_sync(0xffffffffu, m, o);
    float lo = __shfl_xor_sync(0xffffffffu, l, o);
    float mn = fmaxf(m, mo);
    float a = (m == -INFINITY) ? 0.f : l * fast_exp2(m - mn);
    float b = (mo == -INFINITY) ? 0.f : lo * fast_exp2(mo - mn);
    m = mn;
    l = a + b;
  }
  if (cq == 0) {
    m2s[row] = m;
    lis[row] = (l > 0.f) ? 1.f / l : 0.f;
    if (row < nr) {
      float *rs = p.row_stats + (static_cast<int64_t>(h) * p.n_s + r_begin + row) * 2;
      rs[0] = m;
      rs[1] = (l > 0.f) ? 1.f / l : 0.f;
    }
  }

  // ---- pass 2: P tiles and line partials
  for (int t = 0; t < n_tiles; ++t) {
    const int c0 = t * BN;
    __syncthreads();
    load_krows(Ks, ld, kbase, c0, p.n_total, d);
    __syncthreads();
    float acc[8];
    tile_scores(Qs, Ks, ld, d, row, cq, acc);
    const float mr = m2s[row], li = lis[row];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int cl = cq + 8 * i;
      const int c = c0 + cl;
      float pv = 0.f;
      if (row < nr && c <= my_g) pv = fast_exp2(acc[i] * p.scale_log2 - mr) * li;
      Ps[row * (BN + 1) + cl] = pv;
    }
    __syncthreads();
    // verticals: one thread per column, rows ascending
    if (threadIdx.x < BN) {
      const int c = c0 + threadIdx.x;
      if (c < p.n_total) {
        double sw = 0.0;
        float mx = 0.f;
        for (int r = 0; r < nr; ++r) {
          float v = Ps[r * (BN + 1) + threadIdx.x];
          sw += static_cast<double>(v);
          mx = fmaxf(mx, v);
        }
        vpart[c] = sw;
        vmaxp[c] = mx;
      }
    }
    // slashes: thread owns diagonal d, rows ascending (g_r in [c0+d, c0+d+BN))
    const int d_lo = max(0, g_first - (c0 + BN - 1));
    const int d_hi = g_last - c0;
    for (int dd = d_lo + static_cast<int>(threadIdx.x); dd <= d_hi; dd += blockDim.x) {
      const int glo = c0 + dd, ghi = c0 + dd + BN - 1;
      int r = lower_bound_dev(gs, nr, glo);
      if (r >= nr || gs[r] > ghi) continue;
      double sw = spart[dd];
      float mx = smaxp[dd];
      for (; r < nr && gs[r] <= ghi; ++r) {
        float v = Ps[r * (BN + 1) + (gs[r] - dd - c0)];
        sw += static_cast<double>(v);
        mx = fmaxf(mx, v);
      }
      spart[dd] = sw;
      smaxp[dd] = mx;
    }
  }
}

// Sum row-tile partials in order; lines exist for every index < n_total.
__global__ void reduce_kernel(const double *vpart, const float *vmaxp, const double *spart, const float *smaxp,
                              const int32_t *rows, int n_s, int n_rt, int n_total, int row_offset, double *v_w,
                              float *v_max, double *s_w, float *s_max, int bm) {
  const int h = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_total) return;
  const int32_t *rows_h = rows + static_cast<int64_t>(h) * n_s;
  double vw = 0.0, sw = 0.0;
  float vm = 0.f, sm = 0.f;
  for (int rt = 0; rt < n_rt; ++rt) {
    const int last = min(n_s, (rt + 1) * bm) - 1;
    const int g_last = row_offset + rows_h[last];
    if (i > g_last) continue;  // this tile never reached index i
    const int64_t off = (static_cast<int64_t>(h) * n_rt + rt) * n_total + i;
    vw += vpart[off];
    vm = fmaxf(vm, vmaxp[off]);
    sw += spart[off];
    sm = fmaxf(sm, smaxp[off]);
  }
  const int64_t o = static_cast<int64_t>(h) * n_total + i;
  v_w[o] = vw;
  v_max[o] = vm;
  s_w[o] = sw;
  s_max[o] = sm;
}

// total weight (sum of vertical weights, fixed tree order) and score count
__global__ void total_kernel(const double *v_w, const int32_t *rows, int n_s, int n_total, int row_offset,
                             double *total, int64_t *score_count) {
  __shared__ double sd[32];
  __shared__ long long sc[32];
  const int h = blockIdx.x;
  double acc = 0.0;
  long long cnt = 0;
  for (int i = threadIdx.x; i < n_total; i += blockDim.x) acc += v_w[static_cast<int64_t>(h) * n_total + i];
  for (int r = threadIdx.x; r < n_s; r += blockDim.x) {
    long long g = row_offset + rows[static_cast<int64_t>(h) * n_s + r];
    cnt += min(g, static_cast<long long>(n_total - 1)) + 1;  // prefill.py:386-389
  }
  acc = warp_sum_d(acc);
  cnt = warp_sum_ll(cnt);
  if ((threadIdx.x & 31) == 0) {
    sd[threadIdx.x >> 5] = acc;
    sc[threadIdx.x >> 5] = cnt;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    int nw = blockDim.x >> 5;
    acc = threadIdx.x < nw ? sd[threadIdx.x] : 0.0;
    cnt = threadIdx.x < nw ? sc[threadIdx.x] : 0;
    acc = warp_sum_d(acc);
    cnt = warp_sum_ll(cnt);
    if (threadIdx.x == 0) {
      total[h] = acc;
      score_count[h] = cnt;
    }
  }
}

inline size_t smem_bytes(int d) {
  int ld = d + 1;
  return static_cast<size_t>(BM * ld + BN * ld + BM * (BN + 1)) * 4 + BM * 16 + 64;
}

}  // namespace k1
}  // namespace ls

using namespace ls;

static size_t score_ws(const ls_layer_desc *L, int32_t n_s, int bm) {
  size_t n_rt = static_cast<size_t>(ceil_div(n_s, bm));
  size_t per = static_cast<size_t>(L->n_heads) * n_rt * L->n_total;
  return per * (8 + 4 + 8 + 4) + 4 * 256 + 4096;
}

namespace ls {
size_t score_lines_tc_workspace(const ls_layer_desc *L, int32_t n_s);
int score_lines_tc(const ls_layer_desc *L, int32_t n_s, const uint16_t *q, const uint16_t *k, const int32_t *rows,
                   double *v_w, float *v_max, double *s_w, float *s_max, float *row_stats, double *total,
                   int64_t *score_count, void *ws, size_t ws_bytes, cudaStream_t st);
}  // namespace ls

extern "C" size_t ls_score_lines_workspace(const ls_layer_desc *L, int32_t n_s) {
  const size_t a = score_ws(L, n_s, k1::BM), b = score_lines_tc_workspace(L, n_s);
  return a > b ? a : b;
}

static int score_lines_impl(const ls_layer_desc *L, int32_t n_s, const uint16_t *q, const uint16_t *k,
                            const int32_t *rows, double *v_w, float *v_max, double *s_w, float *s_max,
                            float *row_stats, double *total, int64_t *score_count, void *ws, size_t ws_bytes,
                            ls_stream_t stream, bool tensor_cores) {
  LS_REQUIRE(L->head_dim == 64 || L->head_dim == 128, LS_ERR_UNSUPPORTED, "head_dim must be 64 or 128");
  LS_REQUIRE(L->n_heads > 0 && L->n_kv_heads > 0 && L->n_heads % L->n_kv_heads == 0, LS_ERR_DIMENSION_MISMATCH,
             "n_heads must be a multiple of n_kv_heads");
  LS_REQUIRE(n_s > 0 && L->n_total > 0 && L->row_offset == L->n_total - L->n_new && L->n_new > 0,
             LS_ERR_DIMENSION_MISMATCH, "row_offset must equal n_total - n_new >= 0");
  LS_REQUIRE(ws_bytes >= ls_score_lines_workspace(L, n_s), LS_ERR_WORKSPACE, "score_lines workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (tensor_cores)
    return score_lines_tc(L, n_s, q, k, rows, v_w, v_max, s_w, s_max, row_stats, total, score_count, ws, ws_bytes, st);
  const int bm = k1::BM;
  const int n_rt = ceil_div(n_s, bm);
  Carver c(ws, ws_bytes);
  const size_t per = static_cast<size_t>(L->n_heads) * n_rt * L->n_total;
  k1::Params p;
  p.vpart = c.take<double>(per);
  p.spart = c.take<double>(per);
  p.vmaxp = c.take<float>(per);
  p.smaxp = c.take<float>(per);
  p.q = q;
  p.k = k;
  p.rows = rows;
  p.n_heads = L->n_heads;
  p.group = L->n_heads / L->n_kv_heads;
  p.d = L->head_dim;
  p.n_s = n_s;
  p.n_total = L->n_total;
  p.row_offset = L->row_offset;
  p.n_rt = n_rt;
  p.q_head_stride = L->q_head_stride;
  p.kv_head_stride = L->kv_head_stride;
  p.scale_log2 = kLog2e / sqrtf(static_cast<float>(L->head_dim));
  p.row_stats = row_stats;
  {
    const size_t smem = k1::smem_bytes(L->head_dim);
    LS_CUDA(cudaFuncSetAttribute(k1::score_lines_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    k1::score_lines_kernel<<<dim3(n_rt, L->n_heads), k1::THREADS, smem, st>>>(p);
    LS_LAUNCH_CHECK("score_lines_kernel");
  }
  k1::reduce_kernel<<<dim3(ceil_div(L->n_total, 256), L->n_heads), 256, 0, st>>>(
      p.vpart, p.vmaxp, p.spart, p.smaxp, rows, n_s, n_rt, L->n_total, L->row_offset, v_w, v_max, s_w, s_max, bm);
  LS_LAUNCH_CHECK("k1_reduce_kernel");
  k1::total_kernel<<<L->n_heads, 1024, 0, st>>>(v_w, rows, n_s, L->n_total, L->row_offset, total, score_count);
  LS_LAUNCH_CHECK("k1_total_kernel");
  return LS_OK;
}

extern "C" int ls_score_lines(const ls_layer_desc *L, int32_t n_s, const uint16_t *q, const uint16_t *k,
                              const int32_t *rows, double *v_w, float *v_max, double *s_w, float *s_max,
                              float *row_stats, double *total, int64_t *score_count, void *ws, size_t ws_bytes,
                              ls_stream_t stream) {
  return score_lines_impl(L, n_s, q, k, rows, v_w, v_max, s_w, s_max, row_stats, total, score_count, ws, ws_bytes,
                          stream, true);
}

extern "C" int ls_score_lines_simt(const ls_layer_desc *L, int32_t n_s, const uint16_t *q, const uint16_t *k,
                                   const int32_t *rows, double *v_w, float *v_max, double *s_w, float *s_max,
                                   float *row_stats, double *total, int64_t *score_count, void *ws,
                                   size_t ws_bytes, ls_stream_t stream) {
  return score_lines_impl(L, n_s, q, k, rows, v_w, v_max, s_w, s_max, row_stats, total, score_count, ws, ws_bytes,
                          stream, false);
}
