// Reference-API decode primitives on the device (the drop-in boundary of
// reference kvcompress.py / model.py that the engine's fused K6/K7/K8 launches
// do not expose one call at a time):
//
//   ls_accumulate_scores   accumulate_scores   kvcompress.py:67-83
//   ls_top_by_score        _top_by_score       kvcompress.py:86-90
//   ls_retained_union      retained_union      kvcompress.py:126-130
//   ls_kv_compact          compact_cache       kvcompress.py:133-147 (K8 gather)
//   ls_gather_attention    working-set branch  model.py:232-241 (decode_step)
//
// These serve callers that hold their state on the host in the reference's
// types (numpy ids / rows): they take plain device arrays, keep the
// reference's arithmetic order (rows oldest -> newest per id, fp64 sums),
// and are exact on ties ((score desc, id asc) via integer keys).
#include <algorithm>

#include "ls_common.cuh"

namespace ls {
namespace dropin {

constexpr int kThreads = 1024;
constexpr int kAccChunk = 4096;  // ids per CTA in accumulate_scores (32 KB of fp64)

__device__ __forceinline__ unsigned long long score_key(double x) {
  // order-preserving map of fp64 to uint64 (negative scores allowed); -0 == +0
  if (x == 0.0) x = 0.0;
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// exclusive block scan in thread order; *tot = block total (blockDim % 32 == 0)
__device__ int excl_scan(int v, int *sh, int *tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  __syncthreads();
  if (lane == 31) sh[wid] = incl;
  __syncthreads();
  int before = 0, all = 0;
  for (int i = 0; i < nw; ++i) {
    if (i < wid) before += sh[i];
    all += sh[i];
  }
  __syncthreads();
  *tot = all;
  return before + incl - v;
}

// ---------------------------------------------------- accumulate_scores
// One CTA per chunk of kAccChunk ids. Rows are added strictly in order
// (barrier between rows); inside a row every id is distinct (the reference's
// rows are working-set columns) so the per-id add order is the reference's
// dict-loop order: acc = 0.0 + w_row0 + w_row1 + ... (kvcompress.py:75-79).
__global__ void __launch_bounds__(kThreads) accumulate_kernel(int n_rows, const int64_t *row_ptr, const int32_t *ids,
                                                               const double *w, int id_cap, double *acc,
                                                               uint8_t *touched) {
  __shared__ double acc_sh[kAccChunk];
  __shared__ uint8_t t_sh[kAccChunk];
  const int lo = blockIdx.x * kAccChunk;
  const int hi = min(id_cap, lo + kAccChunk);
  for (int i = threadIdx.x; i < kAccChunk; i += blockDim.x) {
    acc_sh[i] = 0.0;
    t_sh[i] = 0;
  }
  __syncthreads();
  for (int r = 0; r < n_rows; ++r) {
    const int64_t b = row_ptr[r], e = row_ptr[r + 1];
    for (int64_t j = b + threadIdx.x; j < e; j += blockDim.x) {
      const int id = ids[j];
      if (id >= lo && id < hi) {
        atomicAdd(acc_sh + (id - lo), w[j]);  // one add per id per row: ordered by the barrier
        t_sh[id - lo] = 1;
      }
    }
    __syncthreads();
  }
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    acc[i] = acc_sh[i - lo];
    touched[i] = t_sh[i - lo];
  }
}

// ------------------------------------------------------- _top_by_score
// One CTA: radix-select the budget-th largest score key (8 x 8-bit digits),
// then among keys equal to it the smallest ids (4 x 8-bit digits of the
// sign-flipped id), then emit the picked ids in ascending id order through a
// bitmap over [id_lo, id_lo + id_range).
struct Select {
  unsigned long long prefix = 0ull, pmask = 0ull;
  int need = 0;
};

template <typename KeyFn>
__device__ void radix_select_desc(int n, KeyFn key_of, int bits, Select &s, int *hist, int *s_digit, int *s_above) {
  for (int shift = bits - 8; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      bool ok;
      const unsigned long long k = key_of(i, ok);
      if (ok && (k & s.pmask) == s.prefix) atomicAdd(&hist[(k >> shift) & 0xff], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int above = 0;
      for (int dgt = 255; dgt >= 0; --dgt) {
        if (above + hist[dgt] >= s.need) {
          *s_digit = dgt;
          *s_above = above;
          break;
        }
        above += hist[dgt];
      }
    }
    __syncthreads();
    s.prefix |= static_cast<unsigned long long>(*s_digit) << shift;
    s.pmask |= 0xffull << shift;
    s.need -= *s_above;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kThreads) top_by_score_kernel(int n, const int32_t *ids, const double *scores,
                                                                 int budget, int32_t id_lo, int32_t id_range,
                                                                 uint32_t *bitmap, int32_t *out, int32_t *n_out) {
  __shared__ int hist[256];
  __shared__ int sh[32];
  __shared__ int s_digit, s_above;
  const int words = (id_range + 31) / 32;
  for (int i = threadIdx.x; i < words; i += blockDim.x) bitmap[i] = 0u;
  // (1) budget-th largest score key; ids with a larger key are all picked
  Select s1;
  s1.need = budget;
  radix_select_desc(n, [&](int i, bool &ok) { ok = true; return score_key(scores[i]); }, 64, s1, hist, &s_digit,
                    &s_above);
  const unsigned long long thr = s1.prefix;
  // (2) among key == thr, the need smallest ids: the need largest ~id keys
  Select s2;
  s2.need = s1.need;
  radix_select_desc(
      n,
      [&](int i, bool &ok) {
        ok = score_key(scores[i]) == thr;
        return static_cast<unsigned long long>(~(static_cast<uint32_t>(ids[i]) ^ 0x80000000u));
      },
      32, s2, hist, &s_digit, &s_above);
  const uint32_t id_thr = static_cast<uint32_t>(s2.prefix);  // ~(flipped id) of the last tied id taken
  __syncthreads();
  // (3) mark: key > thr, or key == thr and id < the tied threshold id, and the
  // first s2.need occurrences (index order) of the threshold id itself
  int eq_seen = 0;
  for (int i0 = 0; i0 < n; i0 += blockDim.x) {
    const int i = i0 + threadIdx.x;
    int pick = 0, at_thr = 0;
    if (i < n) {
      const unsigned long long k = score_key(scores[i]);
      const uint32_t ik = ~(static_cast<uint32_t>(ids[i]) ^ 0x80000000u);
      pick = k > thr || (k == thr && ik > id_thr);
      at_thr = k == thr && ik == id_thr;
    }
    int tot;
    const int rank = excl_scan(at_thr, sh, &tot);
    if (at_thr && eq_seen + rank < s2.need) pick = 1;
    eq_seen += tot;
    if (pick) {
      const int o = ids[i] - id_lo;
      atomicOr(bitmap + (o >> 5), 1u << (o & 31));
    }
  }
  __syncthreads();
  // (4) ids in ascending order
  int base = 0;
  for (int w0 = 0; w0 < words; w0 += blockDim.x) {
    const int w = w0 + threadIdx.x;
    uint32_t x = w < words ? bitmap[w] : 0u;
    int tot;
    int pos = base + excl_scan(__popc(x), sh, &tot);
    while (x) {
      const int b = __ffs(x) - 1;
      x &= x - 1;
      if (pos < budget) out[pos] = id_lo + w * 32 + b;
      ++pos;
    }
    base += tot;
  }
  if (threadIdx.x == 0) *n_out = base;
}

// ------------------------------------------------------ retained_union
__global__ void __launch_bounds__(kThreads) union_kernel(int n_sel, const int32_t *sel, int32_t recent_window,
                                                          int32_t full_len, int32_t cap, uint32_t *bitmap,
                                                          int32_t *out, int32_t *n_out) {
  __shared__ int sh[32];
  const int words = (cap + 31) / 32;
  for (int i = threadIdx.x; i < words; i += blockDim.x) bitmap[i] = 0u;
  __syncthreads();
  for (int i = threadIdx.x; i < n_sel; i += blockDim.x) {
    const int g = sel[i];
    if (g >= 0 && g < cap) atomicOr(bitmap + (g >> 5), 1u << (g & 31));
  }
  for (int g = max(0, full_len - recent_window) + threadIdx.x; g < full_len; g += blockDim.x)
    atomicOr(bitmap + (g >> 5), 1u << (g & 31));
  __syncthreads();
  int base = 0;
  for (int w0 = 0; w0 < words; w0 += blockDim.x) {
    const int w = w0 + threadIdx.x;
    uint32_t x = w < words ? bitmap[w] : 0u;
    int tot;
    int pos = base + excl_scan(__popc(x), sh, &tot);
    while (x) {
      const int b = __ffs(x) - 1;
      x &= x - 1;
      out[pos++] = w * 32 + b;
    }
    base += tot;
  }
  if (threadIdx.x == 0) *n_out = base;
}

// ----------------------------------------------------------- K8 gather
// keep_ids -> rows of the source cache (src_ids strictly increasing, binary
// search), then a coalesced 16-byte row copy of K and V. A keep id missing
// from the source sets *status to 1 + its index (the host raises InvalidIds).
__global__ void kv_compact_kernel(int n_src, const int32_t *src_ids, const uint8_t *src_k, const uint8_t *src_v,
                                  int n_keep, const int32_t *keep_ids, int k_row_bytes, int v_row_bytes,
                                  uint8_t *dst_k, uint8_t *dst_v, int32_t *status) {
  const int vk = k_row_bytes / 16, vv = v_row_bytes / 16, vec = max(vk, vv);
  const int64_t total = static_cast<int64_t>(n_keep) * vec;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(t / vec), c = static_cast<int>(t - static_cast<int64_t>(r) * vec);
    const int g = keep_ids[r];
    const int j = lower_bound_dev(src_ids, n_src, g);
    if (j >= n_src || src_ids[j] != g) {
      if (c == 0) atomicCAS(status, 0, r + 1);
      continue;
    }
    if (c < vk)
      *reinterpret_cast<uint4 *>(dst_k + static_cast<int64_t>(r) * k_row_bytes + 16ll * c) =
          __ldg(reinterpret_cast<const uint4 *>(src_k + static_cast<int64_t>(j) * k_row_bytes + 16ll * c));
    if (c < vv)
      *reinterpret_cast<uint4 *>(dst_v + static_cast<int64_t>(r) * v_row_bytes + 16ll * c) =
          __ldg(reinterpret_cast<const uint4 *>(src_v + static_cast<int64_t>(j) * v_row_bytes + 16ll * c));
  }
}

// ------------------------------------------------- working-set attention
// model.py:232-241 for every head of a layer in one launch: head h attends to
// cols[col_ptr[h] .. col_ptr[h+1]) of its K/V archive. bf16 operands, fp64
// arithmetic (the reference's working-set branch is fp64): logits
// (K[cols] . q) / sqrt(d), w = exp(s - max) / sum, out = w . V[cols]; w is
// also written out (the observation row the decode loop buffers).
constexpr int kGaThreads = 256;

__global__ void __launch_bounds__(kGaThreads) gather_attention_kernel(int d, const uint16_t *q, int64_t q_head_stride,
                                                                       const uint16_t *k, const uint16_t *v,
                                                                       int64_t kv_head_stride, int group,
                                                                       const int64_t *col_ptr, const int32_t *cols,
                                                                       double *out, double *w_out) {
  extern __shared__ double qs[];  // [d] q, then [kGaThreads / 32] partials, then [4][d] out partials
  __shared__ double red[kGaThreads / 32];
  const int h = blockIdx.x;
  const int64_t b = col_ptr[h], e = col_ptr[h + 1];
  const int n = static_cast<int>(e - b);
  const uint16_t *kh = k + static_cast<int64_t>(h / group) * kv_head_stride;
  const uint16_t *vh = v + static_cast<int64_t>(h / group) * kv_head_stride;
  for (int i = threadIdx.x; i < d; i += blockDim.x) qs[i] = static_cast<double>(bf2f(q[h * q_head_stride + i]));
  __syncthreads();
  const double scale = 1.0 / sqrt(static_cast<double>(d));
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // logits: one warp per column, lanes split d, fixed shuffle tree
  double mx = -INFINITY;
  for (int j = wid; j < n; j += nw) {
    const uint16_t *kr = kh + static_cast<int64_t>(cols[b + j]) * d;
    double a = 0.0;
    for (int i = lane; i < d; i += 32) a += qs[i] * static_cast<double>(bf2f(kr[i]));
    a = warp_sum_d(a) * scale;
    if (lane == 0) w_out[b + j] = a;
    mx = fmax(mx, a);
  }
  if (lane == 0) red[wid] = mx;
  __syncthreads();
  mx = -INFINITY;
  for (int i = 0; i < nw; ++i) mx = fmax(mx, red[i]);
  __syncthreads();
  // exp and the sum: thread-strided partials, then a fixed-order combine
  double part = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double ex = exp(w_out[b + j] - mx);
    w_out[b + j] = ex;
    part += ex;
  }
  part = warp_sum_d(part);
  if (lane == 0) red[wid] = part;
  __syncthreads();
  double sum = 0.0;
  for (int i = 0; i < nw; ++i) sum += red[i];
  const double inv = 1.0 / sum;
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) w_out[b + j] = w_out[b + j] / sum;
  __syncthreads();
  (void)inv;
  // out = w . V[cols]: column groups g = tid / d, dims tid % d
  double *op = qs + d;  // [groups][d]
  const int groups = blockDim.x / d;
  const int g = threadIdx.x / d, dim = threadIdx.x - g * d;
  if (g < groups) {
    double a = 0.0;
    for (int j = g; j < n; j += groups) a += w_out[b + j] * static_cast<double>(bf2f(vh[static_cast<int64_t>(cols[b + j]) * d + dim]));
    op[g * d + dim] = a;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    double a = 0.0;
    for (int gg = 0; gg < groups; ++gg) a += op[gg * d + i];
    out[static_cast<int64_t>(h) * d + i] = a;
  }
}

// ------------------------------------------------ obswindow selection
// session.py:215-225: per (layer, head) unit, the buffered dense observation
// rows accumulated in row order (accumulate_scores), then summed over the
// units in unit order (numpy's axis-0 sum of the stacked per-head arrays).
// Thread per column: ((s_0 + s_1) + s_2) + ..., s_u = ((0 + w_u0) + w_u1) + ...
__global__ void obs_sum_kernel(int n_units, int n_rows, const float *rows, int64_t unit_stride, int64_t row_stride,
                               int n_cols, double *scores) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_cols) return;
  double acc = 0.0;
  for (int u = 0; u < n_units; ++u) {
    const float *ru = rows + u * unit_stride + c;
    double su = 0.0;
    for (int r = 0; r < n_rows; ++r) su += static_cast<double>(__ldg(ru + r * row_stride));
    acc = u == 0 ? su : acc + su;
  }
  scores[c] = acc;
}

// dst[slice][r] = src[slice][ids[r]] for 16-byte-multiple rows (the obswindow
// baseline's one-shot compaction of the shared working set)
__global__ void gather_rows_kernel(int n_slices, int n_ids, const int32_t *ids, const uint8_t *src,
                                   int64_t src_slice_bytes, uint8_t *dst, int64_t dst_slice_bytes, int row_bytes) {
  const int vec = row_bytes / 16;
  const int64_t per_slice = static_cast<int64_t>(n_ids) * vec;
  const int64_t total = per_slice * n_slices;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int sl = static_cast<int>(t / per_slice);
    const int64_t rem = t - sl * per_slice;
    const int r = static_cast<int>(rem / vec), c = static_cast<int>(rem - static_cast<int64_t>(r) * vec);
    const uint4 v = __ldg(reinterpret_cast<const uint4 *>(src + sl * src_slice_bytes +
                                                          static_cast<int64_t>(ids[r]) * row_bytes) + c);
    reinterpret_cast<uint4 *>(dst + sl * dst_slice_bytes + static_cast<int64_t>(r) * row_bytes)[c] = v;
  }
}

}  // namespace dropin
}  // namespace ls

using namespace ls;

extern "C" int ls_obs_window_scores(int32_t n_units, int32_t n_rows, const float *rows, int64_t unit_stride,
                                    int64_t row_stride, int32_t n_cols, double *scores, ls_stream_t stream) {
  LS_REQUIRE(n_units >= 1 && n_rows >= 1, LS_ERR_EMPTY_WINDOW, "need at least one observation row");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  dropin::obs_sum_kernel<<<ceil_div(n_cols, 256), 256, 0, st>>>(n_units, n_rows, rows, unit_stride, row_stride, n_cols,
                                                               scores);
  LS_LAUNCH_CHECK("obs_sum_kernel");
  return LS_OK;
}

extern "C" int ls_gather_rows(int32_t n_slices, int32_t n_ids, const int32_t *ids, const void *src,
                              int64_t src_slice_bytes, void *dst, int64_t dst_slice_bytes, int32_t row_bytes,
                              ls_stream_t stream) {
  LS_REQUIRE(row_bytes > 0 && row_bytes % 16 == 0, LS_ERR_UNSUPPORTED, "row_bytes must be a multiple of 16");
  if (n_ids == 0 || n_slices == 0) return LS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const long long total = static_cast<long long>(n_slices) * n_ids * (row_bytes / 16);
  const int grid = static_cast<int>(std::min<long long>(ceil_div_ll(total, 256), 148 * 8));
  dropin::gather_rows_kernel<<<grid, 256, 0, st>>>(n_slices, n_ids, ids, static_cast<const uint8_t *>(src),
                                                   src_slice_bytes, static_cast<uint8_t *>(dst), dst_slice_bytes,
                                                   row_bytes);
  LS_LAUNCH_CHECK("gather_rows_kernel");
  return LS_OK;
}

extern "C" int ls_accumulate_scores(int32_t n_rows, const int64_t *row_ptr, const int32_t *ids, const double *w,
                                    int32_t id_cap, double *acc, uint8_t *touched, ls_stream_t stream) {
  LS_REQUIRE(n_rows >= 1, LS_ERR_EMPTY_WINDOW, "need at least one observation row");
  LS_REQUIRE(id_cap >= 1, LS_ERR_INVALID_IDS, "id_cap must be >= 1");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  dropin::accumulate_kernel<<<ceil_div(id_cap, dropin::kAccChunk), dropin::kThreads, 0, st>>>(n_rows, row_ptr, ids, w,
                                                                                              id_cap, acc, touched);
  LS_LAUNCH_CHECK("accumulate_kernel");
  return LS_OK;
}

extern "C" size_t ls_top_by_score_workspace(int32_t id_range) {
  return static_cast<size_t>((id_range + 31) / 32) * 4 + 256;
}

extern "C" int ls_top_by_score(int32_t n, const int32_t *ids, const double *scores, int32_t budget, int32_t id_lo,
                               int32_t id_range, int32_t *out, int32_t *n_out, void *ws, size_t ws_bytes,
                               ls_stream_t stream) {
  LS_REQUIRE(budget >= 1 && budget <= n, LS_ERR_INVALID_CONFIG, "budget %d outside [1, n=%d]", budget, n);
  LS_REQUIRE(id_range >= 1, LS_ERR_INVALID_IDS, "id_range must be >= 1");
  LS_REQUIRE(ws_bytes >= ls_top_by_score_workspace(id_range), LS_ERR_WORKSPACE, "top_by_score workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  dropin::top_by_score_kernel<<<1, dropin::kThreads, 0, st>>>(n, ids, scores, budget, id_lo, id_range,
                                                              static_cast<uint32_t *>(ws), out, n_out);
  LS_LAUNCH_CHECK("top_by_score_kernel");
  return LS_OK;
}

extern "C" int ls_retained_union(int32_t n_sel, const int32_t *sel, int32_t recent_window, int32_t full_len,
                                 int32_t cap, int32_t *out, int32_t *n_out, void *ws, size_t ws_bytes,
                                 ls_stream_t stream) {
  LS_REQUIRE(full_len >= 0 && recent_window >= 0 && cap >= full_len, LS_ERR_INVALID_CONFIG, "bad union bounds");
  LS_REQUIRE(ws_bytes >= static_cast<size_t>((cap + 31) / 32) * 4, LS_ERR_WORKSPACE, "retained_union workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  dropin::union_kernel<<<1, dropin::kThreads, 0, st>>>(n_sel, sel, recent_window, full_len, cap,
                                                       static_cast<uint32_t *>(ws), out, n_out);
  LS_LAUNCH_CHECK("union_kernel");
  return LS_OK;
}

extern "C" int ls_kv_compact(int32_t n_src, const int32_t *src_ids, const void *src_k, const void *src_v,
                             int32_t n_keep, const int32_t *keep_ids, int32_t k_row_bytes, int32_t v_row_bytes,
                             void *dst_k, void *dst_v, int32_t *status, ls_stream_t stream) {
  LS_REQUIRE(k_row_bytes > 0 && k_row_bytes % 16 == 0 && v_row_bytes > 0 && v_row_bytes % 16 == 0,
             LS_ERR_UNSUPPORTED, "row bytes must be multiples of 16");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  LS_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t), st));
  if (n_keep == 0) return LS_OK;
  const long long total = static_cast<long long>(n_keep) * (std::max(k_row_bytes, v_row_bytes) / 16);
  const int grid = static_cast<int>(std::min<long long>(ceil_div_ll(total, 256), 148 * 8));
  dropin::kv_compact_kernel<<<grid, 256, 0, st>>>(n_src, src_ids, static_cast<const uint8_t *>(src_k),
                                                  static_cast<const uint8_t *>(src_v), n_keep, keep_ids, k_row_bytes,
                                                  v_row_bytes, static_cast<uint8_t *>(dst_k),
                                                  static_cast<uint8_t *>(dst_v), status);
  LS_LAUNCH_CHECK("kv_compact_kernel");
  return LS_OK;
}

extern "C" int ls_gather_attention(int32_t n_heads, int32_t n_kv_heads, int32_t head_dim, const uint16_t *q,
                                   int64_t q_head_stride, const uint16_t *k, const uint16_t *v, int64_t kv_head_stride,
                                   const int64_t *col_ptr, const int32_t *cols, double *out, double *w_out,
                                   ls_stream_t stream) {
  LS_REQUIRE(n_heads >= 1 && n_kv_heads >= 1 && n_heads % n_kv_heads == 0, LS_ERR_DIMENSION_MISMATCH,
             "n_heads %% n_kv_heads != 0");
  LS_REQUIRE(head_dim >= 1 && head_dim <= dropin::kGaThreads, LS_ERR_UNSUPPORTED, "head_dim outside [1, 256]");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int groups = dropin::kGaThreads / head_dim;
  const size_t smem = static_cast<size_t>(head_dim) * (1 + groups) * sizeof(double);
  if (smem > 48 * 1024)
    LS_CUDA(cudaFuncSetAttribute(dropin::gather_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  dropin::gather_attention_kernel<<<n_heads, dropin::kGaThreads, smem, st>>>(
      head_dim, q, q_head_stride, k, v, kv_head_stride, n_heads / n_kv_heads, col_ptr, cols, out, w_out);
  LS_LAUNCH_CHECK("gather_attention_kernel");
  return LS_OK;
}
