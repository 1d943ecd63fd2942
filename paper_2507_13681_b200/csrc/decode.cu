// K6 + K7 + K8 -- progressive decode with periodic KV compression.
//
// K6 decode attention replaces the working-set branch of forward_extend
// (reference model.py:232-241) inside decode_step (model.py:289-311): per
// q-head, cols = working set U {new position}, softmax over
// K[cols].q / sqrt(d), out = w . V[cols], and the observation row (cols, w)
// (kvcompress.py:233) is written to the head's ring slot. Working set:
//   before the first event: [0, length)                 (kvcompress.py:194, 237)
//   after it: selected U [length - W, length)           (kvcompress.py:235)
// The selected rows are read from the compacted per-head cache ck/cv
// (segment A, ids < length - W so the recent window is not double counted);
// the recent window and the new row are read from the archive (segment B).
// Split-K over columns (K6a) + a combine kernel (K6b) that normalises the
// output and rescales the ring row in place.
//
// K7 (event) replaces accumulate_scores + _top_by_score + retained_union
// (kvcompress.py:67-90, 126-130, 210-224): rows are accumulated oldest ->
// newest in fp64 (each row has distinct ids, so a row is added in parallel
// without races and the per-id order is the reference's), candidates are
// the touched ids only (kvcompress.py:73-83), then an 8-pass radix select
// on the fp64 bits finds the B-th largest (score desc, id asc) and the
// picked ids are emitted in id order.
//
// K8 replaces compact_cache (kvcompress.py:133-147): coalesced 16-byte
// gather of the picked rows into the contiguous per-head cache.

#include "ls_common.cuh"

namespace ls {
namespace dec {

constexpr int COLS_PER_SPLIT = 256;
constexpr int K6_THREADS = 128;  // 4 warps, 8 column groups of 4 lanes per warp

struct Part {  // per (head, split)
  float m, l;
  float o[128];
};

struct Geo {  // column geometry of one head for this step
  int n_a;   // compacted selected rows used (ids < lo)
  int lo;    // archive segment start
  int n_cols;
};

__device__ __forceinline__ Geo geometry(const ls_decode_state &S, int h, int length, int compressed) {
  Geo g;
  if (compressed) {
    g.lo = max(0, length - S.window);
    const int32_t *sel = S.sel_ids + static_cast<int64_t>(h) * S.budget_cap;
    g.n_a = lower_bound_dev(sel, S.n_sel[h], g.lo);
  } else {
    g.lo = 0;
    g.n_a = 0;
  }
  g.n_cols = g.n_a + (length - g.lo + 1);
  return g;
}

__global__ void __launch_bounds__(K6_THREADS) decode_partial_kernel(ls_decode_state S, const uint16_t *q,
                                                                    const uint16_t *k, const uint16_t *v,
                                                                    int length, int compressed, int slot,
                                                                    float scale_log2, Part *parts, int n_split) {
  __shared__ float red_m[4];
  __shared__ float red_l[4];
  __shared__ float red_o[4][128];
  const int h = blockIdx.y, split = blockIdx.x;
  const int d = S.head_dim;
  const Geo g = geometry(S, h, length, compressed);
  const int c_begin = split * COLS_PER_SPLIT;
  const int c_end = min(g.n_cols, c_begin + COLS_PER_SPLIT);
  Part &part = parts[static_cast<int64_t>(h) * n_split + split];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane >> 2, sub = lane & 3;  // 8 groups of 4 lanes
  const int dpl = d / 4;                      // dims per lane: 32 (d=128) or 16
  const int kv = h / (S.n_heads / S.n_kv_heads);
  const uint16_t *kb = k + static_cast<int64_t>(kv) * S.kv_head_stride;
  const uint16_t *vb = v + static_cast<int64_t>(kv) * S.kv_head_stride;
  const uint16_t *ckb = S.ck + static_cast<int64_t>(h) * S.budget_cap * d;
  const uint16_t *cvb = S.cv + static_cast<int64_t>(h) * S.budget_cap * d;
  const int32_t *sel = S.sel_ids + static_cast<int64_t>(h) * S.budget_cap;
  float *wrow = S.ring_w + (static_cast<int64_t>(h) * S.window + slot) * S.row_cap;
  int32_t *idrow = S.ring_ids + (static_cast<int64_t>(h) * S.window + slot) * S.sparse_cap;

  if (c_begin >= g.n_cols) {
    if (threadIdx.x == 0) {
      part.m = -INFINITY;
      part.l = 0.f;
    }
    for (int i = threadIdx.x; i < d; i += blockDim.x) part.o[i] = 0.f;
    return;
  }
  // q slice of this lane
  float qv[32];
  const uint16_t *qh = q + static_cast<int64_t>(h) * d + sub * dpl;
  for (int i = 0; i < dpl; ++i) qv[i] = bf2f(qh[i]);

  constexpr int PER = COLS_PER_SPLIT / 32;  // columns per lane group
  float sv[PER];
  int cid[PER];
  float m = -INFINITY;
#pragma unroll
  for (int t = 0; t < PER; ++t) {
    const int j = c_begin + (t * 4 + warp) * 8 + grp;
    const bool valid = j < c_end;
    sv[t] = -INFINITY;
    cid[t] = -1;
    float acc = 0.f;
    if (valid) {
      const uint16_t *kr;
      int id;
      if (j < g.n_a) {
        id = sel[j];
        kr = ckb + static_cast<int64_t>(j) * d;
      } else {
        id = g.lo + (j - g.n_a);
        kr = kb + static_cast<int64_t>(id) * d;
      }
      cid[t] = id;
      for (int vv = 0; vv < dpl / 8; ++vv) {
        uint4 u = *reinterpret_cast<const uint4 *>(kr + sub * dpl + vv * 8);
        float f[8];
        bf16x8_to_f32(u, f);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc = fmaf(qv[vv * 8 + e], f[e], acc);
      }
    }
    // lanes of a group share j; shuffles stay converged across the warp
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (valid) {
      sv[t] = acc * scale_log2;
      m = fmaxf(m, sv[t]);
    }
  }
  m = warp_max(m);
  if (lane == 0) red_m[warp] = m;
  __syncthreads();
  m = fmaxf(fmaxf(red_m[0], red_m[1]), fmaxf(red_m[2], red_m[3]));
  float l = 0.f;
  float o[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) o[i] = 0.f;
#pragma unroll
  for (int t = 0; t < PER; ++t) {
    const int j = c_begin + (t * 4 + warp) * 8 + grp;
    if (j < c_end) {
      const float p = fast_exp2(sv[t] - m);
      if (sub == 0) {
        l += p;
        wrow[j] = p;
        if (compressed) idrow[j] = cid[t];
      }
      const uint16_t *vr = (j < g.n_a) ? cvb + static_cast<int64_t>(j) * d : vb + static_cast<int64_t>(cid[t]) * d;
      for (int vv = 0; vv < dpl / 8; ++vv) {
        uint4 u = *reinterpret_cast<const uint4 *>(vr + sub * dpl + vv * 8);
        float f[8];
        bf16x8_to_f32(u, f);
#pragma unroll
        for (int e = 0; e < 8; ++e) o[vv * 8 + e] = fmaf(p, f[e], o[vv * 8 + e]);
      }
    }
  }
  // reduce over the 8 groups of the warp (lanes with equal sub)
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    l += __shfl_xor_sync(0xffffffffu, l, off);
#pragma unroll
    for (int i = 0; i < 32; ++i) o[i] += __shfl_xor_sync(0xffffffffu, o[i], off);
  }
  if (lane == 0) red_l[warp] = l;
  if (grp == 0)
    for (int i = 0; i < dpl; ++i) red_o[warp][sub * dpl + i] = o[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    part.m = m;
    part.l = red_l[0] + red_l[1] + red_l[2] + red_l[3];
  }
  for (int i = threadIdx.x; i < d; i += blockDim.x)
    part.o[i] = red_o[0][i] + red_o[1][i] + red_o[2][i] + red_o[3][i];
}

__global__ void __launch_bounds__(256) decode_combine_kernel(ls_decode_state S, int length, int compressed,
                                                             int slot, const Part *parts, int n_split, void *out,
                                                             int out_bf16) {
  __shared__ float scl[512];
  __shared__ float Msh, Lsh;
  const int h = blockIdx.x;
  const int d = S.head_dim;
  const Geo g = geometry(S, h, length, compressed);
  const int ns = (g.n_cols + COLS_PER_SPLIT - 1) / COLS_PER_SPLIT;
  const Part *pp = parts + static_cast<int64_t>(h) * n_split;
  if (threadIdx.x == 0) {
    float M = -INFINITY;
    for (int s = 0; s < ns; ++s) M = fmaxf(M, pp[s].m);
    float Ls = 0.f;
    for (int s = 0; s < ns; ++s) Ls += pp[s].l * fast_exp2(pp[s].m - M);
    Msh = M;
    Lsh = Ls;
  }
  __syncthreads();
  const float M = Msh, inv = 1.f / Lsh;
  for (int s = threadIdx.x; s < ns; s += blockDim.x) scl[s] = fast_exp2(pp[s].m - M) * inv;
  __syncthreads();
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < ns; ++s) acc += pp[s].o[i] * scl[s];
    if (out_bf16)
      reinterpret_cast<uint16_t *>(out)[static_cast<int64_t>(h) * d + i] = f2bf(acc);
    else
      reinterpret_cast<float *>(out)[static_cast<int64_t>(h) * d + i] = acc;
  }
  float *wrow = S.ring_w + (static_cast<int64_t>(h) * S.window + slot) * S.row_cap;
  for (int j = threadIdx.x; j < g.n_cols; j += blockDim.x) wrow[j] *= scl[j / COLS_PER_SPLIT];
  if (threadIdx.x == 0) {
    S.ring_n[h * S.window + slot] = g.n_cols;
    S.ring_dense[h * S.window + slot] = compressed ? 0 : 1;
  }
}

// ------------------------------------------------------------------ K7
constexpr int K7_THREADS = 1024;

__device__ __forceinline__ unsigned long long dkey(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x));  // x >= 0: monotone
}

__device__ int block_sum_int(int v, int *sh) {
  v = __reduce_add_sync(0xffffffffu, v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  int tot = 0;
  const int nw = blockDim.x >> 5;
  for (int i = 0; i < nw; ++i) tot += sh[i];
  __syncthreads();
  return tot;
}

__device__ double block_sum_double(double v, double *sh) {
  v = warp_sum_d(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double tot = 0.0;
  const int nw = blockDim.x >> 5;
  for (int i = 0; i < nw; ++i) tot += sh[i];
  __syncthreads();
  return tot;
}

// exclusive block scan of a 0/1 flag; returns the rank, total via *tot
__device__ int block_rank(int flag, int *sh, int *tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned b = __ballot_sync(0xffffffffu, flag);
  __syncthreads();
  if (lane == 0) sh[wid] = __popc(b);
  __syncthreads();
  int before = 0, all = 0;
  const int nw = blockDim.x >> 5;
  for (int i = 0; i < nw; ++i) {
    if (i < wid) before += sh[i];
    all += sh[i];
  }
  *tot = all;
  return before + __popc(b & ((1u << lane) - 1u));
}

__global__ void __launch_bounds__(K7_THREADS) decode_select_kernel(ls_decode_state S, const int32_t *slot_order,
                                                                   int n_rows, int length, int budget,
                                                                   double *acc_ws, uint8_t *touched_ws,
                                                                   int32_t *retained_n, double *score_cov) {
  __shared__ int hist[256];
  __shared__ int shi[32];
  __shared__ double shd[32];
  __shared__ int s_digit, s_above;
  const int h = blockIdx.x;
  double *acc = acc_ws + static_cast<int64_t>(h) * S.row_cap;
  uint8_t *touched = touched_ws + static_cast<int64_t>(h) * S.row_cap;
  for (int i = threadIdx.x; i < length; i += blockDim.x) {
    acc[i] = 0.0;
    touched[i] = 0;
  }
  __syncthreads();
  // accumulate rows oldest -> newest (kvcompress.py:75-79)
  for (int rr = 0; rr < n_rows; ++rr) {
    const int slot = slot_order[rr];
    const int n = S.ring_n[h * S.window + slot];
    const int dense = S.ring_dense[h * S.window + slot];
    const float *w = S.ring_w + (static_cast<int64_t>(h) * S.window + slot) * S.row_cap;
    const int32_t *ids = S.ring_ids + (static_cast<int64_t>(h) * S.window + slot) * S.sparse_cap;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const int id = dense ? j : ids[j];
      acc[id] += static_cast<double>(w[j]);
      touched[id] = 1;
    }
    __syncthreads();
  }
  // candidates
  int cnt = 0;
  for (int i = threadIdx.x; i < length; i += blockDim.x) cnt += touched[i];
  const int n_cand = block_sum_int(cnt, shi);
  // radix select of the budget-th largest key among candidates
  unsigned long long prefix = 0ull, pmask = 0ull;
  int need = budget;  // rank from the top still to place
  const bool take_all = budget >= n_cand;
  if (!take_all) {
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < length; i += blockDim.x) {
        if (!touched[i]) continue;
        const unsigned long long key = dkey(acc[i]);
        if ((key & pmask) != prefix) continue;
        atomicAdd(&hist[(key >> shift) & 0xff], 1);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        int above = 0, dg = 255;
        for (; dg >= 0; --dg) {
          if (above + hist[dg] >= need) break;
          above += hist[dg];
        }
        s_digit = dg;
        s_above = above;
      }
      __syncthreads();
      prefix |= static_cast<unsigned long long>(s_digit) << shift;
      pmask |= 0xffull << shift;
      need -= s_above;
      __syncthreads();
    }
  }
  const unsigned long long thr = prefix;  // key of the budget-th largest
  // emit picked ids in id order: key > thr, or key == thr among the first `need` ids
  int32_t *sel = S.sel_ids + static_cast<int64_t>(h) * S.budget_cap;
  int base = 0, eq_seen = 0;
  double tot_mass = 0.0, kept_mass = 0.0;
  int in_window_picked = 0;
  const int lo = max(0, length - S.window);
  for (int i0 = 0; i0 < length; i0 += blockDim.x) {
    const int i = i0 + threadIdx.x;
    int is_t = 0, is_eq = 0, is_gt = 0;
    double sc = 0.0;
    if (i < length && touched[i]) {
      is_t = 1;
      sc = acc[i];
      if (!take_all) {
        const unsigned long long key = dkey(sc);
        is_gt = key > thr;
        is_eq = key == thr;
      }
    }
    int eq_tot;
    const int eq_rank = block_rank(is_eq, shi, &eq_tot);
    const int pick = take_all ? is_t : (is_gt || (is_eq && eq_seen + eq_rank < need));
    int pick_tot;
    const int rank = block_rank(pick, shi, &pick_tot);
    if (pick) sel[base + rank] = i;
    if (is_t) {
      tot_mass += sc;
      if (pick || i >= lo) kept_mass += sc;  // kvcompress.py:215 (working = picked U recent)
    }
    if (pick && i >= lo) in_window_picked += 1;
    base += pick_tot;
    eq_seen += eq_tot;
  }
  const double T = block_sum_double(tot_mass, shd);
  const double Kp = block_sum_double(kept_mass, shd);
  const int iw = block_sum_int(in_window_picked, shi);
  if (threadIdx.x == 0) {
    S.n_sel[h] = base;
    const int w_len = length - lo;
    if (retained_n) retained_n[h] = base + w_len - iw;
    if (score_cov) score_cov[h] = T > 0 ? Kp / T : 1.0;
  }
}

// ------------------------------------------------------------------ K8
__global__ void kv_compact_kernel(ls_decode_state S, const uint16_t *k, const uint16_t *v) {
  const int h = blockIdx.y;
  const int d = S.head_dim;
  const int vec = d / 8;  // 16-byte vectors per row
  const int n = S.n_sel[h];
  const int kv = h / (S.n_heads / S.n_kv_heads);
  const int32_t *sel = S.sel_ids + static_cast<int64_t>(h) * S.budget_cap;
  const uint4 *kb = reinterpret_cast<const uint4 *>(k + static_cast<int64_t>(kv) * S.kv_head_stride);
  const uint4 *vb = reinterpret_cast<const uint4 *>(v + static_cast<int64_t>(kv) * S.kv_head_stride);
  uint4 *ck = reinterpret_cast<uint4 *>(S.ck + static_cast<int64_t>(h) * S.budget_cap * d);
  uint4 *cv = reinterpret_cast<uint4 *>(S.cv + static_cast<int64_t>(h) * S.budget_cap * d);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n * vec; i += gridDim.x * blockDim.x) {
    const int j = i / vec, e = i % vec;
    const int64_t src = static_cast<int64_t>(sel[j]) * vec + e;
    ck[static_cast<int64_t>(j) * vec + e] = kb[src];
    cv[static_cast<int64_t>(j) * vec + e] = vb[src];
  }
}

}  // namespace dec
}  // namespace ls

using namespace ls;

static int check_state(const ls_decode_state *S) {
  LS_REQUIRE(S->head_dim == 64 || S->head_dim == 128, LS_ERR_UNSUPPORTED, "head_dim must be 64 or 128");
  LS_REQUIRE(S->n_heads > 0 && S->n_kv_heads > 0 && S->n_heads % S->n_kv_heads == 0, LS_ERR_DIMENSION_MISMATCH,
             "n_heads must be a multiple of n_kv_heads");
  LS_REQUIRE(S->window >= 1, LS_ERR_INVALID_CONFIG, "obs_window must be >= 1");
  return LS_OK;
}

extern "C" size_t ls_decode_attention_workspace(const ls_decode_state *S, int32_t max_len) {
  const size_t n_split = static_cast<size_t>(ceil_div(max_len + 1, dec::COLS_PER_SPLIT));
  return static_cast<size_t>(S->n_heads) * n_split * sizeof(dec::Part) + 1024;
}

extern "C" int ls_decode_attention(const ls_decode_state *S, const uint16_t *q, const uint16_t *k,
                                   const uint16_t *v, int32_t length, int32_t compressed, int32_t slot, void *out,
                                   int32_t out_bf16, void *ws, size_t ws_bytes, ls_stream_t stream) {
  int c = check_state(S);
  if (c) return c;
  LS_REQUIRE(length >= 0 && length + 1 <= S->row_cap, LS_ERR_SEQUENCE_TOO_LONG,
             "length %d exceeds the ring row capacity %d", length, S->row_cap);
  LS_REQUIRE(slot >= 0 && slot < S->window, LS_ERR_INVALID_CONFIG, "ring slot out of range");
  LS_REQUIRE(!compressed || S->budget_cap + S->window + 1 <= S->sparse_cap, LS_ERR_INVALID_CONFIG,
             "sparse_cap must be >= budget_cap + window + 1");
  const int n_split = ceil_div(length + 1, dec::COLS_PER_SPLIT);
  LS_REQUIRE(ws_bytes >= ls_decode_attention_workspace(S, length), LS_ERR_WORKSPACE,
             "decode_attention workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  dec::Part *parts = reinterpret_cast<dec::Part *>(ws);
  const float scale_log2 = kLog2e / sqrtf(static_cast<float>(S->head_dim));
  dec::decode_partial_kernel<<<dim3(n_split, S->n_heads), dec::K6_THREADS, 0, st>>>(
      *S, q, k, v, length, compressed, slot, scale_log2, parts, n_split);
  LS_LAUNCH_CHECK("decode_partial_kernel");
  dec::decode_combine_kernel<<<S->n_heads, 256, 0, st>>>(*S, length, compressed, slot, parts, n_split, out,
                                                         out_bf16);
  LS_LAUNCH_CHECK("decode_combine_kernel");
  return LS_OK;
}

extern "C" size_t ls_decode_select_workspace(const ls_decode_state *S, int32_t max_len) {
  (void)max_len;
  return static_cast<size_t>(S->n_heads) * S->row_cap * 9 + 1024;
}

extern "C" int ls_decode_select(const ls_decode_state *S, const int32_t *slot_order, int32_t n_rows,
                                int32_t length, int32_t budget, int32_t *retained_n, double *score_coverage,
                                void *ws, size_t ws_bytes, ls_stream_t stream) {
  int c = check_state(S);
  if (c) return c;
  LS_REQUIRE(n_rows >= 1, LS_ERR_EMPTY_WINDOW, "need at least one observation row");
  LS_REQUIRE(budget >= 1 && budget <= S->budget_cap, LS_ERR_INVALID_CONFIG, "budget outside [1, budget_cap]");
  LS_REQUIRE(length <= S->row_cap, LS_ERR_SEQUENCE_TOO_LONG, "length exceeds row_cap");
  LS_REQUIRE(ws_bytes >= ls_decode_select_workspace(S, length), LS_ERR_WORKSPACE, "decode_select workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Carver cv(ws, ws_bytes);
  double *acc = cv.take<double>(static_cast<size_t>(S->n_heads) * S->row_cap);
  uint8_t *touched = cv.take<uint8_t>(static_cast<size_t>(S->n_heads) * S->row_cap);
  dec::decode_select_kernel<<<S->n_heads, dec::K7_THREADS, 0, st>>>(*S, slot_order, n_rows, length, budget, acc,
                                                                   touched, retained_n, score_coverage);
  LS_LAUNCH_CHECK("decode_select_kernel");
  return LS_OK;
}

extern "C" int ls_kv_compact(const ls_decode_state *S, const uint16_t *k, const uint16_t *v, ls_stream_t stream) {
  int c = check_state(S);
  if (c) return c;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  dec::kv_compact_kernel<<<dim3(16, S->n_heads), 256, 0, st>>>(*S, k, v);
  LS_LAUNCH_CHECK("kv_compact_kernel");
  return LS_OK;
}
