// K2 + K3 + K4 -- line sort, greedy coverage-alpha selection, plan build.
//
// Replaces the sort in _line_sums (reference prefill.py:168-169) and
// _greedy (prefill.py:178-229).
//
// K2 sort: one CTA per (head, kind) sorts the n_total lines by
//   (weight desc, index asc)  -- a stable LSD radix sort of ~bits(w_fp64)
// (cub::BlockRadixSort, in-shared-memory, up to 16384 lines).
//
// K3 greedy, split so the sequential part is tiny:
//   (a) chain: the pick decisions of _greedy depend only on
//       (approx, ol_s, ol_v, |S|, |V|) -- never on the exact accumulator,
//       which only decides termination (prefill.py:195). One thread per head
//       replays the decision chain in fp64 with the reference's update order
//       (prefill.py:206-220) over shared-memory-staged line chunks, until
//       approx >= target - eps or both lists are exhausted, recording every
//       pick, its approx value and how many lines of the other kind preceded
//       it. Since approx <= exact at every step, the true stopping point is
//       inside this sequence.
//   (b) crossings: one warp per pick sums, in selection order, the crossing
//       cells with the previously picked lines of the other kind
//       (prefill.py:211, 217; _BlockView.cell prefill.py:116-122) -- a cell
//       exists only when c + d is a sampled position; its value is
//       recomputed from q, k and the row statistics of K1.
//   (c) finalize: sequential fp64 exact(t) += w_t - cross_t; the plan is the
//       shortest pick prefix with approx or exact >= target - eps
//       (prefill.py:195), coverage = min(exact / T, 1) (prefill.py:221-222).
// K4: picks -> sorted slash / vertical id lists via bitmaps.

#include <cub/block/block_radix_sort.cuh>

#include "ls_common.cuh"

namespace ls {
namespace sel {

constexpr int SORT_THREADS = 512;
constexpr int SORT_ITEMS = 32;  // capacity 16384
constexpr int SORT_CAP = SORT_THREADS * SORT_ITEMS;
constexpr int CHUNK = 512;      // staged lines per list in the chain kernel
constexpr double EPS = 1e-12;   // prefill.py:188

struct Lists {  // sorted lines, [H][2][n] (kind 0 = slash, 1 = vertical)
  int32_t *idx;
  double *w;
  int32_t *len;
  double *mx;
};

struct Picks {  // [H][cap]
  int32_t *code;    // kind << 31 | line index
  int32_t *other;   // picks of the other kind before this one
  double *w;        // line weight
  double *approx;   // approx after this pick
  double *cross;    // crossing-cell sum (phase b)
  int32_t *n;       // [H] picks recorded by the chain
};

// ---------------------------------------------------------------- K2 sort
using BlockSort = cub::BlockRadixSort<unsigned long long, SORT_THREADS, SORT_ITEMS, int32_t>;

template <typename MaxT>
__global__ void __launch_bounds__(SORT_THREADS) sort_lines_kernel(const double *v_w, const MaxT *v_max,
                                                                  const double *s_w, const MaxT *s_max,
                                                                  const int32_t *rows, int n_s, int n_total,
                                                                  int row_offset, Lists out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto &temp = *reinterpret_cast<typename BlockSort::TempStorage *>(smem_raw);
  int *pos = reinterpret_cast<int *>(smem_raw + sizeof(typename BlockSort::TempStorage));
  const int h = blockIdx.y, kind = blockIdx.x;  // 0 slash, 1 vertical
  const double *w = (kind == 0 ? s_w : v_w) + static_cast<int64_t>(h) * n_total;
  const MaxT *mx = (kind == 0 ? s_max : v_max) + static_cast<int64_t>(h) * n_total;
  for (int r = threadIdx.x; r < n_s; r += blockDim.x) pos[r] = row_offset + rows[static_cast<int64_t>(h) * n_s + r];
  unsigned long long keys[SORT_ITEMS];
  int32_t vals[SORT_ITEMS];
#pragma unroll
  for (int i = 0; i < SORT_ITEMS; ++i) {
    int idx = threadIdx.x * SORT_ITEMS + i;  // blocked arrangement = index order
    if (idx < n_total) {
      keys[i] = ~static_cast<unsigned long long>(__double_as_longlong(w[idx]));
    } else {
      keys[i] = ~0ull;
    }
    vals[i] = idx;
  }
  __syncthreads();
  BlockSort(temp).Sort(keys, vals);  // ascending ~bits == descending weight, stable
  __syncthreads();
  const int64_t base = (static_cast<int64_t>(h) * 2 + kind) * n_total;
#pragma unroll
  for (int i = 0; i < SORT_ITEMS; ++i) {
    int o = threadIdx.x * SORT_ITEMS + i;
    if (o < n_total) {
      int idx = vals[i];
      out.idx[base + o] = idx;
      out.w[base + o] = w[idx];
      out.mx[base + o] = static_cast<double>(mx[idx]);
      out.len[base + o] = n_s - lower_bound_dev(pos, n_s, idx);  // #{rows with g >= idx}, prefill.py:144,155
    }
  }
}

// ------------------------------------------------------- crossing cells
// Cell source 1: recompute P[r, c] from q, k and K1 row statistics.
struct RecomputeCells {
  const uint16_t *q, *k;
  const int32_t *row_of;  // [H][n_total] sampled row index of position g, or -1
  const float *row_stats;
  int n_s, n_total, row_offset, d, group;
  int64_t q_head_stride, kv_head_stride;
  float scale_log2;

  __device__ __forceinline__ int row(int h, int g) const {
    return g < n_total ? row_of[static_cast<int64_t>(h) * n_total + g] : -1;
  }
  __device__ __forceinline__ double value(int h, int r, int g, int c) const {
    const uint16_t *qr = q + static_cast<int64_t>(h) * q_head_stride + static_cast<int64_t>(g - row_offset) * d;
    const uint16_t *kr = k + static_cast<int64_t>(h / group) * kv_head_stride + static_cast<int64_t>(c) * d;
    float acc = 0.f;
    for (int v = 0; v < d / 8; ++v) {
      uint4 a = *reinterpret_cast<const uint4 *>(qr + v * 8);
      uint4 b = *reinterpret_cast<const uint4 *>(kr + v * 8);
      float fa[8], fb[8];
      bf16x8_to_f32(a, fa);
      bf16x8_to_f32(b, fb);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc = fmaf(fa[j], fb[j], acc);
    }
    const float *rs = row_stats + (static_cast<int64_t>(h) * n_s + r) * 2;
    return static_cast<double>(fast_exp2(acc * scale_log2 - rs[0]) * rs[1]);
  }
};

// Cell source 2: a dense fp64 weight matrix (greedy_select_lines parity path).
struct DenseCells {
  const double *weights;  // [n_rows][n_total]
  const int32_t *row_of;  // [n_total]
  int n_total;
  __device__ __forceinline__ int row(int /*h*/, int g) const { return g < n_total ? row_of[g] : -1; }
  __device__ __forceinline__ double value(int /*h*/, int r, int /*g*/, int c) const {
    return weights[static_cast<int64_t>(r) * n_total + c];
  }
};

// ------------------------------------------------------------ K3 greedy
// One CTA per head. Rounds of: (A) thread 0 advances the decision chain by up
// to PCH picks (prefill.py:195-220, approx-only decisions), (B) every warp
// sums the crossing cells of some of the new picks with the other kind's
// already-picked prefix, in selection order (prefill.py:211, 217), (C) thread
// 0 replays exact += w - cross in order and applies the reference's dual
// termination test (prefill.py:195). Stops at the first pick count where
// approx or exact reaches alpha*T - eps, or when both lists are exhausted.
struct Stage {
  int32_t idx[CHUNK];
  int32_t len[CHUNK];
  double w[CHUNK];
  double mx[CHUNK];
};

constexpr int PCH = 64;             // picks per round
constexpr int G_THREADS = 512;      // 16 warps
constexpr int G_WARPS = G_THREADS / 32;

// gain_s >= gain_v with gain = num / den (prefill.py:206-208). Decided by
// cross-multiplication unless the two sides are within 1e-13 relative, in
// which case the reference's own fp64 divisions decide (bit-identical result).
__device__ __forceinline__ bool take_slash_decision(double a, int ds, double b, int dv) {
  const double x = a * static_cast<double>(dv);
  const double y = b * static_cast<double>(ds);
  const double diff = x - y;
  const double mag = fmax(fabs(x), fabs(y));
  if (fabs(diff) > 1e-13 * mag) return diff > 0.0;
  return a / static_cast<double>(ds) >= b / static_cast<double>(dv);
}

template <typename Cells>
__global__ void __launch_bounds__(G_THREADS) greedy_kernel(Lists L, int n_total, double alpha, const double *total,
                                                            Picks P, int cap, Cells cells, int32_t *n_final,
                                                            double *coverage, double *approx_out) {
  __shared__ Stage st[2];  // 0 slash, 1 vertical
  __shared__ int c_code[PCH], c_other[PCH];
  __shared__ double c_w[PCH], c_approx[PCH], c_cross[PCH];
  __shared__ double vals[G_WARPS][32];
  __shared__ int s_base[2], s_idx_sh, v_idx_sh, n_sh, n_chunk, done, exhausted;
  __shared__ double ol_s_sh, ol_v_sh, approx_sh, exact_sh;
  const int h = blockIdx.x;
  const double T = total[h];
  const double target = alpha * T;
  const int64_t lb = static_cast<int64_t>(h) * 2 * n_total;
  const int64_t pb = static_cast<int64_t>(h) * cap;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    s_idx_sh = v_idx_sh = n_sh = 0;
    ol_s_sh = ol_v_sh = approx_sh = exact_sh = 0.0;
    s_base[0] = s_base[1] = -1;
    done = !(0.0 < target - EPS);  // the while condition fails before any pick
    exhausted = 0;
  }
  __syncthreads();
  while (!done) {
    // (re)stage whichever list's cursor left its chunk
    for (int kind = 0; kind < 2; ++kind) {
      const int cur = kind == 0 ? s_idx_sh : v_idx_sh;
      const int want = (cur / CHUNK) * CHUNK;
      if (want != s_base[kind] && cur < n_total) {
        for (int i = threadIdx.x; i < CHUNK; i += blockDim.x) {
          const int o = want + i;
          if (o < n_total) {
            const int64_t g = lb + static_cast<int64_t>(kind) * n_total + o;
            st[kind].idx[i] = L.idx[g];
            st[kind].len[i] = L.len[g];
            st[kind].w[i] = L.w[g];
            st[kind].mx[i] = L.mx[g];
          }
        }
      }
    }
    __syncthreads();
    // (A) decision chain
    if (threadIdx.x == 0) {
      for (int kind = 0; kind < 2; ++kind) s_base[kind] = ((kind == 0 ? s_idx_sh : v_idx_sh) / CHUNK) * CHUNK;
      int s_idx = s_idx_sh, v_idx = v_idx_sh, k = 0;
      double ol_s = ol_s_sh, ol_v = ol_v_sh, approx = approx_sh;
      const int s_end = s_base[0] + CHUNK, v_end = s_base[1] + CHUNK;
      while (k < PCH) {
        const bool has_s = s_idx < n_total, has_v = v_idx < n_total;
        if (!has_s && !has_v) break;
        if ((has_s && s_idx >= s_end) || (has_v && v_idx >= v_end)) break;  // restage first
        bool take_slash;
        const int so = s_idx - s_base[0], vo = v_idx - s_base[1];
        if (!has_s) {
          take_slash = false;
        } else if (!has_v) {
          take_slash = true;
        } else {
          // |V| = v_idx, |S| = s_idx (prefill.py:206-207)
          take_slash = take_slash_decision(st[0].w[so] - ol_v, max(1, st[0].len[so] - v_idx),
                                           st[1].w[vo] - ol_s, max(1, st[1].len[vo] - s_idx));
        }
        if (take_slash) {
          approx += st[0].w[so] - ol_v;
          ol_s += st[0].mx[so];
          c_code[k] = st[0].idx[so];
          c_other[k] = v_idx;
          c_w[k] = st[0].w[so];
          ++s_idx;
        } else {
          approx += st[1].w[vo] - ol_s;
          ol_v += st[1].mx[vo];
          c_code[k] = st[1].idx[vo] | static_cast<int32_t>(0x80000000u);
          c_other[k] = s_idx;
          c_w[k] = st[1].w[vo];
          ++v_idx;
        }
        c_approx[k] = approx;
        ++k;
        // the reference re-tests the loop condition after every pick; stop the
        // chain at the approx target (exact is applied in phase C)
        if (!(approx < target - EPS)) break;
      }
      s_idx_sh = s_idx;
      v_idx_sh = v_idx;
      ol_s_sh = ol_s;
      ol_v_sh = ol_v;
      approx_sh = approx;
      n_chunk = k;
      exhausted = (s_idx >= n_total && v_idx >= n_total) ? 1 : 0;
    }
    __syncthreads();
    const int nk = n_chunk;
    // (B) crossing sums, one warp per new pick, selection order
    for (int j = warp; j < nk; j += G_WARPS) {
      const int32_t code = c_code[j];
      const bool is_vert = code < 0;
      const int idx = code & 0x7fffffff;
      const int n_other = c_other[j];
      const int32_t *other = L.idx + lb + static_cast<int64_t>(is_vert ? 0 : 1) * n_total;
      double sum = 0.0;
      for (int j0 = 0; j0 < n_other; j0 += 32) {
        const int jj = j0 + lane;
        double v = 0.0;
        if (jj < n_other) {
          const int o = other[jj];
          // slash d=idx x vertical c=o at g=o+idx; vertical c=idx x slash d=o at g=idx+o
          const int g = idx + o;
          const int c = is_vert ? idx : o;
          const int r = cells.row(h, g);
          if (r >= 0) v = cells.value(h, r, g, c);
        }
        const unsigned any = __ballot_sync(0xffffffffu, v != 0.0);
        if (any) {
          vals[warp][lane] = v;
          __syncwarp();
          if (lane == 0) {
            const int m = min(32, n_other - j0);
            for (int i = 0; i < m; ++i) sum += vals[warp][i];  // python sum(): left to right
          }
          __syncwarp();
        }
      }
      if (lane == 0) c_cross[j] = sum;
    }
    __syncthreads();
    // (C) exact accumulator + dual termination, in order
    if (threadIdx.x == 0) {
      double exact = exact_sh;
      int n = n_sh;
      int stop = 0;
      for (int j = 0; j < nk; ++j) {
        exact += c_w[j] - c_cross[j];
        P.code[pb + n] = c_code[j];
        P.approx[pb + n] = c_approx[j];
        ++n;
        if (!(c_approx[j] < target - EPS && exact < target - EPS)) {
          stop = 1;
          approx_sh = c_approx[j];
          break;
        }
      }
      if (!stop && nk > 0) approx_sh = c_approx[nk - 1];
      exact_sh = exact;
      n_sh = n;
      if (stop || exhausted || n >= cap) done = 1;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    P.n[h] = n_sh;
    n_final[h] = n_sh;
    const double cov = T > 0 ? exact_sh / T : 0.0;  // prefill.py:221
    coverage[h] = cov < 1.0 ? cov : 1.0;
    approx_out[h] = n_sh > 0 ? approx_sh : 0.0;
  }
}

// ------------------------------------------------------------------ K4 plan
__global__ void plan_bits_kernel(Picks P, int cap, const int32_t *n_final, int n_total, int words,
                                 uint32_t *sbits, uint32_t *vbits, int32_t *picks_out) {
  const int h = blockIdx.y;
  const int n = n_final[h];
  const int64_t pb = static_cast<int64_t>(h) * cap;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int32_t code = P.code[pb + t];
    const int idx = code & 0x7fffffff;
    uint32_t *bits = (code < 0 ? vbits : sbits) + static_cast<int64_t>(h) * words;
    atomicOr(bits + (idx >> 5), 1u << (idx & 31));
    if (picks_out) picks_out[static_cast<int64_t>(h) * 2 * n_total + t] = code;
  }
}

// bitmap -> sorted ids (one CTA per (head, kind))
__global__ void __launch_bounds__(1024) compact_bits_kernel(const uint32_t *sbits, const uint32_t *vbits, int words,
                                                            int n_total, int32_t *slash_ids, int32_t *vert_ids,
                                                            int32_t *counts) {
  __shared__ int warp_tot[32];
  __shared__ int carry;
  const int h = blockIdx.y, kind = blockIdx.x;
  const uint32_t *bits = (kind == 0 ? sbits : vbits) + static_cast<int64_t>(h) * words;
  int32_t *out = (kind == 0 ? slash_ids : vert_ids) + static_cast<int64_t>(h) * n_total;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int w0 = 0; w0 < words; w0 += blockDim.x) {
    const int w = w0 + threadIdx.x;
    const uint32_t x = w < words ? bits[w] : 0u;
    const int c = __popc(x);
    // block exclusive scan of c
    int incl = c;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      int v = lane < (blockDim.x >> 5) ? warp_tot[lane] : 0;
      int vi = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, vi, o);
        if (lane >= o) vi += y;
      }
      if (lane < (blockDim.x >> 5)) warp_tot[lane] = vi - v;  // exclusive
    }
    __syncthreads();
    int pos = carry + warp_tot[wid] + incl - c;
    uint32_t y = x;
    while (y) {
      int b = __ffs(y) - 1;
      y &= y - 1;
      out[pos++] = w * 32 + b;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = pos;
    __syncthreads();
  }
  if (threadIdx.x == 0) counts[h * 2 + kind] = carry;
}

__global__ void row_of_kernel(const int32_t *rows, int n_s, int n_total, int row_offset, int32_t *row_of) {
  const int h = blockIdx.y;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_total; i += gridDim.x * blockDim.x)
    row_of[static_cast<int64_t>(h) * n_total + i] = -1;
  // (second launch sets the sampled positions)
}

__global__ void row_of_set_kernel(const int32_t *rows, int n_s, int n_total, int row_offset, int32_t *row_of) {
  const int h = blockIdx.y;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_s; r += gridDim.x * blockDim.x)
    row_of[static_cast<int64_t>(h) * n_total + row_offset + rows[static_cast<int64_t>(h) * n_s + r]] = r;
}

struct Work {
  Lists lists;
  Picks picks;
  int32_t *row_of;
  uint32_t *sbits, *vbits;
  int32_t *n_final;
  int words, cap;
};

inline Work carve(Carver &c, int H, int n_total, bool with_row_of) {
  Work w;
  const size_t nl = static_cast<size_t>(H) * 2 * n_total;
  w.cap = 2 * n_total;
  const size_t np = static_cast<size_t>(H) * w.cap;
  w.lists.idx = c.take<int32_t>(nl);
  w.lists.len = c.take<int32_t>(nl);
  w.lists.w = c.take<double>(nl);
  w.lists.mx = c.take<double>(nl);
  w.picks.code = c.take<int32_t>(np);
  w.picks.other = c.take<int32_t>(np);
  w.picks.w = c.take<double>(np);
  w.picks.approx = c.take<double>(np);
  w.picks.cross = c.take<double>(np);
  w.picks.n = c.take<int32_t>(H);
  w.n_final = c.take<int32_t>(H);
  w.words = (n_total + 31) / 32;
  w.sbits = c.take<uint32_t>(static_cast<size_t>(H) * w.words);
  w.vbits = c.take<uint32_t>(static_cast<size_t>(H) * w.words);
  w.row_of = with_row_of ? c.take<int32_t>(static_cast<size_t>(H) * n_total) : nullptr;
  return w;
}

inline size_t sort_smem() { return sizeof(typename BlockSort::TempStorage) + 4 * 16384 + 64; }

int run_tail(Work &w, int H, int n_total, double alpha, const double *total, int32_t *slash_ids,
             int32_t *vert_ids, int32_t *counts, double *coverage, double *approx, int32_t *picks_out,
             int32_t *n_picks_out, cudaStream_t st) {
  LS_CUDA(cudaMemsetAsync(w.sbits, 0, sizeof(uint32_t) * H * w.words, st));
  LS_CUDA(cudaMemsetAsync(w.vbits, 0, sizeof(uint32_t) * H * w.words, st));
  plan_bits_kernel<<<dim3(8, H), 256, 0, st>>>(w.picks, w.cap, w.n_final, n_total, w.words, w.sbits, w.vbits,
                                               picks_out);
  LS_LAUNCH_CHECK("plan_bits_kernel");
  compact_bits_kernel<<<dim3(2, H), 1024, 0, st>>>(w.sbits, w.vbits, w.words, n_total, slash_ids, vert_ids,
                                                    counts);
  LS_LAUNCH_CHECK("compact_bits_kernel");
  if (n_picks_out) LS_CUDA(cudaMemcpyAsync(n_picks_out, w.n_final, sizeof(int32_t) * H, cudaMemcpyDeviceToDevice, st));
  return LS_OK;
}

}  // namespace sel
}  // namespace ls

using namespace ls;

extern "C" size_t ls_select_lines_workspace(const ls_layer_desc *L, int32_t /*n_s*/) {
  Carver c(nullptr, 0);
  sel::carve(c, L->n_heads, L->n_total, true);
  return c.off + 4096;
}

extern "C" int ls_select_lines(const ls_layer_desc *L, int32_t n_s, double alpha, const uint16_t *q,
                               const uint16_t *k, const int32_t *rows, const double *v_w, const float *v_max,
                               const double *s_w, const float *s_max, const float *row_stats, const double *total,
                               int32_t *slash_ids, int32_t *vert_ids, int32_t *counts, double *coverage,
                               double *approx, int32_t *picks, int32_t *n_picks, void *ws, size_t ws_bytes,
                               ls_stream_t stream) {
  LS_REQUIRE(alpha >= 0.0 && alpha <= 1.0, LS_ERR_INVALID_ALPHA, "alpha=%g outside [0, 1]", alpha);
  LS_REQUIRE(L->n_total <= sel::SORT_CAP, LS_ERR_UNSUPPORTED, "n_total=%d exceeds the in-SM sort capacity %d",
             L->n_total, sel::SORT_CAP);
  LS_REQUIRE(ws_bytes >= ls_select_lines_workspace(L, n_s), LS_ERR_WORKSPACE, "select_lines workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int H = L->n_heads, n_total = L->n_total;
  Carver c(ws, ws_bytes);
  sel::Work w = sel::carve(c, H, n_total, true);
  const size_t smem = sel::sort_smem();
  LS_CUDA(cudaFuncSetAttribute(sel::sort_lines_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  sel::sort_lines_kernel<float><<<dim3(2, H), sel::SORT_THREADS, smem, st>>>(v_w, v_max, s_w, s_max, rows, n_s,
                                                                            n_total, L->row_offset, w.lists);
  LS_LAUNCH_CHECK("sort_lines_kernel");
  sel::row_of_kernel<<<dim3(ceil_div(n_total, 256), H), 256, 0, st>>>(rows, n_s, n_total, L->row_offset, w.row_of);
  sel::row_of_set_kernel<<<dim3(ceil_div(n_s, 256), H), 256, 0, st>>>(rows, n_s, n_total, L->row_offset, w.row_of);
  LS_LAUNCH_CHECK("row_of_kernel");
  sel::RecomputeCells cells;
  cells.q = q;
  cells.k = k;
  cells.row_of = w.row_of;
  cells.row_stats = row_stats;
  cells.n_s = n_s;
  cells.n_total = n_total;
  cells.row_offset = L->row_offset;
  cells.d = L->head_dim;
  cells.group = L->n_heads / L->n_kv_heads;
  cells.q_head_stride = L->q_head_stride;
  cells.kv_head_stride = L->kv_head_stride;
  cells.scale_log2 = kLog2e / sqrtf(static_cast<float>(L->head_dim));
  sel::greedy_kernel<sel::RecomputeCells><<<H, sel::G_THREADS, 0, st>>>(w.lists, n_total, alpha, total, w.picks,
                                                                        w.cap, cells, w.n_final, coverage, approx);
  LS_LAUNCH_CHECK("greedy_kernel");
  return sel::run_tail(w, H, n_total, alpha, total, slash_ids, vert_ids, counts, coverage, approx, picks, n_picks,
                       st);
}

// Dense-weights greedy for caller-provided sorted lists (one head).
namespace ls {
namespace sel {
__global__ void load_lists_kernel(int n, const int32_t *idx, const double *w, const int32_t *len,
                                  const double *mx, int kind, int n_total, Lists L) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_total; i += gridDim.x * blockDim.x) {
    const int64_t o = static_cast<int64_t>(kind) * n_total + i;
    if (i < n) {
      L.idx[o] = idx[i];
      L.w[o] = w[i];
      L.len[o] = len[i];
      L.mx[o] = mx[i];
    }
  }
}
}  // namespace sel
}  // namespace ls

extern "C" int ls_greedy_dense(int32_t n_slash, const int32_t *s_idx, const double *s_w, const int32_t *s_len,
                               const double *s_max, int32_t n_vert, const int32_t *v_idx, const double *v_w,
                               const int32_t *v_len, const double *v_max, double alpha, double total_weight,
                               const double *weights, const int32_t *positions, int32_t n_rows, int32_t n_total,
                               int32_t *slash_ids, int32_t *vert_ids, int32_t *counts, double *coverage,
                               double *approx, void *ws, size_t ws_bytes, ls_stream_t stream) {
  LS_REQUIRE(alpha >= 0.0 && alpha <= 1.0, LS_ERR_INVALID_ALPHA, "alpha=%g outside [0, 1]", alpha);
  LS_REQUIRE(n_slash == n_total && n_vert == n_total, LS_ERR_SIZE_MISMATCH,
             "ls_greedy_dense expects exactly n_total lines of each kind");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Carver c(ws, ws_bytes);
  sel::Work w = sel::carve(c, 1, n_total, true);
  double *tot = c.take<double>(1);
  LS_REQUIRE(c.ok(), LS_ERR_WORKSPACE, "greedy_dense workspace too small (%zu > %zu)", c.off, ws_bytes);
  LS_CUDA(cudaMemcpyAsync(tot, &total_weight, sizeof(double), cudaMemcpyHostToDevice, st));
  sel::load_lists_kernel<<<8, 256, 0, st>>>(n_slash, s_idx, s_w, s_len, s_max, 0, n_total, w.lists);
  sel::load_lists_kernel<<<8, 256, 0, st>>>(n_vert, v_idx, v_w, v_len, v_max, 1, n_total, w.lists);
  LS_LAUNCH_CHECK("load_lists_kernel");
  sel::row_of_kernel<<<dim3(ceil_div(n_total, 256), 1), 256, 0, st>>>(positions, n_rows, n_total, 0, w.row_of);
  sel::row_of_set_kernel<<<dim3(ceil_div(n_rows, 256), 1), 256, 0, st>>>(positions, n_rows, n_total, 0, w.row_of);
  sel::DenseCells cells{weights, w.row_of, n_total};
  sel::greedy_kernel<sel::DenseCells><<<1, sel::G_THREADS, 0, st>>>(w.lists, n_total, alpha, tot, w.picks, w.cap,
                                                                    cells, w.n_final, coverage, approx);
  LS_LAUNCH_CHECK("greedy_kernel");
  return sel::run_tail(w, 1, n_total, alpha, tot, slash_ids, vert_ids, counts, coverage, approx, nullptr, nullptr,
                       st);
}
