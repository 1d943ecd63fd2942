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

// ---------------------------------------------------------------- K3a chain
struct Stage {
  int32_t idx[CHUNK];
  int32_t len[CHUNK];
  double w[CHUNK];
  double mx[CHUNK];
};

__global__ void __launch_bounds__(128) chain_kernel(Lists L, int n_total, double alpha, const double *total,
                                                    Picks P, int cap) {
  __shared__ Stage st[2];  // 0 slash, 1 vertical
  __shared__ int s_base[2], s_stop;
  __shared__ int s_idx_sh, v_idx_sh, n_pick_sh;
  __shared__ double ol_s_sh, ol_v_sh, approx_sh;
  const int h = blockIdx.x;
  const double T = total[h];
  const double target = alpha * T;
  const int64_t lb = static_cast<int64_t>(h) * 2 * n_total;
  const int64_t pb = static_cast<int64_t>(h) * cap;
  if (threadIdx.x == 0) {
    s_idx_sh = v_idx_sh = n_pick_sh = 0;
    ol_s_sh = ol_v_sh = approx_sh = 0.0;
    s_base[0] = s_base[1] = -1;
    s_stop = 0;
  }
  __syncthreads();
  while (true) {
    // (re)stage whichever list's cursor left its chunk
    for (int kind = 0; kind < 2; ++kind) {
      const int cur = kind == 0 ? s_idx_sh : v_idx_sh;
      const int want = (cur / CHUNK) * CHUNK;
      if (want != s_base[kind] && cur < n_total) {
        for (int i = threadIdx.x; i < CHUNK; i += blockDim.x) {
          int o = want + i;
          if (o < n_total) {
            int64_t g = lb + static_cast<int64_t>(kind) * n_total + o;
            st[kind].idx[i] = L.idx[g];
            st[kind].len[i] = L.len[g];
            st[kind].w[i] = L.w[g];
            st[kind].mx[i] = L.mx[g];
          }
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int kind = 0; kind < 2; ++kind) {
        const int cur = kind == 0 ? s_idx_sh : v_idx_sh;
        s_base[kind] = (cur / CHUNK) * CHUNK;
      }
      int s_idx = s_idx_sh, v_idx = v_idx_sh, n = n_pick_sh;
      double ol_s = ol_s_sh, ol_v = ol_v_sh, approx = approx_sh;
      const int s_end = s_base[0] + CHUNK, v_end = s_base[1] + CHUNK;
      int stop = 0;
      while (true) {
        if (!(approx < target - EPS)) {  // exact is checked by finalize
          stop = 1;
          break;
        }
        const bool has_s = s_idx < n_total, has_v = v_idx < n_total;
        if (!has_s && !has_v) {
          stop = 1;
          break;
        }
        if (n >= cap) {
          stop = 1;
          break;
        }
        if ((has_s && s_idx >= s_end) || (has_v && v_idx >= v_end)) break;  // restage
        bool take_slash;
        double ws = 0, wv = 0;
        int ls_ = 0, lv = 0;
        if (has_s) {
          ws = st[0].w[s_idx - s_base[0]];
          ls_ = st[0].len[s_idx - s_base[0]];
        }
        if (has_v) {
          wv = st[1].w[v_idx - s_base[1]];
          lv = st[1].len[v_idx - s_base[1]];
        }
        if (!has_s) {
          take_slash = false;
        } else if (!has_v) {
          take_slash = true;
        } else {
          // prefill.py:206-208, |V| = v_idx, |S| = s_idx
          const int den_s = max(1, ls_ - v_idx);
          const int den_v = max(1, lv - s_idx);
          const double gain_s = (ws - ol_v) / static_cast<double>(den_s);
          const double gain_v = (wv - ol_s) / static_cast<double>(den_v);
          take_slash = gain_s >= gain_v;
        }
        if (take_slash) {
          approx += ws - ol_v;
          ol_s += st[0].mx[s_idx - s_base[0]];
          P.code[pb + n] = st[0].idx[s_idx - s_base[0]];
          P.other[pb + n] = v_idx;
          P.w[pb + n] = ws;
          ++s_idx;
        } else {
          approx += wv - ol_s;
          ol_v += st[1].mx[v_idx - s_base[1]];
          P.code[pb + n] = st[1].idx[v_idx - s_base[1]] | static_cast<int32_t>(0x80000000u);
          P.other[pb + n] = s_idx;
          P.w[pb + n] = wv;
          ++v_idx;
        }
        P.approx[pb + n] = approx;
        ++n;
      }
      s_idx_sh = s_idx;
      v_idx_sh = v_idx;
      n_pick_sh = n;
      ol_s_sh = ol_s;
      ol_v_sh = ol_v;
      approx_sh = approx;
      s_stop = stop;
    }
    __syncthreads();
    if (s_stop) break;
  }
  if (threadIdx.x == 0) P.n[h] = n_pick_sh;
}

// ------------------------------------------------------------ K3b crossings
// Cell source 1: recompute P[r, c] from q, k and K1 row statistics.
struct RecomputeCells {
  const uint16_t *q, *k;
  const int32_t *rows;
  const int32_t *row_of;  // [H][n_total] sampled row index of position g, or -1
  const float *row_stats;
  int n_s, n_total, row_offset, d, group;
  int64_t q_head_stride, kv_head_stride;
  float scale_log2;

  __device__ __forceinline__ double cell(int h, int g, int c) const {
    if (g >= n_total) return 0.0;
    const int r = row_of[static_cast<int64_t>(h) * n_total + g];
    if (r < 0) return 0.0;
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
  __device__ __forceinline__ double cell(int /*h*/, int g, int c) const {
    if (g >= n_total) return 0.0;
    const int r = row_of[g];
    if (r < 0) return 0.0;
    return weights[static_cast<int64_t>(r) * n_total + c];
  }
};

template <typename Cells>
__global__ void __launch_bounds__(256) cross_kernel(Lists L, int n_total, Picks P, int cap, Cells cells) {
  __shared__ double vals[8][32];
  const int h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = P.n[h];
  const int64_t pb = static_cast<int64_t>(h) * cap;
  const int64_t lb = static_cast<int64_t>(h) * 2 * n_total;
  for (int t = blockIdx.x * 8 + warp; t < n; t += gridDim.x * 8) {
    const int32_t code = P.code[pb + t];
    const bool is_vert = code < 0;
    const int idx = code & 0x7fffffff;
    const int n_other = P.other[pb + t];
    const int32_t *other = L.idx + lb + static_cast<int64_t>(is_vert ? 0 : 1) * n_total;  // picked-in-order prefix
    double sum = 0.0;  // python sum() starts at 0, adds in selection order
    for (int j0 = 0; j0 < n_other; j0 += 32) {
      const int j = j0 + lane;
      double v = 0.0;
      if (j < n_other) {
        const int o = other[j];
        // slash pick d=idx crosses vertical c=o at g=c+d; vertical pick c=idx crosses slash d=o
        v = is_vert ? cells.cell(h, idx + o, idx) : cells.cell(h, o + idx, o);
      }
      vals[warp][lane] = v;
      __syncwarp();
      if (lane == 0) {
        const int m = min(32, n_other - j0);
        for (int i = 0; i < m; ++i) sum += vals[warp][i];
      }
      __syncwarp();
    }
    if (lane == 0) P.cross[pb + t] = sum;
  }
}

// ------------------------------------------------------------ K3c finalize
__global__ void finalize_kernel(Picks P, int cap, double alpha, const double *total, int32_t *n_final,
                                double *coverage, double *approx_out) {
  const int h = blockIdx.x, lane = threadIdx.x;
  const double T = total[h];
  const double target = alpha * T;
  const int n = P.n[h];
  const int64_t pb = static_cast<int64_t>(h) * cap;
  double exact = 0.0, approx = 0.0;
  int t_stop = -1;
  if (!(0.0 < target - EPS)) t_stop = 0;  // loop never entered (e.g. alpha = 0)
  for (int t0 = 0; t0 < n && t_stop < 0; t0 += 32) {
    const int t = t0 + lane;
    double inc = 0.0, ap = 0.0;
    if (t < n) {
      inc = P.w[pb + t] - P.cross[pb + t];
      ap = P.approx[pb + t];
    }
    const int m = min(32, n - t0);
    for (int i = 0; i < m; ++i) {
      const double in = __shfl_sync(0xffffffffu, inc, i);
      const double a = __shfl_sync(0xffffffffu, ap, i);
      exact += in;  // prefill.py:211 / 217
      approx = a;
      if (!(approx < target - EPS && exact < target - EPS)) {
        t_stop = t0 + i + 1;
        break;
      }
    }
  }
  if (t_stop < 0) t_stop = n;  // lists exhausted
  if (lane == 0) {
    n_final[h] = t_stop;
    const double cov = T > 0 ? exact / T : 0.0;  // prefill.py:221
    coverage[h] = cov < 1.0 ? cov : 1.0;
    approx_out[h] = approx;
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
  finalize_kernel<<<H, 32, 0, st>>>(w.picks, w.cap, alpha, total, w.n_final, coverage, approx);
  LS_LAUNCH_CHECK("finalize_kernel");
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
  sel::chain_kernel<<<H, 128, 0, st>>>(w.lists, n_total, alpha, total, w.picks, w.cap);
  LS_LAUNCH_CHECK("chain_kernel");
  sel::row_of_kernel<<<dim3(ceil_div(n_total, 256), H), 256, 0, st>>>(rows, n_s, n_total, L->row_offset, w.row_of);
  sel::row_of_set_kernel<<<dim3(ceil_div(n_s, 256), H), 256, 0, st>>>(rows, n_s, n_total, L->row_offset, w.row_of);
  LS_LAUNCH_CHECK("row_of_kernel");
  sel::RecomputeCells cells;
  cells.q = q;
  cells.k = k;
  cells.rows = rows;
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
  sel::cross_kernel<sel::RecomputeCells><<<dim3(32, H), 256, 0, st>>>(w.lists, n_total, w.picks, w.cap, cells);
  LS_LAUNCH_CHECK("cross_kernel");
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
  sel::chain_kernel<<<1, 128, 0, st>>>(w.lists, n_total, alpha, tot, w.picks, w.cap);
  LS_LAUNCH_CHECK("chain_kernel");
  sel::row_of_kernel<<<dim3(ceil_div(n_total, 256), 1), 256, 0, st>>>(positions, n_rows, n_total, 0, w.row_of);
  sel::row_of_set_kernel<<<dim3(ceil_div(n_rows, 256), 1), 256, 0, st>>>(positions, n_rows, n_total, 0, w.row_of);
  sel::DenseCells cells{weights, w.row_of, n_total};
  sel::cross_kernel<sel::DenseCells><<<dim3(32, 1), 256, 0, st>>>(w.lists, n_total, w.picks, w.cap, cells);
  LS_LAUNCH_CHECK("cross_kernel");
  return sel::run_tail(w, 1, n_total, alpha, tot, slash_ids, vert_ids, counts, coverage, approx, nullptr, nullptr,
                       st);
}
