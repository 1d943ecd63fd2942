// K2 + K3 + K4 -- line sort, greedy coverage-alpha selection, plan build.
//
// Replaces the sort in _line_sums (reference prefill.py:168-169) and
// _greedy (prefill.py:178-229).
//
// K2 sort: every (head, kind) list of a layer sorted at once by
//   (weight desc, index asc) -- one device-wide stable LSD radix sort over
// composite (segment, fixed-point weight) keys (sort_keys_kernel ->
// cub::DeviceRadixSort -> sort_scatter_kernel).
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

#include <algorithm>

#include <cuda.h>

#include <cub/block/block_radix_sort.cuh>
#include <cub/device/device_radix_sort.cuh>

#include "ls_common.cuh"

namespace ls {
extern int *g_debug_buffer;
namespace sel {

constexpr double EPS = 1e-12;   // prefill.py:188

struct Lists {  // sorted lines, [H][2][n] (kind 0 = slash, 1 = vertical)
  int32_t *sorted;    // [H][2] length of the sorted prefix (nullptr: every list fully sorted)
  int32_t *overflow;  // [H] set by K3 when it needs a line past a sorted prefix
  int32_t *idx;
  int32_t *inv;     // line index -> position in its sorted list
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

// K4 fused into K3 (per head, by the head's CTA) with a readiness flag, so the
// sparse attention of a head can start while slower heads are still selecting
struct PlanOut {
  uint32_t *sbits, *vbits;  // [H][words] scratch bitmaps
  int words;
  int32_t *slash_ids, *vert_ids, *counts;  // [H][n_total], [H][n_total], [H][2]
  int32_t *picks_out;                      // optional [H][2 n_total]
  int32_t *ready;                          // [H] set to `epoch` once the head's plan is written
  int32_t epoch;
};

// ---------------------------------------------------------------- K2 sort
// K2 (device-wide): every (head, kind) list of a layer sorted at once by one
// stable LSD radix sort over composite keys
//   (segment << fix_bits) | (2^fix_bits - 1 - fixed point weight)
// K1's line weights are exact multiples of 2^-40 and at most n_s (every row
// sums to 1), so a fix_bits = 40 + bits(n_s) integer orders them exactly;
// ties keep index order (stable). The whole GPU sorts, and n_total is not
// bounded by one SM's shared memory.
inline int fix_bits_for(int n_s) {
  int b = 0;
  while ((1ll << b) <= static_cast<long long>(n_s)) ++b;
  return 40 + b;
}

__global__ void sort_keys_kernel(const double *v_w, const double *s_w, int H, int n_total, int FIX_BITS,
                                 unsigned long long *keys, int32_t *vals) {
  const int64_t n = static_cast<int64_t>(2) * H * n_total;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t seg = i / n_total;  // h * 2 + kind
    const int idx = static_cast<int>(i - seg * n_total);
    const int h = static_cast<int>(seg >> 1), kind = static_cast<int>(seg & 1);
    const double w = (kind == 0 ? s_w : v_w)[static_cast<int64_t>(h) * n_total + idx];
    const unsigned long long fix = static_cast<unsigned long long>(w * 1099511627776.0);
    keys[i] = (static_cast<unsigned long long>(seg) << FIX_BITS) | (((1ull << FIX_BITS) - 1ull) - fix);
    vals[i] = idx;
  }
}

constexpr int kScatterShRows = 12 * 1024;  // 48 KB of positions: the default dynamic shared memory

template <typename MaxT>
__global__ void sort_scatter_kernel(const unsigned long long *keys_sorted, const int32_t *vals_sorted,
                                    const double *v_w, const MaxT *v_max, const double *s_w, const MaxT *s_max,
                                    const int32_t *rows, int n_s, int n_total, int row_offset, int H, Lists out) {
  extern __shared__ int pos_sh[];  // sampled local rows of this head (when they fit in shared memory)
  const int h = blockIdx.y;
  const int32_t *rows_h = rows + static_cast<int64_t>(h) * n_s;
  const bool in_sh = n_s <= kScatterShRows;
  if (in_sh) {
    for (int r = threadIdx.x; r < n_s; r += blockDim.x) pos_sh[r] = rows_h[r];
    __syncthreads();
  }
  const int32_t *pos = in_sh ? pos_sh : rows_h;
  for (int kind = 0; kind < 2; ++kind) {
    const int64_t base = (static_cast<int64_t>(h) * 2 + kind) * n_total;
    const double *w = (kind == 0 ? s_w : v_w) + static_cast<int64_t>(h) * n_total;
    const MaxT *mx = (kind == 0 ? s_max : v_max) + static_cast<int64_t>(h) * n_total;
    for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < n_total; o += gridDim.x * blockDim.x) {
      const int idx = vals_sorted[base + o];
      out.idx[base + o] = idx;
      out.w[base + o] = w[idx];
      out.mx[base + o] = static_cast<double>(mx[idx]);
      // #{rows with g >= idx}, prefill.py:144,155 (g = row_offset + local row)
      out.len[base + o] = n_s - lower_bound_dev(pos, n_s, idx - row_offset);
      out.inv[base + idx] = o;
    }
  }
  (void)keys_sorted;
  (void)H;
}

// K2 for lists of at most 16384 lines (every C2 / C4 turn): the greedy consumes
// only a prefix of each sorted list (picks of one kind), so one CTA per
// (kind, head) finds the PMIN..PCAP best lines by an MSD radix select on the
// same fixed-point keys (2^fix_bits - 1 - w * 2^40: ascending = weight
// descending), sorts just those by (key, index) -- the order of the full stable
// sort -- and marks the rest unsorted (inv = INT_MAX, sorted[h][kind] = P). A
// list with at most PCAP lines is sorted whole. K3 flags a head whose walk would
// leave a sorted prefix; the fallback pair (sort_block_kernel + greedy on the
// flagged heads only) then redoes that head on fully sorted lists, and exits at
// once for every other head.
constexpr int PCAP = 4096;   // prefix capacity (bitonic sort in shared memory)
constexpr int PMIN = 3072;   // at least this many lines (or the whole list) in a prefix
constexpr int PS_THREADS = 1024;
constexpr int PS_ITEMS = 16;  // lines per thread in index order (n_total <= 16384)
constexpr int PS_MAXN = PS_THREADS * PS_ITEMS;
constexpr int PS_BINS = 4096;
inline size_t prefix_sort_smem(int n_s) {
  return PCAP * 12 + PS_BINS * 4 + 256 + (n_s <= kScatterShRows ? 4 * static_cast<size_t>(n_s) : 0);
}

// block exclusive scan of one int per thread (1024 threads); returns the total
__device__ __forceinline__ int block_scan_excl(int v, int &excl, int *warp_sums) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  __syncthreads();
  if (lane == 31) warp_sums[wid] = incl;
  __syncthreads();
  int before = 0, all = 0;
  for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
    const int x = warp_sums[w];
    if (w < wid) before += x;
    all += x;
  }
  excl = before + incl - v;
  return all;
}

// Ascending bitonic sort of PCAP = 4096 distinct u64 keys with 1024 threads:
// thread t holds keys [4t, 4t + 4) in registers; partners within a thread
// (j < 4) by register exchange, within a warp (j < 128) by shuffles, across
// warps through shared memory (15 of the 78 stages).
__device__ void bitonic_sort_pcap(unsigned long long *skey) {
  static_assert(PCAP == 4 * PS_THREADS, "4 entries per thread");
  const int t = threadIdx.x;
  unsigned long long k[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) k[r] = skey[4 * t + r];
  for (int kk = 2; kk <= PCAP; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      if (j >= 4) {
        unsigned long long pk[4];
        if (j >= 128) {  // across warps
          __syncthreads();
#pragma unroll
          for (int r = 0; r < 4; ++r) skey[4 * t + r] = k[r];
          __syncthreads();
#pragma unroll
          for (int r = 0; r < 4; ++r) pk[r] = skey[(4 * t + r) ^ j];
        } else {  // within a warp: partner lane = lane ^ (j / 4)
#pragma unroll
          for (int r = 0; r < 4; ++r) pk[r] = __shfl_xor_sync(0xffffffffu, k[r], j >> 2);
        }
        // (e & kk) and (e & j) are the same for the four entries of a thread (j >= 4)
        const bool keep_min = (((4 * t) & kk) == 0) == (((4 * t) & j) == 0);
#pragma unroll
        for (int r = 0; r < 4; ++r) k[r] = keep_min ? (pk[r] < k[r] ? pk[r] : k[r]) : (pk[r] > k[r] ? pk[r] : k[r]);
      } else {  // within the thread: pairs (r, r | j)
        auto cas = [&](int r, int q) {
          const bool up = ((4 * t + r) & kk) == 0;  // (kk = 2: the two pairs sort in opposite directions)
          const unsigned long long a = k[r], b = k[q];
          const bool sw = up ? (b < a) : (a < b);
          k[r] = sw ? b : a;
          k[q] = sw ? a : b;
        };
        if (j == 2) {
          cas(0, 2);
          cas(1, 3);
        } else {
          cas(0, 1);
          cas(2, 3);
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 4; ++r) skey[4 * t + r] = k[r];
  __syncthreads();
}

template <typename MaxT>
__global__ void __launch_bounds__(PS_THREADS, 1)
    sort_prefix_kernel(const double *v_w, const MaxT *v_max, const double *s_w, const MaxT *s_max,
                       const int32_t *rows, int n_s, int n_total, int row_offset, int fix_bits, Lists out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned long long *skey = reinterpret_cast<unsigned long long *>(smem_raw);  // [PCAP]
  int *hist = reinterpret_cast<int *>(smem_raw + PCAP * 12);                    // [PS_BINS]
  int *red = hist + PS_BINS;                                                     // [64] scan / select scratch
  int *pos_sh = red + 64;
  const int kind = blockIdx.x, h = blockIdx.y, tid = threadIdx.x;
  const double *w = (kind == 0 ? s_w : v_w) + static_cast<int64_t>(h) * n_total;
  const MaxT *mx = (kind == 0 ? s_max : v_max) + static_cast<int64_t>(h) * n_total;
  const int32_t *rows_h = rows + static_cast<int64_t>(h) * n_s;
  const bool in_sh = n_s <= kScatterShRows;
  if (in_sh)
    for (int r = tid; r < n_s; r += PS_THREADS) pos_sh[r] = rows_h[r];
  const int32_t *pos = in_sh ? pos_sh : rows_h;
  if (kind == 0 && tid == 0) out.overflow[h] = 0;
  // select / sort key: the inverted fp64 bits of the weight (weights are exact
  // multiples of 2^-40, non-negative: bit order = value order = the fixed-point
  // order of the full sort); ascending key = weight descending, ties by index
  unsigned long long key[PS_ITEMS];
#pragma unroll
  for (int i = 0; i < PS_ITEMS; ++i) {
    const int idx = tid * PS_ITEMS + i;
    key[i] = idx < n_total ? ~static_cast<unsigned long long>(__double_as_longlong(w[idx])) : 0ull;
  }
  const int n_mine = max(0, min(PS_ITEMS, n_total - tid * PS_ITEMS));  // valid items of this thread
  // ---- MSD radix select (12-bit digits, warp-aggregated histograms, block scans):
  // selection = keys < thr, plus the first `take_eq` lines (index order) with key ==
  // eq_key when a run of equal weights straddles the prefix end
  unsigned long long thr = ~0ull, eq_key = 0ull;
  bool sel_all = n_total <= PCAP;
  int take_eq = 0;
  if (!sel_all) {
    unsigned long long hi_val = 0ull;  // the candidates' key bits above `hi`
    int hi = 64, before = 0;
    while (true) {
      const int lo = max(0, hi - 12), nb = 1 << (hi - lo);
      for (int b = tid; b < PS_BINS; b += PS_THREADS) hist[b] = 0;
      __syncthreads();
      const unsigned long long hmask = hi >= 64 ? 0ull : ~((1ull << hi) - 1ull);
#pragma unroll
      for (int i = 0; i < PS_ITEMS; ++i) {
        const bool cand = i < n_mine && (key[i] & hmask) == (hi >= 64 ? 0ull : (hi_val << hi));
        const int bin = cand ? static_cast<int>((key[i] >> lo) & static_cast<unsigned long long>(nb - 1)) : -1;
        const unsigned grp = __match_any_sync(0xffffffffu, bin);
        if (cand && (threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&hist[bin], __popc(grp));
      }
      __syncthreads();
      // first bin where the running count reaches PMIN (4 bins per thread, block scan)
      int loc = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) loc += hist[tid * 4 + e];
      int excl;
      block_scan_excl(loc, excl, red);
      int c = before + excl;
      if (c < PMIN && c + loc >= PMIN) {
        int b = tid * 4;
        while (c + hist[b] < PMIN) c += hist[b++];
        red[32] = b;
        red[33] = c;
      }
      __syncthreads();
      const int b = red[32];
      c = red[33];
      const int cnt = hist[b];
      __syncthreads();
      const unsigned long long binv = (hi_val << (hi - lo)) | static_cast<unsigned long long>(b);
      if (c + cnt <= PCAP) {  // every candidate up to the end of bin b
        const unsigned long long nxt = binv + 1ull;
        if (lo > 0 ? (nxt >> (64 - lo)) != 0ull : nxt == 0ull)
          sel_all = true;  // bin b ends the key space
        else
          thr = nxt << lo;
        break;
      }
      if (lo == 0) {  // cnt lines of exactly this key: take the first PCAP - c of them
        thr = binv;
        eq_key = binv;
        take_eq = PCAP - c;
        break;
      }
      before = c;
      hi_val = binv;
      hi = lo;
    }
  }
  // ---- compaction in index order
  int mine = 0, mine_eq = 0;
#pragma unroll
  for (int i = 0; i < PS_ITEMS; ++i) {
    mine += (i < n_mine && (sel_all || key[i] < thr)) ? 1 : 0;
    mine_eq += (i < n_mine && take_eq > 0 && key[i] == eq_key) ? 1 : 0;
  }
  int off, off_eq = 0;
  const int n_lt = block_scan_excl(mine, off, red);
  if (take_eq > 0) block_scan_excl(mine_eq, off_eq, red);
  const int P = take_eq > 0 ? PCAP : n_lt;
  // sort keys: (2^fix_bits - 1 - w * 2^40) << 14 | index -- distinct, ascending =
  // (weight desc, index asc); fix_bits <= 50 and n_total <= 2^14 (host-checked)
  const unsigned long long top = (1ull << fix_bits) - 1ull;
  auto packed = [&](int idx) {
    return ((top - static_cast<unsigned long long>(w[idx] * 1099511627776.0)) << 14) |
           static_cast<unsigned long long>(idx);
  };
#pragma unroll
  for (int i = 0; i < PS_ITEMS; ++i) {
    const int idx = tid * PS_ITEMS + i;
    if (i >= n_mine) continue;
    if (sel_all || key[i] < thr) {
      skey[off++] = packed(idx);
    } else if (take_eq > 0 && key[i] == eq_key) {
      if (off_eq < take_eq) skey[n_lt + off_eq] = packed(idx);
      ++off_eq;
    }
  }
  for (int i = P + tid; i < PCAP; i += PS_THREADS) skey[i] = ~0ull;
  // every line starts unsorted (K3 reads inv < picks-of-that-kind as "picked")
  const int64_t base = (static_cast<int64_t>(h) * 2 + kind) * n_total;
  for (int i = tid; i < n_total; i += PS_THREADS) out.inv[base + i] = 0x7fffffff;
  __syncthreads();
  bitonic_sort_pcap(skey);
  for (int o = tid; o < P; o += PS_THREADS) {
    const int idx = static_cast<int>(skey[o] & 16383ull);
    out.idx[base + o] = idx;
    out.w[base + o] = w[idx];
    out.mx[base + o] = static_cast<double>(mx[idx]);
    // #{rows with g >= idx}, prefill.py:144,155 (g = row_offset + local row)
    out.len[base + o] = n_s - lower_bound_dev(pos, n_s, idx - row_offset);
    out.inv[base + idx] = o;
  }
  if (tid == 0) out.sorted[h * 2 + kind] = P;
}

// K2 fallback: the full stable sort of the lists of the heads K3 flagged (one
// CTA per (kind, head) in shared memory); every other CTA exits at once.
constexpr int BS_THREADS = 512;
constexpr int BS_ITEMS = PS_MAXN / BS_THREADS;
using BlockSort = cub::BlockRadixSort<unsigned long long, BS_THREADS, BS_ITEMS, int32_t, 6>;
inline size_t block_sort_smem(int n_s) {
  return sizeof(typename BlockSort::TempStorage) + (n_s <= kScatterShRows ? 4 * static_cast<size_t>(n_s) : 0) + 16;
}

template <typename MaxT>
__global__ void __launch_bounds__(BS_THREADS, 1)
    sort_block_kernel(const double *v_w, const MaxT *v_max, const double *s_w, const MaxT *s_max, const int32_t *rows,
                      int n_s, int n_total, int row_offset, int fix_bits, Lists out) {
  const int kind = blockIdx.x, h = blockIdx.y;
  if (!out.overflow[h]) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto &temp = *reinterpret_cast<typename BlockSort::TempStorage *>(smem_raw);
  int *pos_sh = reinterpret_cast<int *>(smem_raw + sizeof(typename BlockSort::TempStorage));
  const double *w = (kind == 0 ? s_w : v_w) + static_cast<int64_t>(h) * n_total;
  const MaxT *mx = (kind == 0 ? s_max : v_max) + static_cast<int64_t>(h) * n_total;
  const int32_t *rows_h = rows + static_cast<int64_t>(h) * n_s;
  const bool in_sh = n_s <= kScatterShRows;
  if (in_sh)
    for (int r = threadIdx.x; r < n_s; r += BS_THREADS) pos_sh[r] = rows_h[r];
  const int32_t *pos = in_sh ? pos_sh : rows_h;
  const unsigned long long top = (1ull << fix_bits) - 1ull;
  unsigned long long keys[BS_ITEMS];
  int32_t vals[BS_ITEMS];
#pragma unroll
  for (int i = 0; i < BS_ITEMS; ++i) {
    const int idx = threadIdx.x * BS_ITEMS + i;  // blocked arrangement = index order (stability -> idx asc)
    keys[i] = idx < n_total ? top - static_cast<unsigned long long>(w[idx] * 1099511627776.0) : top;
    vals[i] = idx;
  }
  BlockSort(temp).Sort(keys, vals, 0, fix_bits);
  __syncthreads();  // pos_sh (written before the sort) visible
  const int64_t base = (static_cast<int64_t>(h) * 2 + kind) * n_total;
#pragma unroll
  for (int i = 0; i < BS_ITEMS; ++i) {
    const int o = threadIdx.x * BS_ITEMS + i;
    if (o < n_total) {
      const int idx = vals[i];
      out.idx[base + o] = idx;
      out.w[base + o] = w[idx];
      out.mx[base + o] = static_cast<double>(mx[idx]);
      out.len[base + o] = n_s - lower_bound_dev(pos, n_s, idx - row_offset);
      out.inv[base + idx] = o;
    }
  }
  if (threadIdx.x == 0) out.sorted[h * 2 + kind] = n_total;
}

// ------------------------------------------------------- crossing cells
// Cell source 1: recompute P[r, c] from q, k and K1 row statistics.
struct RecomputeCells {
  const uint16_t *q, *k;
  const int32_t *rows;  // [H][n_s] sorted local rows of the sampled block
  const float *row_stats;
  int n_s, n_total, row_offset, d, group;
  int64_t q_head_stride, kv_head_stride;
  float scale_log2;

  __device__ __forceinline__ int n_rows() const { return n_s; }
  __device__ __forceinline__ int pos(int h, int r) const { return row_offset + rows[static_cast<int64_t>(h) * n_s + r]; }
  __device__ __forceinline__ double value(int h, int r, int g, int c) const {
    const uint4 *qr = reinterpret_cast<const uint4 *>(q + static_cast<int64_t>(h) * q_head_stride +
                                                      static_cast<int64_t>(g - row_offset) * d);
    const uint4 *kr = reinterpret_cast<const uint4 *>(k + static_cast<int64_t>(h / group) * kv_head_stride +
                                                      static_cast<int64_t>(c) * d);
    float acc4[4] = {0.f, 0.f, 0.f, 0.f};  // four independent FMA chains
    // two batches of loads in flight (2 L2 round trips per cell at d = 128)
    for (int v = 0; v < d / 8; v += 8) {
      uint4 a[8], b[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a[u] = __ldg(qr + v + u);
        b[u] = __ldg(kr + v + u);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        float fa[8], fb[8];
        bf16x8_to_f32(a[u], fa);
        bf16x8_to_f32(b[u], fb);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc4[j & 3] = fmaf(fa[j], fb[j], acc4[j & 3]);
      }
    }
    const float acc = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
    const float *rs = row_stats + (static_cast<int64_t>(h) * n_s + r) * 2;
    return static_cast<double>(fast_exp2(acc * scale_log2 - rs[0]) * rs[1]);
  }
  // 1/PARTS of the q . k dot product (dims [part * d/PARTS, +d/PARTS)), one batch of loads
  template <int PARTS>
  __device__ __forceinline__ float dot_part(int h, int g, int c, int part) const {
    constexpr int MAXU = 16 / PARTS;  // 16-B chunks per lane at d = 128
    const int nu = d / (8 * PARTS);
    const uint4 *qr = reinterpret_cast<const uint4 *>(q + static_cast<int64_t>(h) * q_head_stride +
                                                      static_cast<int64_t>(g - row_offset) * d) + part * nu;
    const uint4 *kr = reinterpret_cast<const uint4 *>(k + static_cast<int64_t>(h / group) * kv_head_stride +
                                                      static_cast<int64_t>(c) * d) + part * nu;
    uint4 a[MAXU], b[MAXU];
#pragma unroll
    for (int u = 0; u < MAXU; ++u) {
      if (u < nu) {
        a[u] = __ldg(qr + u);
        b[u] = __ldg(kr + u);
      }
    }
    float acc4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int u = 0; u < MAXU; ++u) {
      if (u < nu) {
        float fa[8], fb[8];
        bf16x8_to_f32(a[u], fa);
        bf16x8_to_f32(b[u], fb);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc4[j & 3] = fmaf(fa[j], fb[j], acc4[j & 3]);
      }
    }
    return (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
  }
  __device__ __forceinline__ double finish(int h, int r, float dot, int, int) const {
    const float *rs = row_stats + (static_cast<int64_t>(h) * n_s + r) * 2;
    return static_cast<double>(fast_exp2(dot * scale_log2 - rs[0]) * rs[1]);
  }
};

// Cell source 2: a dense fp64 weight matrix (greedy_select_lines parity path).
struct DenseCells {
  const double *weights;     // [n_rows][n_total]
  const int32_t *positions;  // [n_rows] sorted global positions
  int n_rows_, n_total;
  __device__ __forceinline__ int n_rows() const { return n_rows_; }
  __device__ __forceinline__ int pos(int /*h*/, int r) const { return positions[r]; }
  __device__ __forceinline__ double value(int /*h*/, int r, int /*g*/, int c) const {
    return weights[static_cast<int64_t>(r) * n_total + c];
  }
  template <int PARTS>
  __device__ __forceinline__ float dot_part(int, int, int, int) const { return 0.f; }
  __device__ __forceinline__ double finish(int h, int r, float, int g, int c) const { return value(h, r, g, c); }
};

// ------------------------------------------------------------ K3 greedy
// One CTA per head, warp-specialised so that only the decision chain is
// sequential and the exact-mass bookkeeping runs concurrently with it:
//   warp 0, lane 0  producer: replays the decision chain of _greedy
//                   (prefill.py:195-220) in fp64 over the sorted lists staged
//                   in shared memory -- decisions depend on approx, ol_s, ol_v,
//                   |S|, |V| only -- and publishes every pick (code, weight,
//                   approx after it, picks of the other kind before it).
//   warps 2..15     crossing sums, one warp per pick (prefill.py:211, 217): the
//                   cells of the pick's line with the other kind's picked
//                   prefix. A cell exists only at a sampled row g = c + d
//                   (_BlockView.cell, prefill.py:116-122), so the warp walks the
//                   sampled rows g >= line index and tests the other line's
//                   sorted-list position against the prefix length (an
//                   inverse permutation from K2) -- O(n_s) per pick, fully
//                   independent of the other picks. Fixed-order warp sum.
//   warp 1, lane 0  finalizer: exact += w - cross in selection order and the
//                   reference's dual termination test (prefill.py:195); it
//                   stops the producer as soon as the plan is complete.
constexpr int WIN = 1024;            // staged lines per list
constexpr int TAB_CAP = 16384;       // n_total up to which position tables live in shared memory
constexpr int G_THREADS = 640;       // 20 warps
constexpr int RING = 1024;           // pick slots between producer and finalizer
constexpr int AHEAD = 512;           // the producer runs at most this far ahead of the finalizer: picks
                                     // past the plan's end cost crossing sums for nothing
constexpr int GS_CAP = 8192;         // sampled positions kept in shared memory
constexpr int BM_WORDS = TAB_CAP;    // bitmap words when n_total > TAB_CAP (the tables' space): n_total <= 2^19

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

struct GreedySmem {
  int32_t idx[2][WIN];
  int32_t len[2][WIN];
  double w[2][WIN];
  double mx[2][WIN];
  double r_w[RING], r_approx[RING], r_cross[RING];
  int32_t r_code[RING], r_other[RING], r_seq[RING];
  int32_t gs[GS_CAP];
  union {
    struct {
      int16_t rowof[TAB_CAP];    // position -> sampled row, or -1
      uint16_t inv[2][TAB_CAP];  // line index -> sorted position (clamped to 65535)
    } t;                         // n_total <= TAB_CAP
    struct {
      uint32_t bits[BM_WORDS];   // sampled positions (bit g)
      int16_t rank[BM_WORDS];    // sampled positions before word w
    } b;                         // larger n_total: position -> row by bitmap rank
  } tab;
  int32_t hitq[G_THREADS / 32][64];  // per consumer warp: sampled rows of crossing cells awaiting a value
  double fold_w[32], fold_m[32];     // producer: the round's R-side weights / max cells
};

__device__ __forceinline__ int vload(const volatile int *p) { return *p; }

// spin-wait guard: a protocol bug surfaces as a launch error after ~10 s
// instead of a hung device (the clock is read once every 1024 polls)
struct SpinGuard {
  long long t0 = -1;
  unsigned n = 0;
  __device__ __forceinline__ void tick() {
    if ((++n & 1023u) != 0u) return;
    const long long now = clock64();
    if (t0 < 0) t0 = now;
    else if (now - t0 > 20000000000LL) __trap();
  }
};

#ifndef LS_GREEDY_IDLE_SMSP
#define LS_GREEDY_IDLE_SMSP 0  // measured: idling warps 4, 8, 12, 16 starves the crossing sums
#endif
constexpr bool g_idle_producer_smsp = LS_GREEDY_IDLE_SMSP != 0;

template <typename Cells>
__global__ void __launch_bounds__(G_THREADS, 1) greedy_kernel(Lists L, int n_total, double alpha, const double *total,
                                                               Picks P, int cap, Cells cells, int32_t *n_final,
                                                               double *coverage, double *approx_out, int *dbg,
                                                               int only_overflowed, PlanOut po) {
  extern __shared__ __align__(16) unsigned char g_smem[];
  const long long t_start = clock64();
  GreedySmem &S = *reinterpret_cast<GreedySmem *>(g_smem);
  __shared__ volatile int n_prod, prod_done, fin_pos, stop_at;
  __shared__ int next_j;
  __shared__ unsigned long long busy_cyc;  // diagnostics: consumer cycles spent on crossing sums
  const int h = blockIdx.x;
  // the K2 fallback pass re-runs only the heads whose walk left a sorted prefix
  if (only_overflowed && !L.overflow[h]) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double T = total[h];
  // sorted prefix of each list (K2 prefix sort); a walk that would read past one
  // stops and flags the head for the fallback pass
  const int srt_s = L.sorted ? L.sorted[h * 2] : n_total, srt_v = L.sorted ? L.sorted[h * 2 + 1] : n_total;
  const double target = alpha * T;
  const int64_t lb = static_cast<int64_t>(h) * 2 * n_total;
  const int64_t pb = static_cast<int64_t>(h) * cap;
  const int n_rows = cells.n_rows();
  const bool gs_smem = n_rows <= GS_CAP;
  const int win = min(WIN, n_total);
  for (int i = threadIdx.x; i < 2 * win; i += blockDim.x) {
    const int kind = i / win, o = i % win;
    const int64_t g = lb + static_cast<int64_t>(kind) * n_total + o;
    S.idx[kind][o] = L.idx[g];
    S.len[kind][o] = L.len[g];
    S.w[kind][o] = L.w[g];
    S.mx[kind][o] = L.mx[g];
  }
  if (gs_smem)
    for (int r = threadIdx.x; r < n_rows; r += blockDim.x) S.gs[r] = cells.pos(h, r);
  for (int i = threadIdx.x; i < RING; i += blockDim.x) S.r_seq[i] = 0;
  const bool tabs = n_total <= TAB_CAP && gs_smem;
  const int bm_words = (n_total + 31) >> 5;
  const bool bmap = !tabs && gs_smem && bm_words <= BM_WORDS;
  if (tabs) {
    for (int i = threadIdx.x; i < n_total; i += blockDim.x) {
      S.tab.t.rowof[i] = -1;
      S.tab.t.inv[0][i] = static_cast<uint16_t>(min(L.inv[lb + i], 65535));
      S.tab.t.inv[1][i] = static_cast<uint16_t>(min(L.inv[lb + n_total + i], 65535));
    }
    __syncthreads();
    for (int r = threadIdx.x; r < n_rows; r += blockDim.x) S.tab.t.rowof[S.gs[r]] = static_cast<int16_t>(r);
  } else if (bmap) {
    for (int w = threadIdx.x; w < bm_words; w += blockDim.x) S.tab.b.bits[w] = 0u;
    __syncthreads();
    for (int r = threadIdx.x; r < n_rows; r += blockDim.x) atomicOr(&S.tab.b.bits[S.gs[r] >> 5], 1u << (S.gs[r] & 31));
    __syncthreads();
    // rank of word w = sampled rows before it = first row with position >= 32 w (rows are sorted)
    for (int w = threadIdx.x; w < bm_words; w += blockDim.x)
      S.tab.b.rank[w] = static_cast<int16_t>(lower_bound_dev(S.gs, n_rows, w << 5));
  }
  // sampled row at position g (< n_total), or -1
  auto row_at = [&](int g) -> int {
    if (tabs) return S.tab.t.rowof[g];
    const uint32_t wbits = S.tab.b.bits[g >> 5], bit = 1u << (g & 31);
    return (wbits & bit) ? S.tab.b.rank[g >> 5] + __popc(wbits & (bit - 1u)) : -1;
  };
  if (threadIdx.x == 0) {
    n_prod = 0;
    prod_done = 0;
    fin_pos = 0;
    stop_at = 0x7fffffff;
    next_j = 0;
    busy_cyc = 0ull;
  }
  __syncthreads();
  const int32_t *inv_s = L.inv + lb, *inv_v = L.inv + lb + n_total;

  if (warp == 0) {
    // ================================================= producer (chain)
    // Run speculation: most picks come in runs of one kind. While kind R is
    // being picked, the other kind's head, ol_other, and its count are
    // fixed, and the R-side state after j more R picks follows from
    // sequential folds over the next R heads. Each round the warp evaluates
    // the decisions for the next K picks of kind R in parallel (lane j = "j R
    // picks taken"), the folds being computed redundantly by every lane in
    // the reference's order (bit-identical approx / ol), then takes the
    // longest prefix of R picks plus the O pick that breaks the run.
    int s_idx = 0, v_idx = 0, n = 0, R = 1, K = 8;
    double ol_s = 0.0, ol_v = 0.0, approx = 0.0;
    bool go = 0.0 < target - EPS;  // the while condition before any pick
    int stop_seen = 0x7fffffff, fin_seen = 0;
    long long wait_cycles = 0;
    auto head = [&](int kind, int i, double &w, double &mx, int &len, int &ix) {
      if (i >= n_total) {
        w = 0.0; mx = 0.0; len = 0; ix = 0;
      } else if (i < win) {
        w = S.w[kind][i]; mx = S.mx[kind][i]; len = S.len[kind][i]; ix = S.idx[kind][i];
      } else {
        const int64_t g = lb + static_cast<int64_t>(kind) * n_total + i;
        w = L.w[g]; mx = L.mx[g]; len = L.len[g]; ix = L.idx[g];
      }
    };
    int rounds = 0;
    int pf_kind = -1, pf_base = -1;  // prefetched R-side window of the next round
    double pf_w = 0.0, pf_mx = 0.0;
    int pf_len = 0, pf_ix = 0;
    long long ph[4] = {0, 0, 0, 0};  // diagnostics: producer phase cycles (dbg)
    while (go) {
      ++rounds;
      if ((s_idx >= n_total && v_idx >= n_total) || n >= cap) break;
      // a round reads at most 64 entries past either walk position (window + prefetch)
      if ((srt_s < n_total && s_idx + 64 > srt_s) || (srt_v < n_total && v_idx + 64 > srt_v)) {
        if (lane == 0) L.overflow[h] = 1;
        break;
      }
      stop_seen = __shfl_sync(0xffffffffu, lane == 0 ? stop_at : 0, 0);  // one read: the warp must agree
      if (n >= stop_seen) break;
      int stopped = 0;
      if (lane == 0 && n + 33 - fin_seen > AHEAD) {
        fin_seen = fin_pos;
        const long long tw = clock64();
        SpinGuard guard;
        while (n + 33 - fin_seen > AHEAD) {  // far enough ahead: wait for the finalizer
          if (stop_at <= n) {  // the finalizer has stopped the plan: it will not free the ring
            stopped = 1;
            break;
          }
          __nanosleep(64);
          fin_seen = fin_pos;
          guard.tick();
        }
        wait_cycles += clock64() - tw;
      }
      if (__shfl_sync(0xffffffffu, stopped, 0)) break;
      fin_seen = __shfl_sync(0xffffffffu, fin_seen, 0);
      const bool prof = dbg != nullptr;  // phase clocks only when profiling (ls_debug_set_buffer)
      const long long c0 = prof ? clock64() : 0;
      const int O = 1 - R;
      const int base_R = R ? v_idx : s_idx, base_O = R ? s_idx : v_idx;
      double wR, mxR, wO, mxO;
      int lR, iR, lO, iO;
      if (pf_kind == R && pf_base == base_R) {  // the window loaded during the previous round
        wR = pf_w; mxR = pf_mx; lR = pf_len; iR = pf_ix;
      } else {
        head(R, base_R + lane, wR, mxR, lR, iR);
      }
      head(O, base_O, wO, mxO, lO, iO);
      const double olR0 = R ? ol_v : ol_s, olO = R ? ol_s : ol_v;
      const long long c1 = prof ? clock64() + (static_cast<long long>(wR + wO + mxR + mxO + lR + lO + iR + iO) & 0) : 0;
      // folds in reference order: state before R pick j (ol_R, approx)
      double my_ol = olR0, my_ap = approx, ol_run = olR0, ap_run = approx;
      // the round's R-side values, lane j = entry base_R + j, staged for the fold
      // (which every lane runs redundantly in the reference's sequential order)
      S.fold_w[lane] = wR;
      S.fold_m[lane] = mxR;
      __syncwarp();
#pragma unroll
      for (int c = 0; c < 32; c += 8) {
        if (c < K) {
          double wv[8], mv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {  // 16 broadcast loads in flight, then the chains
            wv[u] = S.fold_w[c + u] - olO;
            mv[u] = S.fold_m[c + u];
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int i = c + u;
            const bool take = lane == i;
            my_ol = take ? ol_run : my_ol;
            my_ap = take ? ap_run : my_ap;
            if (i < K) {
              ap_run += wv[u];  // approx += w - ol_other (prefill.py:210, 216)
              ol_run += mv[u];  // ol_R += max_cell (prefill.py:212, 218)
            }
          }
        }
      }
      __syncwarp();
      const long long c2 = prof ? clock64() + (static_cast<long long>(my_ol + my_ap + ol_run + ap_run) & 0) : 0;
      // decision at (j = lane) R picks taken
      const int sj = R ? s_idx : s_idx + lane, vj = R ? v_idx + lane : v_idx;
      const bool has_s = sj < n_total, has_v = vj < n_total;
      bool take_slash;
      if (!has_s) {
        take_slash = false;
      } else if (!has_v) {
        take_slash = true;
      } else if (R) {  // vertical run: slash side fixed, ol_v = my_ol
        take_slash = take_slash_decision(wO - my_ol, max(1, lO - vj), wR - olO, max(1, lR - sj));
      } else {         // slash run: vertical side fixed, ol_s = my_ol
        take_slash = take_slash_decision(wR - olO, max(1, lR - vj), wO - my_ol, max(1, lO - sj));
      }
      const bool exists = has_s || has_v;
      const bool takes_R = exists && (take_slash == (R == 0));
      const double ap_after = my_ap + (wR - olO);  // approx after this R pick
      const bool stops = takes_R && !(ap_after < target - EPS);
      // run = leading lanes (< K) taking R; cut after the first approx stop, at cap
      const unsigned not_r = __ballot_sync(0xffffffffu, !takes_R || lane >= K);
      int f = not_r ? __ffs(not_r) - 1 : 32;
      const unsigned st_b = __ballot_sync(0xffffffffu, stops && lane < f);
      bool chain_end = false;
      if (st_b) {
        f = __ffs(st_b);
        chain_end = true;
      }
      if (n + f >= cap) {
        f = cap - n;
        chain_end = true;
      }
      // the next round most likely continues this kind at base_R + f: start its
      // window's loads now (L2 beyond the staged WIN entries) so they land while
      // this round publishes
      pf_kind = R;
      pf_base = base_R + f;
      head(R, pf_base + lane, pf_w, pf_mx, pf_len, pf_ix);
      const long long c3 = prof ? clock64() : 0;
      if (lane < f) {  // publish the R picks
        const int slot = (n + lane) % RING;
        S.r_code[slot] = R ? (iR | static_cast<int32_t>(0x80000000u)) : iR;
        S.r_other[slot] = base_O;
        S.r_w[slot] = wR;
        S.r_approx[slot] = ap_after;
      }
      // state after the f R picks (lane f's "before" state)
      const double ol_f = __shfl_sync(0xffffffffu, my_ol, f & 31);
      const double ap_f = __shfl_sync(0xffffffffu, my_ap, f & 31);
      const bool run_broke = !chain_end && f < K;           // lane f decided for O
      const bool o_exists = R ? (s_idx < n_total) : (v_idx < n_total);
      const bool exists_f = __shfl_sync(0xffffffffu, exists ? 1 : 0, f & 31);
      double ol_R = f == 0 ? olR0 : (f < 32 ? ol_f : ol_run), ap = f == 0 ? approx : (f < 32 ? ap_f : ap_run);
      if (f == K && K < 32) {  // whole window taken: fold state after K picks
        ol_R = ol_run;
        ap = ap_run;
      }
      int np = f;
      bool o_pick = run_broke && o_exists && exists_f;
      if (o_pick) {  // the O pick that breaks the run (ol_R, |R| after the f R picks)
        ap += wO - ol_R;
        if (lane == 0) {
          const int slot = (n + f) % RING;
          S.r_code[slot] = O ? (iO | static_cast<int32_t>(0x80000000u)) : iO;
          S.r_other[slot] = base_R + f;
          S.r_w[slot] = wO;
          S.r_approx[slot] = ap;
        }
        np = f + 1;
        if (!(ap < target - EPS)) chain_end = true;
      }
      __syncwarp();
      n += np;
      if (lane == 0) {
        __threadfence_block();
        n_prod = n;
      }
      // advance the state
      if (R) { v_idx += f; ol_v = ol_R; } else { s_idx += f; ol_s = ol_R; }
      if (o_pick) {
        if (R) { ++s_idx; ol_s += mxO; } else { ++v_idx; ol_v += mxO; }
      }
      approx = ap;
      if (chain_end || np == 0) go = false;
      if (!(approx < target - EPS)) go = false;
      if (prof && lane == 0) {
        const long long c4 = clock64();
        ph[0] += c1 - c0;
        ph[1] += c2 - c1;
        ph[2] += c3 - c2;
        ph[3] += c4 - c3;
      }
      // next window: keep speculating on R while its runs are long
      if (f >= 2) {
        K = f >= K ? min(32, 2 * K) : max(4, min(32, 2 * f + 2));
      } else {
        R = 1 - R;
        K = 4;
      }
    }
    if (lane == 0) {
      __threadfence_block();
      prod_done = 1;
      if (dbg) {
        dbg[60000 + blockIdx.x * 8 + 0] = n;
        dbg[60000 + blockIdx.x * 8 + 2] = static_cast<int>(clock64() - t_start);
        dbg[60000 + blockIdx.x * 8 + 4] = static_cast<int>(wait_cycles);
        dbg[60000 + blockIdx.x * 8 + 7] = rounds;
        for (int k = 0; k < 4; ++k) dbg[61000 + blockIdx.x * 4 + k] = static_cast<int>(ph[k]);
      }
    }
  } else if (warp == 1) {
    // ================================================= finalizer
    // The whole warp: lanes test the readiness of picks j .. j+31 at once and
    // load the ready prefix in parallel; the exact-mass chain and the dual
    // termination test then run over it in selection order (every lane
    // redundantly, values by shuffle) -- the reference's sequential fp64 order.
    double exact = 0.0, approx = 0.0;
    int j = 0;
    long long fwait = 0;
    const bool no_cross = dbg && dbg[69999] == 1;
    while (true) {
      const long long tw0 = clock64();
      SpinGuard guard;
      int m = 0;
      bool done = false;
      while (true) {
        const int slot = (j + lane) % RING;
        const bool ready = vload(S.r_seq + slot) == j + lane + 1;
        const unsigned rb = __ballot_sync(0xffffffffu, ready);
        m = rb == 0xffffffffu ? 32 : __ffs(~rb) - 1;  // contiguous ready prefix
        if (m > 0) break;
        int pd = prod_done, np = 0;
        if (pd) {
          __threadfence_block();
          np = n_prod;
        }
        if (__shfl_sync(0xffffffffu, pd && j >= np ? 1 : 0, 0)) {  // every published pick consumed
          done = true;
          break;
        }
        if (lane == 0) guard.tick();
        __nanosleep(32);
      }
      fwait += clock64() - tw0;
      if (done) break;
      __threadfence_block();  // the ready picks' fields were written before their sequence numbers
      const int slot = (j + lane) % RING;
      double wc = 0.0, ap_l = 0.0;
      if (lane < m) {
        wc = static_cast<const volatile double *>(S.r_w)[slot] - static_cast<const volatile double *>(S.r_cross)[slot];
        ap_l = static_cast<const volatile double *>(S.r_approx)[slot];
        P.code[pb + j + lane] = static_cast<const volatile int32_t *>(S.r_code)[slot];
      }
      int took = m;
      bool stop = false;
      for (int k = 0; k < m; ++k) {
        exact += __shfl_sync(0xffffffffu, wc, k);
        approx = __shfl_sync(0xffffffffu, ap_l, k);
        if (!(approx < target - EPS && (exact < target - EPS || no_cross))) {
          took = k + 1;
          stop = true;
          break;
        }
      }
      j += took;
      if (lane == 0) fin_pos = j;
      if (stop) break;
    }
    if (lane == 0) {
      stop_at = j;
      if (dbg) {
        dbg[60000 + blockIdx.x * 8 + 1] = j;
        dbg[60000 + blockIdx.x * 8 + 3] = static_cast<int>(clock64() - t_start);
        dbg[60000 + blockIdx.x * 8 + 5] = static_cast<int>(fwait);
        dbg[60000 + blockIdx.x * 8 + 6] = static_cast<int>(busy_cyc / 16);
      }
      P.n[h] = j;
      n_final[h] = j;
      const double cov = T > 0 ? exact / T : 0.0;  // prefill.py:221
      coverage[h] = cov < 1.0 ? cov : 1.0;
      approx_out[h] = j > 0 ? approx : 0.0;
    }
  } else if ((warp & 3) == 0 && g_idle_producer_smsp) {
    // the producer's scheduler (SM sub-partition) is left to the decision chain
  } else {
    // ================================================= crossing sums
    // (warps 4, 8, 12 share the producer's scheduler: they are consumers too;
    // measured: idling them starves the finalizer)
    while (true) {
      int j = 0;
      if (lane == 0) j = atomicAdd(&next_j, 1);
      j = __shfl_sync(0xffffffffu, j, 0);
      bool ok = false;
      if (lane == 0) {
        SpinGuard guard;
        while (true) {
          guard.tick();
          if (j < n_prod) { ok = true; break; }
          if (j >= stop_at) break;
          if (prod_done) {  // the last n_prod store precedes prod_done: re-read it after the flag
            __threadfence_block();
            ok = j < n_prod;
            break;
          }
          __nanosleep(256);
        }
        if (j >= stop_at) ok = false;
      }
      ok = __shfl_sync(0xffffffffu, ok ? 1 : 0, 0);
      if (!ok) break;
      const long long tb0 = clock64();
      const int slot = j % RING;
      const int32_t code = static_cast<const volatile int32_t *>(S.r_code)[slot];
      const int n_other = static_cast<const volatile int32_t *>(S.r_other)[slot];
      const bool is_vert = code < 0;
      const int idx = code & 0x7fffffff;
      const int32_t *inv_o = is_vert ? inv_s : inv_v;  // other kind's sorted positions
      double sum = 0.0;
      if (n_other > 0 && !(dbg && dbg[69999] == 1)) {
        // sampled rows at or after position idx: g = idx + (other line index).
        // Warp-wide 32-ary search: two probe rounds for n_rows <= 1024
        int lo = 0;
        {
          int hi = n_rows;  // first row with g >= idx lies in [lo, hi]
          while (hi - lo > 32) {
            const int stp = (hi - lo + 31) / 32;
            const int p = lo + lane * stp;
            const bool lt = p < hi && (gs_smem ? S.gs[p] : cells.pos(h, p)) < idx;
            const int c = __popc(__ballot_sync(0xffffffffu, lt));
            const int nlo = c == 0 ? lo : lo + (c - 1) * stp + 1;
            hi = min(hi, lo + c * stp);
            lo = nlo;
          }
          const int p = lo + lane;
          const bool lt = p < hi && (gs_smem ? S.gs[p] : cells.pos(h, p)) < idx;
          lo += __popc(__ballot_sync(0xffffffffu, lt));
        }
        const int okind = is_vert ? 0 : 1;
        // crossing cells are sparse among the walked candidates: queue their
        // sampled rows and evaluate them 32 at a time, one per lane, so each
        // cell recompute (two L2 round trips) runs with the whole warp busy
        int *q = S.hitq[warp];
        int qn = 0;
        const unsigned lt = (1u << lane) - 1u;
        auto eval = [&](int n) {  // value of queue entries [0, n)
          if (n <= 8) {
            // few cells (most vertical picks): four lanes per cell, a quarter of
            // the dot product each -- one L2 round trip instead of two
            const int e = lane >> 2, part = lane & 3;
            const bool act = e < n;
            const int r = act ? q[e] : 0;
            const int g = act ? (gs_smem ? S.gs[r] : cells.pos(h, r)) : 0;
            float dot = act ? cells.template dot_part<4>(h, g, is_vert ? idx : g - idx, part) : 0.f;
            dot += __shfl_xor_sync(0xffffffffu, dot, 1);
            dot += __shfl_xor_sync(0xffffffffu, dot, 2);
            if (act && part == 0) sum += cells.finish(h, r, dot, g, is_vert ? idx : g - idx);
            return;
          }
          const bool act = lane < n;  // lane i takes entry i
          const int r = act ? q[lane] : 0;
          const int g = act ? (gs_smem ? S.gs[r] : cells.pos(h, r)) : 0;
          if (act) sum += cells.value(h, r, g, is_vert ? idx : g - idx);
        };
        auto push = [&](bool hit, int r) {
          const unsigned b = __ballot_sync(0xffffffffu, hit);
          if (hit) q[qn + __popc(b & lt)] = r;
          qn += __popc(b);
          __syncwarp();
          if (qn >= 32) {
            eval(32);
            const int t = lane < qn - 32 ? q[32 + lane] : 0;
            __syncwarp();
            if (lane < qn - 32) q[lane] = t;
            qn -= 32;
            __syncwarp();
          }
        };
        if ((tabs || bmap) && n_other < n_rows - lo) {
          // walk the other kind's picked prefix: cell at g = idx + o if g is sampled
          for (int i0 = 0; i0 < n_other; i0 += 32) {
            const int i = i0 + lane;
            int o = -1;
            if (i < n_other) o = i < win ? S.idx[okind][i] : __ldg(L.idx + lb + static_cast<int64_t>(okind) * n_total + i);
            const int g = idx + o;
            const int r = (o >= 0 && g < n_total) ? row_at(g) : -1;
            push(r >= 0, r);
          }
        } else {
          // walk the sampled rows: the other line o = g - idx is picked iff its
          // sorted position is below the prefix length
          const int32_t *inv_o = is_vert ? inv_s : inv_v;
          if (tabs) {
            for (int r0 = lo; r0 < n_rows; r0 += 32) {
              const int r = r0 + lane;
              bool hit = false;
              if (r < n_rows) hit = static_cast<int>(S.tab.t.inv[okind][S.gs[r] - idx]) < n_other;
              push(hit, r);
            }
          } else {
            // positions from L2: four independent loads per lane in flight
            for (int r0 = lo; r0 < n_rows; r0 += 128) {
              int pos[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int r = r0 + 32 * u + lane;
                pos[u] = r < n_rows ? __ldg(inv_o + ((gs_smem ? S.gs[r] : cells.pos(h, r)) - idx)) : 0x7fffffff;
              }
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                if (r0 + 32 * u >= n_rows) break;  // warp-uniform
                push(pos[u] < n_other, r0 + 32 * u + lane);
              }
            }
          }
        }
        eval(qn);
        __syncwarp();
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane == 0) {
        static_cast<volatile double *>(S.r_cross)[slot] = sum;
        __threadfence_block();
        static_cast<volatile int32_t *>(S.r_seq)[slot] = j + 1;
        if (dbg) atomicAdd(&busy_cyc, static_cast<unsigned long long>(clock64() - tb0));
      }
    }
  }
  if (po.ready == nullptr) return;
  // ---- fused K4: picks -> bitmaps -> sorted id lists of this head, then its flag
  // (a head that left a sorted prefix publishes only from the fallback pass)
  __syncthreads();
  const bool publish = only_overflowed || L.overflow == nullptr || !L.overflow[h];
  if (!publish) return;
  uint32_t *sb = po.sbits + static_cast<int64_t>(h) * po.words, *vb = po.vbits + static_cast<int64_t>(h) * po.words;
  for (int w = threadIdx.x; w < po.words; w += blockDim.x) sb[w] = vb[w] = 0u;
  __syncthreads();
  const int nf = static_cast<const volatile int32_t *>(n_final)[h];
  for (int t = threadIdx.x; t < nf; t += blockDim.x) {
    const int32_t code = P.code[pb + t];
    const int idx = code & 0x7fffffff;
    atomicOr((code < 0 ? vb : sb) + (idx >> 5), 1u << (idx & 31));
    if (po.picks_out) po.picks_out[static_cast<int64_t>(h) * 2 * n_total + t] = code;
  }
  __syncthreads();
  __shared__ int scan_sh[G_THREADS / 32];
  for (int kind = 0; kind < 2; ++kind) {
    const uint32_t *bits = kind == 0 ? sb : vb;
    int32_t *out = (kind == 0 ? po.slash_ids : po.vert_ids) + static_cast<int64_t>(h) * n_total;
    int base = 0;
    for (int w0 = 0; w0 < po.words; w0 += blockDim.x) {
      const int w = w0 + threadIdx.x;
      uint32_t x = w < po.words ? bits[w] : 0u;
      // block exclusive scan of the popcounts
      const int c = __popc(x);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) scan_sh[warp] = incl;
      __syncthreads();
      int before = 0, all = 0;
      for (int k = 0; k < G_THREADS / 32; ++k) {
        if (k < warp) before += scan_sh[k];
        all += scan_sh[k];
      }
      int pos = base + before + incl - c;
      while (x) {
        const int b = __ffs(x) - 1;
        x &= x - 1;
        out[pos++] = w * 32 + b;
      }
      base += all;
      __syncthreads();
    }
    if (threadIdx.x == 0) po.counts[h * 2 + kind] = base;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicExch(po.ready + h, po.epoch);
  }
}

template <typename Cells>
int launch_greedy(const Lists &lists, int H, int n_total, double alpha, const double *total, Picks &picks, int cap,
                  const Cells &cells, int32_t *n_final, double *coverage, double *approx, cudaStream_t st,
                  int only_overflowed = 0, PlanOut po = PlanOut{}) {
  const int smem = static_cast<int>(sizeof(GreedySmem));
  LS_CUDA(cudaFuncSetAttribute(greedy_kernel<Cells>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  greedy_kernel<Cells><<<H, G_THREADS, smem, st>>>(lists, n_total, alpha, total, picks, cap, cells, n_final, coverage,
                                                   approx, g_debug_buffer, only_overflowed, po);
  LS_LAUNCH_CHECK("greedy_kernel");
  return LS_OK;
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

struct Work {
  Lists lists;
  Picks picks;
  uint32_t *sbits, *vbits;
  int32_t *n_final;
  int words, cap;
};

inline Work carve(Carver &c, int H, int n_total) {
  Work w;
  const size_t nl = static_cast<size_t>(H) * 2 * n_total;
  w.cap = 2 * n_total;
  const size_t np = static_cast<size_t>(H) * w.cap;
  w.lists.sorted = nullptr;  // set by the K2 prefix path
  w.lists.overflow = c.take<int32_t>(static_cast<size_t>(H) * 3);
  w.lists.idx = c.take<int32_t>(nl);
  w.lists.inv = c.take<int32_t>(nl);
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
  return w;
}


inline size_t radix_temp_bytes(int H, int n_total) {
  size_t bytes = 0;
  const int n = 2 * H * n_total;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, static_cast<const unsigned long long *>(nullptr),
                                  static_cast<unsigned long long *>(nullptr), static_cast<const int32_t *>(nullptr),
                                  static_cast<int32_t *>(nullptr), n, 0, 64);
  return bytes;
}

struct SortWork {
  unsigned long long *k_in, *k_out;
  int32_t *v_in, *v_out;
  void *temp;
  size_t temp_bytes;
};

inline SortWork carve_sort(Carver &c, int H, int n_total) {
  SortWork w;
  const size_t n = static_cast<size_t>(2) * H * n_total;
  w.k_in = c.take<unsigned long long>(n);
  w.k_out = c.take<unsigned long long>(n);
  w.v_in = c.take<int32_t>(n);
  w.v_out = c.take<int32_t>(n);
  w.temp_bytes = radix_temp_bytes(H, n_total);
  w.temp = c.take<unsigned char>(w.temp_bytes);
  return w;
}

int run_tail(Work &w, int H, int n_total, double alpha, const double *total, int32_t *slash_ids,
             int32_t *vert_ids, int32_t *counts, double *coverage, double *approx, int32_t *picks_out,
             int32_t *n_picks_out, cudaStream_t st) {
  // sbits and vbits are consecutive in the workspace: one memset
  LS_CUDA(cudaMemsetAsync(w.sbits, 0, reinterpret_cast<char *>(w.vbits + static_cast<size_t>(H) * w.words) -
                                          reinterpret_cast<char *>(w.sbits), st));
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
  sel::carve(c, L->n_heads, L->n_total);
  sel::carve_sort(c, L->n_heads, L->n_total);
  return c.off + 4096;
}

extern "C" int ls_select_lines_ready(const ls_layer_desc *L, int32_t n_s, double alpha, const uint16_t *q,
                                     const uint16_t *k, const int32_t *rows, const double *v_w, const float *v_max,
                                     const double *s_w, const float *s_max, const float *row_stats,
                                     const double *total, int32_t *slash_ids, int32_t *vert_ids, int32_t *counts,
                                     double *coverage, double *approx, int32_t *picks, int32_t *n_picks,
                                     int32_t *plan_ready, int32_t epoch, void *ws, size_t ws_bytes,
                                     ls_stream_t stream) {
  LS_REQUIRE(alpha >= 0.0 && alpha <= 1.0, LS_ERR_INVALID_ALPHA, "alpha=%g outside [0, 1]", alpha);
  const int fix_bits = sel::fix_bits_for(n_s);
  int seg_bits = 1;
  while ((1 << seg_bits) < 2 * L->n_heads) ++seg_bits;
  LS_REQUIRE(fix_bits + seg_bits <= 64, LS_ERR_UNSUPPORTED, "sort key too wide (%d heads, %d sampled rows)",
             L->n_heads, n_s);
  LS_REQUIRE(ws_bytes >= ls_select_lines_workspace(L, n_s), LS_ERR_WORKSPACE, "select_lines workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int H = L->n_heads, n_total = L->n_total;
  Carver c(ws, ws_bytes);
  sel::Work w = sel::carve(c, H, n_total);
  sel::SortWork sw = sel::carve_sort(c, H, n_total);
  // fused K4 + per-head readiness flags (plan_ready): the head's CTA writes its plan
  const sel::PlanOut po = plan_ready ? sel::PlanOut{w.sbits, w.vbits, w.words, slash_ids, vert_ids, counts, picks,
                                                    plan_ready, epoch}
                                     : sel::PlanOut{};
  const bool prefix = n_total <= sel::PS_MAXN && fix_bits <= 50;  // packed (key, index) sort keys fit 64 bits
  if (!prefix) w.lists.overflow = nullptr;  // fully sorted lists: no fallback pass
  if (prefix) {
    w.lists.sorted = w.lists.overflow + H;
    const size_t smem = sel::prefix_sort_smem(n_s);
    LS_CUDA(cudaFuncSetAttribute(sel::sort_prefix_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    sel::sort_prefix_kernel<float><<<dim3(2, H), sel::PS_THREADS, smem, st>>>(v_w, v_max, s_w, s_max, rows, n_s,
                                                                            n_total, L->row_offset, fix_bits, w.lists);
    LS_LAUNCH_CHECK("sort_prefix_kernel");
  } else {
    const int n = 2 * H * n_total;
    sel::sort_keys_kernel<<<std::min(ceil_div(n, 256), 148 * 8), 256, 0, st>>>(v_w, s_w, H, n_total, fix_bits,
                                                                                sw.k_in, sw.v_in);
    LS_LAUNCH_CHECK("sort_keys_kernel");
    size_t tb = sw.temp_bytes;
    LS_CUDA(cub::DeviceRadixSort::SortPairs(sw.temp, tb, sw.k_in, sw.k_out, sw.v_in, sw.v_out, n, 0,
                                            fix_bits + seg_bits, st));
    const int smem_pos = n_s <= sel::kScatterShRows ? n_s * 4 : 0;
    sel::sort_scatter_kernel<float><<<dim3(std::max(1, std::min(ceil_div(n_total, 256), 16)), H), 256, smem_pos, st>>>(
        sw.k_out, sw.v_out, v_w, v_max, s_w, s_max, rows, n_s, n_total, L->row_offset, H, w.lists);
    LS_LAUNCH_CHECK("sort_scatter_kernel");
  }
  sel::RecomputeCells cells;
  cells.q = q;
  cells.k = k;
  cells.rows = rows;
  cells.row_stats = row_stats;
  cells.n_s = n_s;
  cells.n_total = n_total;
  cells.row_offset = L->row_offset;
  cells.d = L->head_dim;
  cells.group = L->n_heads / L->n_kv_heads;
  cells.q_head_stride = L->q_head_stride;
  cells.kv_head_stride = L->kv_head_stride;
  cells.scale_log2 = kLog2e / sqrtf(static_cast<float>(L->head_dim));
  int s = sel::launch_greedy(w.lists, H, n_total, alpha, total, w.picks, w.cap, cells, w.n_final, coverage, approx,
                             st, 0, po);
  if (!s && prefix) {  // heads that left a sorted prefix: full sort + greedy again (no-op launches otherwise)
    const size_t smem = sel::block_sort_smem(n_s);
    LS_CUDA(cudaFuncSetAttribute(sel::sort_block_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    sel::sort_block_kernel<float><<<dim3(2, H), sel::BS_THREADS, smem, st>>>(v_w, v_max, s_w, s_max, rows, n_s,
                                                                           n_total, L->row_offset, fix_bits, w.lists);
    LS_LAUNCH_CHECK("sort_block_kernel");
    s = sel::launch_greedy(w.lists, H, n_total, alpha, total, w.picks, w.cap, cells, w.n_final, coverage, approx, st,
                           1, po);
  }
  if (s) return s;
  if (plan_ready) {  // the plans were written by the greedy CTAs
    if (n_picks) LS_CUDA(cudaMemcpyAsync(n_picks, w.n_final, sizeof(int32_t) * H, cudaMemcpyDeviceToDevice, st));
    return LS_OK;
  }
  return sel::run_tail(w, H, n_total, alpha, total, slash_ids, vert_ids, counts, coverage, approx, picks, n_picks,
                       st);
}

extern "C" int ls_select_lines(const ls_layer_desc *L, int32_t n_s, double alpha, const uint16_t *q,
                               const uint16_t *k, const int32_t *rows, const double *v_w, const float *v_max,
                               const double *s_w, const float *s_max, const float *row_stats, const double *total,
                               int32_t *slash_ids, int32_t *vert_ids, int32_t *counts, double *coverage,
                               double *approx, int32_t *picks, int32_t *n_picks, void *ws, size_t ws_bytes,
                               ls_stream_t stream) {
  return ls_select_lines_ready(L, n_s, alpha, q, k, rows, v_w, v_max, s_w, s_max, row_stats, total, slash_ids,
                               vert_ids, counts, coverage, approx, picks, n_picks, nullptr, 0, ws, ws_bytes, stream);
}

// ------------------------------------------------------- device-value stream wait
typedef CUresult (*StreamWaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

extern "C" int ls_stream_wait_value(ls_stream_t stream, const int32_t *addr, int32_t value) {
  static StreamWaitValue32Fn fn = nullptr;
  if (!fn) {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<StreamWaitValue32Fn>(ptr);
  }
  LS_REQUIRE(fn != nullptr, LS_ERR_CUDA, "cuStreamWaitValue32 unavailable");
  const CUresult r = fn(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(addr),
                        static_cast<cuuint32_t>(value), CU_STREAM_WAIT_VALUE_GEQ);
  LS_REQUIRE(r == CUDA_SUCCESS, LS_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", static_cast<int>(r));
  return LS_OK;
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
      L.inv[static_cast<int64_t>(kind) * n_total + idx[i]] = i;
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
  sel::Work w = sel::carve(c, 1, n_total);
  double *tot = c.take<double>(1);
  LS_REQUIRE(c.ok(), LS_ERR_WORKSPACE, "greedy_dense workspace too small (%zu > %zu)", c.off, ws_bytes);
  LS_CUDA(cudaMemcpyAsync(tot, &total_weight, sizeof(double), cudaMemcpyHostToDevice, st));
  sel::load_lists_kernel<<<8, 256, 0, st>>>(n_slash, s_idx, s_w, s_len, s_max, 0, n_total, w.lists);
  sel::load_lists_kernel<<<8, 256, 0, st>>>(n_vert, v_idx, v_w, v_len, v_max, 1, n_total, w.lists);
  LS_LAUNCH_CHECK("load_lists_kernel");
  sel::DenseCells cells{weights, positions, n_rows, n_total};
  int s = sel::launch_greedy(w.lists, 1, n_total, alpha, tot, w.picks, w.cap, cells, w.n_final, coverage, approx, st);
  if (s) return s;
  return sel::run_tail(w, 1, n_total, alpha, tot, slash_ids, vert_ids, counts, coverage, approx, nullptr, nullptr,
                       st);
}
