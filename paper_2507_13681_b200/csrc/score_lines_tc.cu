// K1 (tensor-core path) -- sampled-row scoring and line sums on tcgen05.
//
// Replaces the scoring part of sparsify_head (reference prefill.py:377-390),
// softmax_rows (tensor_ops.py:24-40) and _line_sums (prefill.py:138-169).
//
// Work grid: (key chunk of CHUNK columns, tile of 128 sampled rows, head).
//   k1_stats   : S = Qs K^T per 128-key tile on tcgen05 (TMEM double-
//                buffered so tile t+1's MMA overlaps tile t's math), online
//                (max, sum) per row and chunk -> partial stats.
//   k1_lines   : combines the chunk stats of its rows in chunk order, then
//                recomputes S, P = exp2(s - m) / l (fp32) into shared memory
//                and reduces it: vertical sums (column, rows in order, fp64)
//                and slash sums (thread owns d = g - c, rows in order, fp64,
//                accumulated over the chunk in shared memory).
// Partials of different CTAs are merged with 64-bit integer atomics on a
// 2^-40 fixed-point scale: integer addition is associative, so the result is
// bit-identical whatever the CTA schedule (the reference's determinism
// contract), and the quantisation (<= 2^-41 per partial) is
// far below the fp32 error of P itself. Maxima use integer atomicMax on the
// (non-negative) float bits.

#include <cuda.h>

#include "ls_common.cuh"
#include "tc_common.cuh"

namespace ls {
extern int *g_debug_buffer;
// bf16 [heads][rows][d] tensor map, box 64 columns x 128 rows, 128-B swizzle (vs_attention_ws.cu)
int make_tmap_bf16_3d(CUtensorMap *m, const void *base, int d, int64_t rows, int heads, int64_t row_stride_el,
                      int64_t head_stride_el);
}

namespace ls {
namespace k1tc {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int CHUNK = 1024;        // key columns per statistics / slash-accumulator chunk
constexpr int LDP = BN + 4;        // fp32 P row stride (16-B rows: conflict-free STS.128 / column LDS)
constexpr int P_PRE = 4;           // zero floats before each P buffer (slash reads reach 2 columns left of row 0)
constexpr int PBUF = P_PRE + BM * LDP;  // floats per P buffer
constexpr int SQ = 3;              // slash diagonals per lane (stride 3: lanes on one row hit distinct banks)
constexpr int ACC_CAP = 3072;      // shared slash accumulator (diagonals per chunk)
constexpr int RP_CAP = 2048;       // row-pointer table: first sampled row at or after a position
constexpr int LINES_THREADS = 512; // 16 warps: 4 per TMEM lane quadrant
constexpr int STATS_THREADS = 256; // two threads per sampled row (column halves)
constexpr double FIX = 1099511627776.0;  // 2^40
constexpr double UNFIX = 1.0 / 1099511627776.0;

// Work decomposition (both passes, persistent CTAs). A row tile ("item") is
// (head h, row tile rt): the n_s sampled rows of a head are split into n_rt =
// ceil(n_s / 128) tiles of near-equal size (rows [rt*n_s/n_rt, (rt+1)*n_s/n_rt)),
// and item i = h*n_rt + rt covers key tiles [0, ceil(c_end_i / 128)), c_end_i =
// the causal end of its last row. The items' key tiles form one flat list
// (prefix table `tstart`, written by k1_tiles_kernel); CTA b of G processes the
// contiguous slice [T*b/G, T*(b+1)/G), so every SM gets the same number of
// 128 x 128 score tiles and a CTA's setup (TMEM, barriers, Q gather) is paid
// once per slice, not once per 1024-key chunk.
struct Params {
  const uint16_t *q;
  const uint16_t *k;
  const int32_t *rows;
  int n_heads, group, n_s, n_total, row_offset, n_rt, n_chunks;
  int64_t q_head_stride, kv_head_stride;
  float scale_log2;
  const int32_t *tstart;            // [H*n_rt + 1] prefix of key tiles per item
  float2 *pstats;                   // [H][n_chunks][n_s][2 slots][2 halves] (max, sum) per row
  unsigned long long *vfix, *sfix;  // [H][n_total]
  unsigned int *vmaxb, *smaxb;      // [H][n_total]
  float *row_stats;                 // [H][n_s][2]
  int32_t *status;                  // device validation word (NonFiniteInput / AllMaskedRow)
  int *dbg;                         // optional host-mapped phase clocks (ls_debug_set_buffer)
};

__device__ __forceinline__ int rt_begin(const Params &p, int rt) {
  return static_cast<int>((static_cast<long long>(rt) * p.n_s) / p.n_rt);
}

// key tiles of every item and their exclusive prefix (one CTA)
__global__ void __launch_bounds__(1024) k1_tiles_kernel(Params p, int32_t *tstart) {
  __shared__ int sh[32];
  const int n_items = p.n_heads * p.n_rt;
  int base = 0;
  for (int i0 = 0; i0 < n_items; i0 += blockDim.x) {
    const int i = i0 + threadIdx.x;
    int nt = 0;
    if (i < n_items) {
      const int h = i / p.n_rt, rt = i - h * p.n_rt;
      const int r_last = rt_begin(p, rt + 1) - 1;
      const int g_last = p.row_offset + p.rows[static_cast<int64_t>(h) * p.n_s + r_last];
      const int c_end = min(p.n_total, g_last + 1);
      nt = (c_end + BN - 1) / BN;
    }
    // block exclusive scan
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = nt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    __syncthreads();
    if (lane == 31) sh[wid] = incl;
    __syncthreads();
    int before = 0, all = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
      if (w < wid) before += sh[w];
      all += sh[w];
    }
    if (i < n_items) tstart[i] = base + before + incl - nt;
    base += all;
  }
  if (threadIdx.x == 0) tstart[n_items] = base;
}

// Position in the flat tile list: item i, tile j of the item (columns [j*BN, +BN)).
struct TileCursor {
  int x, i, j, i_end_tile;  // global tile, item, local tile, first global tile of item i + 1
  __device__ void seek(const int32_t *tstart, int n_items, int x_) {
    x = x_;
    int lo = 0, hi = n_items - 1;  // last item with tstart <= x
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (tstart[mid] <= x) lo = mid; else hi = mid - 1;
    }
    i = lo;
    while (tstart[i + 1] <= x) ++i;  // skip empty items
    j = x - tstart[i];
    i_end_tile = tstart[i + 1];
  }
  __device__ void next(const int32_t *tstart) {
    ++x;
    ++j;
    while (x >= i_end_tile) {  // next non-empty item
      ++i;
      j = x - tstart[i];
      i_end_tile = tstart[i + 1];
    }
  }
};

// first tile at or after global tile x that starts a 1024-key chunk of its item
__device__ __forceinline__ int chunk_start_at_or_after(const int32_t *tstart, int n_items, int x, int T) {
  if (x >= T) return T;
  TileCursor c;
  c.seek(tstart, n_items, x);
  const int r = c.j % (CHUNK / BN);
  if (r == 0) return x;
  return min(x + (CHUNK / BN - r), c.i_end_tile);  // (the next item starts a chunk)
}

// this CTA's slice [x0, x1) of the flat tile list: balanced by tile count, with
// both ends moved to chunk starts, so every 1024-key chunk is processed whole by
// one CTA in tile order -- the results do not depend on the grid size or on
// how many heads share the launch (head-sharded runs equal the unsharded one)
__device__ __forceinline__ bool tile_slice(const Params &p, int &x0, int &x1) {
  const int n_items = p.n_heads * p.n_rt;
  const int T = p.tstart[n_items];
  const int G = gridDim.x;
  x0 = chunk_start_at_or_after(p.tstart, n_items, static_cast<int>((static_cast<long long>(T) * blockIdx.x) / G), T);
  x1 = chunk_start_at_or_after(p.tstart, n_items,
                               static_cast<int>((static_cast<long long>(T) * (blockIdx.x + 1)) / G), T);
  return x0 < x1;
}

template <int D>
struct StatsSmem {
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = BM * D * 2;
  static constexpr int OFF_MISC = OFF_K + 2 * BN * D * 2;
  static constexpr int TOTAL = OFF_MISC + 1024 + 1024;  // barriers, TMEM address, row positions
};

template <int D>
struct LinesSmem {  // (Qs lives in TMEM)
  static constexpr int OFF_K = 0;                                // one K stage
  static constexpr int OFF_P = OFF_K + BN * D * 2;              // two fp32 P buffers [BM][LDP]
  static constexpr int OFF_ACC = OFF_P + 2 * PBUF * 4;          // double[ACC_CAP]
  static constexpr int OFF_ACCM = OFF_ACC + ACC_CAP * 8;        // float[ACC_CAP]
  static constexpr int OFF_RP = OFF_ACCM + ACC_CAP * 4;         // int[RP_CAP] row pointer by position
  static constexpr int OFF_MISC = OFF_RP + RP_CAP * 4;          // barriers | TMEM address | counters | gs | m | 1/l | row bases
  static constexpr int TOTAL = OFF_MISC + 2560;
};

__device__ __forceinline__ void zfill16(uint32_t saddr, const void *g, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(ok ? 16 : 0) : "memory");
}

__device__ __forceinline__ unsigned long long to_fix(double x) {
  return static_cast<unsigned long long>(__double2ll_rn(x * FIX));
}

// gather the Q rows of item (h, rt) into the swizzled Q tile (cp.async, all
// threads) and their positions into gs[]; returns the item's row count
template <int D>
__device__ __forceinline__ int load_item_q(const Params &p, unsigned char *smem, int *gs, int h, int rt) {
  const int r0 = rt_begin(p, rt), nr = rt_begin(p, rt + 1) - r0;
  const int32_t *rows_h = p.rows + static_cast<int64_t>(h) * p.n_s + r0;
  constexpr int CH = D / 8;
  const uint32_t qs = tc::smem_u32(smem);
  for (int idx = threadIdx.x; idx < BM * CH; idx += blockDim.x) {
    const int r = idx / CH, ch = idx - r * CH;
    const bool ok = r < nr;
    const int lr = ok ? rows_h[r] : 0;
    if (ch == 0) gs[r] = ok ? p.row_offset + lr : 0x7fffffff;
    const uint16_t *qrow = p.q + static_cast<int64_t>(h) * p.q_head_stride + static_cast<int64_t>(lr) * D;
    zfill16(qs + tc::sw128_offset(r, ch, BM), qrow + ch * 8, ok);
  }
  tc::cp_async_commit();
  return nr;
}

// the item's sampled positions into gs[] and its Q rows into TMEM (lane = row,
// 32-bit columns = bf16 pairs: the A operand of S = Qs K^T), zeros past nr;
// warp w writes lanes of quadrant w % 4, columns [16 (w / 4), +16)
template <int D>
__device__ __forceinline__ int load_item_q_tmem(const Params &p, int *gs, uint32_t tmem_q, int h, int rt) {
  const int r0 = rt_begin(p, rt), nr = rt_begin(p, rt + 1) - r0;
  const int32_t *rows_h = p.rows + static_cast<int64_t>(h) * p.n_s + r0;
  for (int r = threadIdx.x; r < BM; r += blockDim.x) gs[r] = r < nr ? p.row_offset + rows_h[r] : 0x7fffffff;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = (warp & 3) * 32 + lane, cb = (warp >> 2) * 16;
  if (cb < D / 2) {
    uint32_t v[16];
    if (row < nr) {
      const uint4 *src = reinterpret_cast<const uint4 *>(p.q + static_cast<int64_t>(h) * p.q_head_stride +
                                                         static_cast<int64_t>(rows_h[row]) * D + cb * 2);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint4 x = __ldg(src + u);
        v[4 * u] = x.x;
        v[4 * u + 1] = x.y;
        v[4 * u + 2] = x.z;
        v[4 * u + 3] = x.w;
      }
    } else {
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = 0u;
    }
    tc::tmem_st16(tmem_q + (static_cast<uint32_t>((warp & 3) * 32) << 16) + cb, v);
  }
  tc::tmem_wait_st();
  return nr;
}

// S(buf) = Qs K^T with Qs from TMEM (no shared-memory operand traffic for A:
// the lines pass keeps shared memory busy with its reductions)
template <int D>
__device__ __forceinline__ void issue_s_tq(unsigned char *smem, int off_k, uint32_t tmem, uint32_t tmem_q, int buf,
                                           uint64_t *mbar) {
  constexpr uint32_t IDESC = tc::make_idesc(BM, BN, false, false);
  const uint32_t ks = tc::smem_u32(smem + off_k);  // (one K stage)
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) {
    const uint64_t bd = tc::make_desc(ks + (kk >> 2) * (BN * 128) + (kk & 3) * 32, 16, 1024);
    tc::mma_bf16_ts(tmem + buf * 128, tmem_q + kk * 8, bd, IDESC, kk > 0);
  }
  tc::mma_commit(&mbar[buf]);
}

// K rows [c0, c0 + 128) of kv head `kv` by TMA (rows past n_total read as zero)
template <int D>
__device__ __forceinline__ void tma_k(const CUtensorMap *tm, unsigned char *smem, int off_k, int buf, uint64_t *full,
                                      int c0, int kv) {
  tc::mbar_expect_tx(full, BN * D * 2);
  const uint32_t ks = tc::smem_u32(smem + off_k + buf * BN * D * 2);
#pragma unroll
  for (int a = 0; a < D / 64; ++a) tc::tma_load_3d(ks + a * BN * 128, tm, full, a * 64, c0, kv);
}

template <int D>
__device__ __forceinline__ void issue_s(unsigned char *smem, int off_k, uint32_t tmem, int buf, uint64_t *mbar) {
  constexpr uint32_t IDESC = tc::make_idesc(BM, BN, false, false);
  const uint32_t qs = tc::smem_u32(smem);
  const uint32_t ks = tc::smem_u32(smem + off_k + buf * BN * D * 2);
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) {
    const uint64_t ad = tc::make_desc(qs + (kk >> 2) * (BM * 128) + (kk & 3) * 32, 16, 1024);
    const uint64_t bd = tc::make_desc(ks + (kk >> 2) * (BN * 128) + (kk & 3) * 32, 16, 1024);
    tc::mma_bf16(tmem + buf * 128, ad, bd, IDESC, kk > 0);
  }
  tc::mma_commit(&mbar[buf]);
}

// cp.async-written Q visible to the tensor core, every thread past the barrier
__device__ __forceinline__ void q_ready_sync() {
  tc::cp_async_wait<0>();
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
}

// Shared pipeline of both passes over the CTA's tile slice [x0, x1):
//   thread 0 keeps the TMA of K two tiles ahead (stage t & 1) and issues
//   S(t + 1) = Q K(t+1)^T into TMEM buffer (t + 1) & 1 before the CTA works on
//   S(t); a TMEM buffer is reused once every thread has read it (the caller's
//   s_empty arrivals or barrier). At an item boundary S(t + 1) needs the next
//   item's Q: it is issued by on_item_switch() after the gather.
struct Pipe {
  uint64_t *s_full;   // [2] MMA -> threads
  uint64_t *k_full;   // [2] TMA -> MMA
  uint64_t *s_empty;  // [2] threads -> MMA (stats pass)
  uint32_t tmem;
};

// ------------------------------------------------------------- pass 1
// 256 threads, two per sampled row (TMEM lane = row, warps 0-3 columns 0-63,
// warps 4-7 columns 64-127), each with its own online (max, sum) over its
// half of every tile of a 1024-key chunk, written per (chunk, row, half) --
// the consumer merges them in a fixed order, so no CTA barrier per tile.
template <int D>
__global__ void __launch_bounds__(STATS_THREADS, 2) k1_stats_kernel(const __grid_constant__ CUtensorMap tm_k, Params p) {
  extern __shared__ unsigned char smem_dyn[];
  using L = StatsSmem<D>;
  unsigned char *smem = tc::align1024(smem_dyn);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L::OFF_MISC);  // s_full[2] k_full[2] s_empty[2]
  uint32_t *tmem_sh = reinterpret_cast<uint32_t *>(smem + L::OFF_MISC + 64);
  int *gs = reinterpret_cast<int *>(smem + L::OFF_MISC + 1024);
  const int n_items = p.n_heads * p.n_rt;
  int x0, x1;
  if (!tile_slice(p, x0, x1)) return;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int row = tid & (BM - 1), hc = tid >> 7;  // column half
  Pipe pp{bars, bars + 2, bars + 4, 0};
  TileCursor cur, pre;  // consumer and TMA producer
  cur.seek(p.tstart, n_items, x0);
  if (warp == 0) tc::tmem_alloc(tmem_sh, 256);
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&pp.s_full[b], 1);
      tc::mbar_init(&pp.k_full[b], 1);
      tc::mbar_init(&pp.s_empty[b], STATS_THREADS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tc::prefetch_tmap(&tm_k);
    pre = cur;
    for (int t = 0; t < 2 && x0 + t < x1; ++t) {
      tma_k<D>(&tm_k, smem, L::OFF_K, t, &pp.k_full[t], pre.j * BN, (pre.i / p.n_rt) / p.group);
      if (x0 + t + 1 < x1) pre.next(p.tstart);
    }
  }
  int h = cur.i / p.n_rt, rt = cur.i - h * p.n_rt;
  int nr = load_item_q<D>(p, smem, gs, h, rt);
  q_ready_sync();
  pp.tmem = *tmem_sh;
  if (tid == 0) {
    tc::mbar_wait(&pp.k_full[0], 0);
    issue_s<D>(smem, L::OFF_K, pp.tmem, 0, pp.s_full);
  }
  int my_g = gs[row], r0 = rt_begin(p, rt);
  bool row_ok = row < nr;
  int c_end = min(p.n_total, gs[nr - 1] + 1);
  const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
  float m = -INFINITY, l = 0.f;
  int seg_slot = (cur.j * BN) % CHUNK != 0 ? 1 : 0;
  for (int x = x0; x < x1; ++x) {
    const int t = x - x0, buf = t & 1;
    const int c0 = cur.j * BN;
    const bool last_in_item = x + 1 >= cur.i_end_tile;
    const bool more = x + 1 < x1;
    if (tid == 0 && more && !last_in_item) {  // S(t+1): its TMEM buffer was read by every thread at t-1
      tc::mbar_wait(&pp.k_full[buf ^ 1], ((t + 1) >> 1) & 1);
      if (t >= 1) tc::mbar_wait(&pp.s_empty[buf ^ 1], ((t - 1) >> 1) & 1);
      tc::fence_after_sync();
      issue_s<D>(smem, L::OFF_K, pp.tmem, buf ^ 1, pp.s_full);
    }
    tc::mbar_wait(&pp.s_full[buf], (t >> 1) & 1);
    tc::fence_after_sync();
    if (tid == 0 && x + 2 < x1) {  // S(t) is done with K stage `buf`
      tma_k<D>(&tm_k, smem, L::OFF_K, buf, &pp.k_full[buf], pre.j * BN, (pre.i / p.n_rt) / p.group);
      if (x + 3 < x1) pre.next(p.tstart);
    }
    const int lim = min(my_g, c_end - 1) - c0 - 64 * hc;  // last valid column of this thread's 64
    float sv[64];
    tc::tmem_ld32(pp.tmem + buf * 128 + lane_base + 64 * hc, sv);
    tc::tmem_ld32(pp.tmem + buf * 128 + lane_base + 64 * hc + 32, sv + 32);
    tc::tmem_wait_ld();
    tc::fence_before_sync();
    tc::mbar_arrive(&pp.s_empty[buf]);
    if (row_ok && lim >= 63) {  // whole half-tile causal: no masking
      float t4[4] = {sv[0], sv[1], sv[2], sv[3]};
#pragma unroll
      for (int j = 4; j < 64; j += 4) {
        t4[0] = fmaxf(t4[0], sv[j]);
        t4[1] = fmaxf(t4[1], sv[j + 1]);
        t4[2] = fmaxf(t4[2], sv[j + 2]);
        t4[3] = fmaxf(t4[3], sv[j + 3]);
      }
      const float tm = fmaxf(fmaxf(t4[0], t4[1]), fmaxf(t4[2], t4[3]));
      const float mn = fmaxf(m, tm * p.scale_log2);
      float a4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int j = 0; j < 64; ++j) a4[j & 3] += fast_exp2(fmaf(sv[j], p.scale_log2, -mn));
      l = (m == -INFINITY ? 0.f : l * fast_exp2(m - mn)) + ((a4[0] + a4[1]) + (a4[2] + a4[3]));
      m = mn;
    } else if (row_ok && lim >= 0) {
      float tm = -INFINITY;
#pragma unroll
      for (int j = 0; j < 64; ++j)
        if (j <= lim) tm = fmaxf(tm, sv[j]);
      const float mn = fmaxf(m, tm * p.scale_log2);
      float acc = 0.f;
#pragma unroll
      for (int j = 0; j < 64; ++j)
        if (j <= lim) acc += fast_exp2(fmaf(sv[j], p.scale_log2, -mn));
      l = (m == -INFINITY ? 0.f : l * fast_exp2(m - mn)) + acc;
      m = mn;
    }
    if (last_in_item || ((c0 + BN) % CHUNK) == 0 || !more) {  // segment of a chunk done
      // slot 0: the segment starting at the chunk's first tile; slot 1: the one a
      // CTA slice starts with in mid-chunk (slices hold >= CHUNK / BN tiles, so a
      // chunk has at most these two)
      if (row_ok) {
        const int ck = c0 / CHUNK;
        p.pstats[(((static_cast<int64_t>(h) * p.n_chunks + ck) * p.n_s + r0 + row) * 2 + seg_slot) * 2 + hc] =
            make_float2(m, l);
      }
      m = -INFINITY;
      l = 0.f;
      seg_slot = 0;
    }
    if (more) {
      cur.next(p.tstart);
      if (last_in_item) {  // next item: S(t) is complete and nothing else is in flight
        h = cur.i / p.n_rt;
        rt = cur.i - h * p.n_rt;
        __syncthreads();  // every thread is done with gs / the TMEM reads of this item
        nr = load_item_q<D>(p, smem, gs, h, rt);
        q_ready_sync();
        my_g = gs[row];
        r0 = rt_begin(p, rt);
        row_ok = row < nr;
        c_end = min(p.n_total, gs[nr - 1] + 1);
        if (tid == 0) {
          tc::mbar_wait(&pp.k_full[buf ^ 1], ((t + 1) >> 1) & 1);
          issue_s<D>(smem, L::OFF_K, pp.tmem, buf ^ 1, pp.s_full);
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(pp.tmem, 256);
}

// ------------------------------------------------------------- pass 2
// 16 compute warps + 1 producer warp, software-pipelined over two P buffers:
// iteration t computes P(t + 1) = exp2(s - m) / l (fp32) from TMEM into
// buffer (t + 1) & 1 (warp w: TMEM lanes of quadrant w % 4, 32 columns of
// block w / 4) and then reduces P(t) from buffer t & 1, so the MUFU-bound
// exponentials of one tile overlap the shared-memory-bound reductions of the
// previous one across warps; one named barrier per tile. Reductions are warp
// tasks handed out by a shared counter: vertical (32 columns x 128 rows; lane
// = 32-row quarter x 4 columns, one 16-B load per row, fp32 partials of 8 rows
// combined in fp64, quarters added in order through shuffles, straight to the
// column's integer atomics) and slash (lane owns SQ = 3 consecutive diagonals
// and walks the rows of their union in ascending order through a row-base
// table, zero pads covering cells outside a diagonal; per-tile fp32 sums
// accumulated per 1024-key chunk in fp64 shared memory and flushed at the
// chunk's end). The producer warp keeps the K TMA (one stage: a second one does
// not fit beside two P buffers) and the S = Qs K^T MMAs (Qs in TMEM as the A
// operand, S double-buffered in TMEM) ahead of the compute warps.
template <int D>
__global__ void __launch_bounds__(LINES_THREADS + 32, 1) k1_lines_kernel(const __grid_constant__ CUtensorMap tm_k, Params p) {
  extern __shared__ unsigned char smem_dyn[];
  using L = LinesSmem<D>;
  unsigned char *smem = tc::align1024(smem_dyn);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L::OFF_MISC);
  uint64_t *s_full = bars, *s_free = bars + 2, *k_full = bars + 4, *q_full = bars + 5;
  uint32_t *tmem_sh = reinterpret_cast<uint32_t *>(smem + L::OFF_MISC + 48);
  int *task_ctr = reinterpret_cast<int *>(smem + L::OFF_MISC + 56);             // [2]
  int *gs = reinterpret_cast<int *>(smem + L::OFF_MISC + 64);                    // [BM + 4]
  float *m_sh = reinterpret_cast<float *>(smem + L::OFF_MISC + 64 + 528);       // [BM]
  float *li_sh = m_sh + BM;                                                      // [BM]
  int *rbase = reinterpret_cast<int *>(li_sh + BM);                              // [BM] r * LDP + g_r
  float *Pb0 = reinterpret_cast<float *>(smem + L::OFF_P) + P_PRE;  // P(t) at Pb0 + (t & 1) * PBUF, rows at stride LDP
  double *acc = reinterpret_cast<double *>(smem + L::OFF_ACC);
  float *accm = reinterpret_cast<float *>(smem + L::OFF_ACCM);
  int *rp = reinterpret_cast<int *>(smem + L::OFF_RP);
  const int n_items = p.n_heads * p.n_rt;
  int x0, x1;
  if (!tile_slice(p, x0, x1)) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_tiles = x1 - x0;
  if (warp == 0) tc::tmem_alloc(tmem_sh, 512);  // S double buffer [0, 256), Qs [256, 256 + D / 2)
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&s_full[b], 1);
      tc::mbar_init(&s_free[b], LINES_THREADS / 32);
    }
    tc::mbar_init(k_full, 1);
    tc::mbar_init(q_full, LINES_THREADS / 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tc::prefetch_tmap(&tm_k);
    task_ctr[0] = task_ctr[1] = 0;
  }
  for (int i = tid; i < ACC_CAP; i += blockDim.x) {  // invariant: zero outside a chunk's use (the flush re-zeroes)
    acc[i] = 0.0;
    accm[i] = 0.f;
  }
  // zero pads of both P buffers: columns [BN, LDP) of every row and the P_PRE floats before row 0
  for (int i = tid; i < 2 * (BM * 4 + P_PRE); i += blockDim.x) {
    const int b = i / (BM * 4 + P_PRE), k = i - b * (BM * 4 + P_PRE);
    float *base = Pb0 + b * PBUF;
    if (k < BM * 4) base[(k >> 2) * LDP + BN + (k & 3)] = 0.f;
    else base[k - BM * 4 - P_PRE] = 0.f;
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_sh, tmem_q = tmem + 256;

  if (warp == LINES_THREADS / 32) {  // ---------------- producer warp
    if (lane == 0) {
      TileCursor pre;
      pre.seek(p.tstart, n_items, x0);
      int item = -1, n_q = 0;
      tma_k<D>(&tm_k, smem, L::OFF_K, 0, k_full, pre.j * BN, (pre.i / p.n_rt) / p.group);
      for (int t = 0; t < n_tiles; ++t) {
        if (pre.i != item) {  // the item's Qs written to TMEM by the compute warps
          item = pre.i;
          tc::mbar_wait(q_full, n_q & 1);
          ++n_q;
        }
        if (t >= 2) tc::mbar_wait(&s_free[t & 1], ((t - 2) >> 1) & 1);  // P(t - 2) read S buffer t & 1
        tc::mbar_wait(k_full, t & 1);
        tc::fence_after_sync();
        issue_s_tq<D>(smem, L::OFF_K, tmem, tmem_q, t & 1, s_full);
        if (t + 1 < n_tiles) {
          tc::mbar_wait(&s_full[t & 1], (t >> 1) & 1);  // S(t) has read the K stage
          pre.next(p.tstart);
          tma_k<D>(&tm_k, smem, L::OFF_K, 0, k_full, pre.j * BN, (pre.i / p.n_rt) / p.group);
        }
      }
    }
    __syncwarp();
  } else {  // ---------------------------------------- 16 compute warps
    const int row = (warp & 3) * 32 + lane;
    const int cblk = (warp >> 2) * 32;
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    TileCursor cur;
    cur.seek(p.tstart, n_items, x0);
    unsigned long long *sfix = nullptr;
    unsigned int *smaxb = nullptr;
    int h = 0, rt = 0, nr = 0, my_g = 0, g_first = 0, g_hi = 0, c_end = 0;
    float mr = INFINITY;
    bool row_ok = false, use_rp = false;
    int d_base = 0, width = 0;
    bool smem_acc = false;
    // diagnostics: per-tile phase clocks of CTA 0, threads 0 / 32 / 256, tiles < 64
    int *rec = nullptr;
    if (p.dbg && blockIdx.x == 0 && (tid == 0 || tid == 32 || tid == 256))
      rec = p.dbg + 40000 + (tid == 0 ? 0 : tid == 32 ? 1 : 2) * 64 * 12;
#define K1REC(tt, k) do { if (rec && (tt) < 64) rec[(tt) * 12 + (k)] = static_cast<int>(clock64()); } while (0)
    // per item: positions, Qs into TMEM (-> producer), the rows' statistics
    // (all chunks, fixed order), position -> row table
    auto begin_item = [&]() {
      h = cur.i / p.n_rt;
      rt = cur.i - h * p.n_rt;
      nr = load_item_q_tmem<D>(p, gs, tmem_q, h, rt);
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(q_full);
      if (tid < 4) gs[BM + tid] = 0x7fffffff;
      const int r0 = rt_begin(p, rt);
      tc::named_sync(1, LINES_THREADS);  // gs visible
      if (tid < BM) {
        float m = -INFINITY, l = 0.f;
        if (tid < nr) {
          const int n_ck = min(gs[tid], p.n_total - 1) / CHUNK + 1;  // chunks of this row's causal range
          const float2 *ps = p.pstats + (static_cast<int64_t>(h) * p.n_chunks * p.n_s + r0 + tid) * 4;
          for (int c = 0; c < n_ck; ++c) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {  // (slot, half) in a fixed order
              const float2 v = ps[static_cast<int64_t>(c) * p.n_s * 4 + e];
              if (v.y == 0.f) continue;  // empty (zeroed) or no causal column
              const float mn = fmaxf(m, v.x);
              l = (m == -INFINITY ? 0.f : l * fast_exp2(m - mn)) + v.y * fast_exp2(v.x - mn);
              m = mn;
            }
          }
          if (cur.j == 0) {  // the CTA holding the item's first tile publishes the row statistics
            float *rs = p.row_stats + (static_cast<int64_t>(h) * p.n_s + r0 + tid) * 2;
            rs[0] = m;
            rs[1] = l > 0.f ? 1.f / l : 0.f;
            // softmax_rows' validation (tensor_ops.py:34-38): a NaN / +inf logit
            // (NaN row max or sum), or a row whose every logit is -inf
            if (isnan(m) || isnan(l) || isinf(l) || (isinf(m) && m > 0.f)) report_status(p.status, LS_ERR_NON_FINITE_INPUT);
            else if (m == -INFINITY) report_status(p.status, LS_ERR_ALL_MASKED_ROW);
          }
        }
        m_sh[tid] = m;
        li_sh[tid] = l > 0.f ? 1.f / l : 0.f;
      }
      if (tid < BM) rbase[tid] = tid * LDP + gs[tid];
      g_first = gs[0];
      g_hi = gs[nr - 1];
      c_end = min(p.n_total, g_hi + 1);
      const int rp_span = g_hi - g_first + 1;
      use_rp = rp_span <= RP_CAP;
      if (use_rp)
        for (int xx = tid; xx < rp_span; xx += LINES_THREADS) rp[xx] = lower_bound_dev(gs, nr, g_first + xx);
      sfix = p.sfix + static_cast<int64_t>(h) * p.n_total;
      smaxb = p.smaxb + static_cast<int64_t>(h) * p.n_total;
      tc::named_sync(1, LINES_THREADS);  // statistics / table visible
      my_g = gs[row];
      row_ok = row < nr;
      mr = li_sh[row] > 0.f ? m_sh[row] - __log2f(li_sh[row]) : INFINITY;
    };
    // slash accumulator window of the chunk holding column c0: d in [d_base, d_base + width)
    auto begin_chunk = [&](int c0) {
      const int cb = (c0 / CHUNK) * CHUNK;
      const int ce = min(cb + CHUNK, c_end);
      d_base = max(0, g_first - (ce - 1));
      width = g_hi - cb - d_base + 1;
      smem_acc = width <= ACC_CAP;
    };
    // P(t) of key tile c0 into buffer t & 1; releases S buffer t & 1 to the producer
    auto exp_tile = [&](int t, int c0) {
      tc::mbar_wait(&s_full[t & 1], (t >> 1) & 1);
      tc::fence_after_sync();
      const int lim = min(my_g, c_end - 1) - c0 - cblk;  // last valid column of this thread's 32
      float sv[32];
      tc::tmem_ld32(tmem + (t & 1) * 128 + lane_base + cblk, sv);
      tc::tmem_wait_ld();
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&s_free[t & 1]);
      float4 *prow = reinterpret_cast<float4 *>(Pb0 + (t & 1) * PBUF + row * LDP + cblk);
      if (row_ok && lim >= 31) {
        // every eighth exponential on the FMA pipe (poly6_exp2, fp32 accuracy): the
        // MUFU ex2, the P stores and the TMEM loads share the MIO queue, the phase's
        // top stall (C2 turn 3: 0.427 -> 0.414 ms/layer, C5 turn 10: 1.341 -> 1.318 ms,
        // identical plans; a quarter 0.419 / 1.341, three eighths 0.427 / 1.359, half 0.449)
#define K1E(u) fast_exp2(fmaf(sv[u], p.scale_log2, -mr))
#define K1F(u) poly6_exp2(fmaf(sv[u], p.scale_log2, -mr))
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          prow[j / 4] = (j & 4) ? make_float4(K1E(j), K1E(j + 1), K1E(j + 2), K1F(j + 3))
                                : make_float4(K1E(j), K1E(j + 1), K1E(j + 2), K1E(j + 3));
#undef K1E
#undef K1F
      } else {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float e[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            e[u] = (row_ok && j + u <= lim) ? fast_exp2(fmaf(sv[j + u], p.scale_log2, -mr)) : 0.f;
          prow[j / 4] = make_float4(e[0], e[1], e[2], e[3]);
        }
      }
    };
    // reductions of P(t) (key tile c0), warp tasks: [0, 4) vertical, [4, 4 + n_sl) slash
    auto reduce_tile = [&](int t, int c0) {
      const float *Pf = Pb0 + (t & 1) * PBUF;
      const int d_lo = max(d_base, g_first - (c0 + BN - 1));
      const int d_hi = g_hi - c0;
      const int n_sl = d_hi >= d_lo ? (d_hi - d_lo) / (32 * SQ) + 1 : 0;
      int *ctr = task_ctr + (t & 1);
      if (tid == 0) task_ctr[(t & 1) ^ 1] = 0;  // the next tile's counter (last used before this tile's barrier)
      for (;;) {
        int task = 0;
        if (lane == 0) task = atomicAdd(ctr, 1);
        task = __shfl_sync(0xffffffffu, task, 0);
        if (task >= 4 + n_sl) break;
        if (task < 4) {
          // vertical, 32 columns: lane = (32-row quarter qq, 4 consecutive
          // columns), one 16-B load per row (rows past nr hold zeros); per
          // column and quarter four fp32 partials of 8 rows, combined in fp64,
          // quarters added in order through shuffles
          const int qq = lane >> 3, j = task * 32 + (lane & 7) * 4;
          const float *pc = Pf + qq * 32 * LDP + j;
          float s4[4][4], m4[4][4];
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int u = 0; u < 4; ++u) s4[c][u] = m4[c][u] = 0.f;
#pragma unroll
          for (int r = 0; r < 32; ++r) {
            const float4 v = *reinterpret_cast<const float4 *>(pc + r * LDP);
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              s4[c][r & 3] += vv[c];
              m4[c][r & 3] = fmaxf(m4[c][r & 3], vv[c]);
            }
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double sw = (static_cast<double>(s4[c][0]) + static_cast<double>(s4[c][1])) +
                        (static_cast<double>(s4[c][2]) + static_cast<double>(s4[c][3]));
            float mx = fmaxf(fmaxf(m4[c][0], m4[c][1]), fmaxf(m4[c][2], m4[c][3]));
            const double q1 = __shfl_down_sync(0xffffffffu, sw, 8), q2 = __shfl_down_sync(0xffffffffu, sw, 16),
                         q3 = __shfl_down_sync(0xffffffffu, sw, 24);
            mx = fmaxf(mx, __shfl_down_sync(0xffffffffu, mx, 8));
            mx = fmaxf(mx, __shfl_down_sync(0xffffffffu, mx, 16));
            if (qq == 0) {
              sw = ((sw + q1) + q2) + q3;
              const int col = c0 + j + c;
              if (col < c_end) {
                if (sw > 0.0) atomicAdd(p.vfix + static_cast<int64_t>(h) * p.n_total + col, to_fix(sw));
                if (mx > 0.f) atomicMax(p.vmaxb + static_cast<int64_t>(h) * p.n_total + col, __float_as_uint(mx));
              }
            }
          }
        } else {
          // slash: lane owns SQ consecutive diagonals dq .. dq + SQ - 1 and walks
          // the rows of their union in ascending order (one row-base load per row
          // for SQ cells; a cell outside a diagonal's own rows reads a zero pad,
          // so each diagonal's fp32 sum is the same as summing its own rows alone)
          const int dq = d_lo + 32 * SQ * (task - 4) + SQ * lane;
          float sw[SQ], mx[SQ];
#pragma unroll
          for (int k = 0; k < SQ; ++k) sw[k] = mx[k] = 0.f;
          if (dq <= d_hi) {
            const int glo = c0 + dq, ghi = min(c0 + dq + SQ - 1 + BN - 1, g_hi);
            int r, r_end;
            if (use_rp) {
              r = rp[max(glo, g_first) - g_first];
              r_end = ghi + 1 <= g_hi ? rp[ghi + 1 - g_first] : nr;
            } else {
              r = lower_bound_dev(gs, nr, glo);
              r_end = lower_bound_dev(gs, nr, ghi + 1);
            }
            const float *pcol = Pf - dq - c0;  // cell (r, g_r - dq - k) at pcol[rbase[r] - k]
#pragma unroll 2
            for (; r < r_end; ++r) {
              const float *pp = pcol + rbase[r];
#pragma unroll
              for (int k = 0; k < SQ; ++k) {
                const float v = pp[-k];
                sw[k] += v;
                mx[k] = fmaxf(mx[k], v);
              }
            }
          }
#pragma unroll
          for (int k = 0; k < SQ; ++k) {
            const int dd = dq + k;
            if (dd > d_hi) break;
            if (smem_acc) {
              acc[dd - d_base] += static_cast<double>(sw[k]);
              accm[dd - d_base] = fmaxf(accm[dd - d_base], mx[k]);
            } else if (sw[k] > 0.f) {
              atomicAdd(sfix + dd, to_fix(static_cast<double>(sw[k])));
              atomicMax(smaxb + dd, __float_as_uint(mx[k]));
            }
          }
        }
      }
    };
    auto flush_chunk = [&]() {
      if (smem_acc)
        for (int i = tid; i < width; i += LINES_THREADS) {
          if (acc[i] > 0.0) atomicAdd(sfix + d_base + i, to_fix(acc[i]));
          if (accm[i] > 0.f) atomicMax(smaxb + d_base + i, __float_as_uint(accm[i]));
          acc[i] = 0.0;
          accm[i] = 0.f;
        }
    };

    begin_item();
    begin_chunk(cur.j * BN);
    exp_tile(0, cur.j * BN);
    tc::named_sync(1, LINES_THREADS);
    for (int t = 0; t < n_tiles; ++t) {
      K1REC(t, 0);
      const int c0 = cur.j * BN;
      const bool last_in_item = x0 + t + 1 >= cur.i_end_tile;
      const bool more = t + 1 < n_tiles;
      const bool chunk_end = last_in_item || ((c0 + BN) % CHUNK) == 0 || !more;
      if (more && !last_in_item) exp_tile(t + 1, c0 + BN);  // P(t + 1) while others reduce P(t)
      K1REC(t, 1);
      reduce_tile(t, c0);
      K1REC(t, 2);
      tc::named_sync(1, LINES_THREADS);  // P(t) reduced, P(t + 1) written
      K1REC(t, 3);
      if (chunk_end) {
        flush_chunk();
        tc::named_sync(1, LINES_THREADS);  // accumulator re-zeroed before the next chunk's tile
      }
      if (more) {
        cur.next(p.tstart);
        if (last_in_item) {
          begin_item();
          begin_chunk(cur.j * BN);
          exp_tile(t + 1, cur.j * BN);
          tc::named_sync(1, LINES_THREADS);
        } else if (chunk_end) {
          begin_chunk(cur.j * BN);
        }
      }
      K1REC(t, 4);
    }
#undef K1REC
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

// fixed point -> fp64 line weights; total = exact integer sum of the verticals.
// Grid (column chunk, head): every CTA converts its chunk and adds its integer
// partial sums to the head's accumulators (integer addition: order-free, so
// the result is bit-identical whatever the schedule); the head's last CTA
// (ticket) writes total and the op count and re-arms the accumulators.
constexpr int FIN_THREADS = 256;
constexpr int FIN_CHUNK = 2048;
__global__ void __launch_bounds__(FIN_THREADS) k1_finish_kernel(const unsigned long long *vfix, const unsigned int *vmaxb,
                                 const unsigned long long *sfix, const unsigned int *smaxb, const int32_t *rows,
                                 int n_s, int n_total, int row_offset, double *v_w, float *v_max, double *s_w,
                                 float *s_max, double *total, int64_t *score_count, unsigned long long *acc_tot,
                                 unsigned long long *acc_cnt, unsigned int *ticket) {
  __shared__ unsigned long long red[FIN_THREADS / 32];
  __shared__ long long redc[FIN_THREADS / 32];
  __shared__ int last;
  const int ck = blockIdx.x, h = blockIdx.y;
  const int c0 = ck * FIN_CHUNK, c1 = min(n_total, c0 + FIN_CHUNK);
  unsigned long long sum = 0;
  long long cnt = 0;
  for (int i = c0 + threadIdx.x; i < c1; i += FIN_THREADS) {
    const int64_t o = static_cast<int64_t>(h) * n_total + i;
    const unsigned long long vf = vfix[o];
    sum += vf;
    v_w[o] = static_cast<double>(vf) * UNFIX;
    v_max[o] = __uint_as_float(vmaxb[o]);
    s_w[o] = static_cast<double>(sfix[o]) * UNFIX;
    s_max[o] = __uint_as_float(smaxb[o]);
  }
  // op count (prefill.py:386-389): the sampled rows, split across the chunks
  const int per = (n_s + gridDim.x - 1) / gridDim.x;
  for (int r = ck * per + threadIdx.x; r < min(n_s, (ck + 1) * per); r += FIN_THREADS) {
    const long long g = row_offset + rows[static_cast<int64_t>(h) * n_s + r];
    cnt += min(g, static_cast<long long>(n_total - 1)) + 1;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = sum;
    redc[threadIdx.x >> 5] = cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    long long c = 0;
    for (int i = 0; i < FIN_THREADS / 32; ++i) {
      s += red[i];
      c += redc[i];
    }
    atomicAdd(acc_tot + h, s);
    atomicAdd(acc_cnt + h, static_cast<unsigned long long>(c));
    __threadfence();
    last = atomicAdd(ticket + h, 1u) == gridDim.x - 1;
    if (last) {
      __threadfence();
      const unsigned long long ts = atomicAdd(acc_tot + h, 0ull), tc = atomicAdd(acc_cnt + h, 0ull);
      total[h] = static_cast<double>(ts) * UNFIX;
      score_count[h] = static_cast<long long>(tc);
      acc_tot[h] = 0ull;
      acc_cnt[h] = 0ull;
      ticket[h] = 0u;
    }
  }
}

// per sampled row: merge the chunk statistics in chunk order (as k1_lines does)
// into log2-sum-exp2 = m + log2(l) over all causal columns (ls_plan_coverage)
__global__ void row_lse_kernel(const float2 *pstats, const int32_t *rows, int n_s, int n_chunks, int row_offset,
                               int n_total, float *lse) {
  const int h = blockIdx.y, r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_s) return;
  const int g = row_offset + rows[static_cast<int64_t>(h) * n_s + r];
  const int n_ck = min(g, n_total - 1) / CHUNK + 1;
  const float2 *ps = pstats + (static_cast<int64_t>(h) * n_chunks * n_s + r) * 4;
  float m = -INFINITY, l = 0.f;
  for (int c = 0; c < n_ck; ++c)
    for (int e = 0; e < 4; ++e) {
      const float2 v = ps[static_cast<int64_t>(c) * n_s * 4 + e];
      if (v.y == 0.f) continue;
      const float mn = fmaxf(m, v.x);
      l = (m == -INFINITY ? 0.f : l * fast_exp2(m - mn)) + v.y * fast_exp2(v.x - mn);
      m = mn;
    }
  lse[static_cast<int64_t>(h) * n_s + r] = l > 0.f ? m + __log2f(l) : -INFINITY;
}

inline int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace k1tc

size_t score_lines_tc_workspace(const ls_layer_desc *L, int32_t n_s) {
  const size_t n_rt = (n_s + k1tc::BM - 1) / k1tc::BM;
  const size_t n_ch = (L->n_total + k1tc::CHUNK - 1) / k1tc::CHUNK;
  const size_t H = L->n_heads;
  return H * n_ch * n_s * 4 * sizeof(float2) + H * L->n_total * (8 + 8 + 4 + 4) + H * 24 + (H * n_rt + 1) * 4 +
         10 * 256 + 4096;
}

namespace {
int k1_prepare(const ls_layer_desc *L, int32_t n_s, const uint16_t *q, const uint16_t *k, const int32_t *rows,
               float *row_stats, void *ws, size_t ws_bytes, k1tc::Params &p, unsigned long long **fin,
               unsigned int **tick, bool accumulators, cudaStream_t st) {
  LS_REQUIRE(ws_bytes >= score_lines_tc_workspace(L, n_s), LS_ERR_WORKSPACE, "score_lines workspace too small");
  p = k1tc::Params{};
  p.q = q;
  p.k = k;
  p.rows = rows;
  p.n_heads = L->n_heads;
  p.group = L->n_heads / L->n_kv_heads;
  p.n_s = n_s;
  p.n_total = L->n_total;
  p.row_offset = L->row_offset;
  p.n_rt = (n_s + k1tc::BM - 1) / k1tc::BM;
  p.n_chunks = (L->n_total + k1tc::CHUNK - 1) / k1tc::CHUNK;
  p.q_head_stride = L->q_head_stride;
  p.kv_head_stride = L->kv_head_stride;
  p.scale_log2 = kLog2e / sqrtf(static_cast<float>(L->head_dim));
  p.row_stats = row_stats;
  p.status = device_status_ptr();
  p.dbg = g_debug_buffer;
  Carver c(ws, ws_bytes);
  const size_t H = L->n_heads;
  p.pstats = c.take<float2>(H * p.n_chunks * n_s * 4);
  // every (chunk, row) has 2 segment slots x 2 column halves; unwritten ones stay (0, 0)
  LS_CUDA(cudaMemsetAsync(p.pstats, 0, H * p.n_chunks * n_s * 4 * sizeof(float2), st));
  int32_t *tstart = c.take<int32_t>(H * p.n_rt + 1);
  p.tstart = tstart;
  if (accumulators) {
    p.vfix = c.take<unsigned long long>(H * L->n_total);
    p.sfix = c.take<unsigned long long>(H * L->n_total);
    p.vmaxb = c.take<unsigned int>(H * L->n_total);
    p.smaxb = c.take<unsigned int>(H * L->n_total);
    fin[0] = c.take<unsigned long long>(H);
    fin[1] = c.take<unsigned long long>(H);
    *tick = c.take<unsigned int>(H);
    // line accumulators and finish counters are consecutive in the workspace (shared
    // with other entries, so zeroed per call): one memset
    LS_CUDA(cudaMemsetAsync(p.vfix, 0, reinterpret_cast<char *>(*tick + H) - reinterpret_cast<char *>(p.vfix), st));
  }
  k1tc::k1_tiles_kernel<<<1, 1024, 0, st>>>(p, tstart);
  LS_LAUNCH_CHECK("k1_tiles_kernel");
  return LS_OK;
}

template <int D>
int k1_stats_launch(const CUtensorMap &tmk, const k1tc::Params &p, cudaStream_t st) {
  const int s1 = k1tc::StatsSmem<D>::TOTAL + 1024;
  LS_CUDA(cudaFuncSetAttribute(k1tc::k1_stats_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, s1));
  k1tc::k1_stats_kernel<D><<<2 * k1tc::sm_count(), k1tc::STATS_THREADS, s1, st>>>(tmk, p);
  LS_LAUNCH_CHECK("k1_stats_kernel");
  return LS_OK;
}

template <int D>
int k1_lines_launch(const CUtensorMap &tmk, const k1tc::Params &p, cudaStream_t st) {
  const int s2 = k1tc::LinesSmem<D>::TOTAL + 1024;
  LS_CUDA(cudaFuncSetAttribute(k1tc::k1_lines_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, s2));
  k1tc::k1_lines_kernel<D><<<k1tc::sm_count(), k1tc::LINES_THREADS + 32, s2, st>>>(tmk, p);
  LS_LAUNCH_CHECK("k1_lines_kernel");
  return LS_OK;
}
}  // namespace

int score_lines_tc(const ls_layer_desc *L, int32_t n_s, const uint16_t *q, const uint16_t *k, const int32_t *rows,
                   double *v_w, float *v_max, double *s_w, float *s_max, float *row_stats, double *total,
                   int64_t *score_count, void *ws, size_t ws_bytes, cudaStream_t st) {
  k1tc::Params p;
  unsigned long long *fin[2];
  unsigned int *tick = nullptr;
  int s = k1_prepare(L, n_s, q, k, rows, row_stats, ws, ws_bytes, p, fin, &tick, true, st);
  if (s) return s;
  CUtensorMap tmk;
  if ((s = make_tmap_bf16_3d(&tmk, k, L->head_dim, L->n_total, L->n_kv_heads, L->head_dim, L->kv_head_stride)))
    return s;
  if (L->head_dim == 128) {
    if ((s = k1_stats_launch<128>(tmk, p, st)) || (s = k1_lines_launch<128>(tmk, p, st))) return s;
  } else {
    if ((s = k1_stats_launch<64>(tmk, p, st)) || (s = k1_lines_launch<64>(tmk, p, st))) return s;
  }
  const dim3 fg((L->n_total + k1tc::FIN_CHUNK - 1) / k1tc::FIN_CHUNK, L->n_heads);
  k1tc::k1_finish_kernel<<<fg, k1tc::FIN_THREADS, 0, st>>>(p.vfix, p.vmaxb, p.sfix, p.smaxb, rows, n_s, L->n_total,
                                                         L->row_offset, v_w, v_max, s_w, s_max, total, score_count,
                                                         fin[0], fin[1], tick);
  LS_LAUNCH_CHECK("k1_finish_kernel");
  return LS_OK;
}

// K1 pass 1 only, for the rows given: log2-sum-exp2 of every row over all its
// causal columns (the dense softmax normaliser), [H][n_s]
int score_row_lse(const ls_layer_desc *L, int32_t n_s, const uint16_t *q, const uint16_t *k, const int32_t *rows,
                  float *lse, void *ws, size_t ws_bytes, cudaStream_t st) {
  k1tc::Params p;
  unsigned long long *fin[2];
  unsigned int *tick = nullptr;
  int s = k1_prepare(L, n_s, q, k, rows, nullptr, ws, ws_bytes, p, fin, &tick, false, st);
  if (s) return s;
  CUtensorMap tmk;
  if ((s = make_tmap_bf16_3d(&tmk, k, L->head_dim, L->n_total, L->n_kv_heads, L->head_dim, L->kv_head_stride)))
    return s;
  if ((s = L->head_dim == 128 ? k1_stats_launch<128>(tmk, p, st) : k1_stats_launch<64>(tmk, p, st))) return s;
  k1tc::row_lse_kernel<<<dim3((n_s + 255) / 256, L->n_heads), 256, 0, st>>>(p.pstats, rows, n_s, p.n_chunks,
                                                                           L->row_offset, L->n_total, lse);
  LS_LAUNCH_CHECK("row_lse_kernel");
  return LS_OK;
}

}  // namespace ls
