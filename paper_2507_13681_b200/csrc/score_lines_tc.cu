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
// bf16 [heads][rows][d] tensor map, box 64 columns x 128 rows, 128-B swizzle (vs_attention_ws.cu)
int make_tmap_bf16_3d(CUtensorMap *m, const void *base, int d, int64_t rows, int heads, int64_t row_stride_el,
                      int64_t head_stride_el);
}

namespace ls {
namespace k1tc {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int CHUNK = 1024;        // key columns per CTA
constexpr int LDP = BN + 4;        // fp32 P row stride (16-B rows: conflict-free STS.128 / column LDS)
constexpr int ACC_CAP = 3072;      // shared slash accumulator (diagonals per chunk)
constexpr int RP_CAP = 2048;       // row-pointer table: first sampled row at or after a position
constexpr int LINES_THREADS = 512; // 16 warps: 4 per TMEM lane quadrant
constexpr double FIX = 1099511627776.0;  // 2^40
constexpr double UNFIX = 1.0 / 1099511627776.0;

struct Params {
  const uint16_t *q;
  const uint16_t *k;
  const int32_t *rows;
  int n_heads, group, n_s, n_total, row_offset, n_rt, n_chunks;
  int64_t q_head_stride, kv_head_stride;
  float scale_log2;
  float2 *pstats;  // [H][n_rt][n_chunks][BM]
  unsigned long long *vfix, *sfix;  // [H][n_total]
  unsigned int *vmaxb, *smaxb;      // [H][n_total]
  float *row_stats;                 // [H][n_s][2]
};

template <int D>
struct StatsSmem {
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = BM * D * 2;
  static constexpr int OFF_MISC = OFF_K + 2 * BN * D * 2;
  static constexpr int TOTAL = OFF_MISC + 1024 + 64 + 1024 + 1024;  // (+ TMA / s_empty barriers, halves' (m, l))
};

template <int D>
struct LinesSmem {
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = BM * D * 2;
  static constexpr int OFF_P = OFF_K + 2 * BN * D * 2;
  static constexpr int OFF_ACC = OFF_P + BM * LDP * 4;         // double[ACC_CAP]
  static constexpr int OFF_ACCM = OFF_ACC + ACC_CAP * 8;       // float[ACC_CAP]
  static constexpr int OFF_RP = OFF_ACCM + ACC_CAP * 4;        // int[RP_CAP] row pointer by position
  static constexpr int OFF_MISC = OFF_RP + RP_CAP * 4;  // barriers | gs | m | 1/l | colp [4][128] f64 | colm [4][128]
  static constexpr int TOTAL = OFF_MISC + 2048 + 4096 + 2048 + 1024;
};

__device__ __forceinline__ void zfill16(uint32_t saddr, const void *g, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(ok ? 16 : 0) : "memory");
}

__device__ __forceinline__ unsigned long long to_fix(double x) {
  return static_cast<unsigned long long>(__double2ll_rn(x * FIX));
}

// shared prologue: TMEM, barriers, row positions, gathered Q tile
template <int D>
__device__ __forceinline__ void setup(const Params &p, unsigned char *smem, int off_misc, int h, int rt, int &nr,
                                      int *gs, uint64_t *mbar, uint32_t *tmem_sh) {
  const int tid = threadIdx.x;
  const int r_begin = rt * BM;
  nr = min(BM, p.n_s - r_begin);
  if ((tid >> 5) == 0) tc::tmem_alloc(tmem_sh, 256);
  if (tid == 0) {
    tc::mbar_init(&mbar[0], 1);
    tc::mbar_init(&mbar[1], 1);
  }
  const int32_t *rows_h = p.rows + static_cast<int64_t>(h) * p.n_s;
  if (tid < BM) {
    const int lr = tid < nr ? rows_h[r_begin + tid] : 0;
    gs[tid] = tid < nr ? p.row_offset + lr : 0x7fffffff;
    const uint16_t *qrow = p.q + static_cast<int64_t>(h) * p.q_head_stride + static_cast<int64_t>(lr) * D;
    const uint32_t qs = tc::smem_u32(smem);
#pragma unroll
    for (int ch = 0; ch < D / 8; ++ch) zfill16(qs + tc::sw128_offset(tid, ch, BM), qrow + ch * 8, tid < nr);
  }
  tc::cp_async_commit();
  (void)off_misc;
}

template <int D>
__device__ __forceinline__ void load_k(const Params &p, unsigned char *smem, int off_k, const uint16_t *kbase, int c0,
                                       int buf) {
  // 128 key rows; threads >= 128 help when blockDim is 256
  const uint32_t ks = tc::smem_u32(smem + off_k + buf * BN * D * 2);
  constexpr int CH = D / 8;
  for (int i = threadIdx.x; i < BN * CH; i += blockDim.x) {
    const int r = i / CH, ch = i % CH;
    const int c = c0 + r;
    const bool ok = c < p.n_total;
    zfill16(ks + tc::sw128_offset(r, ch, BN), kbase + static_cast<int64_t>(ok ? c : 0) * D + ch * 8, ok);
  }
  tc::cp_async_commit();
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

__device__ __forceinline__ void cta_sync_tc() {
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
}

// ------------------------------------------------------------- pass 1
// 256 threads, two per sampled row (TMEM lane = row, warps 0-3 columns 0-63,
// warps 4-7 columns 64-127), each with its own online (max, sum) over its
// half of every tile, merged once at the end. K tiles arrive by TMA (thread
// 0), S = Qs K^T double-buffered in TMEM: S(t+1) is issued before the threads
// process S(t), and a buffer is reused once all threads have read it
// (s_empty, count 256) -- no CTA barrier per tile.
constexpr int STATS_THREADS = 256;
template <int D>
__global__ void __launch_bounds__(STATS_THREADS) k1_stats_kernel(const __grid_constant__ CUtensorMap tm_k, Params p) {
  extern __shared__ unsigned char smem_dyn[];
  using L = StatsSmem<D>;
  unsigned char *smem =
      reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + L::OFF_MISC);          // s_full[2] (setup)
  uint32_t *tmem_sh = reinterpret_cast<uint32_t *>(smem + L::OFF_MISC + 16);
  int *gs = reinterpret_cast<int *>(smem + L::OFF_MISC + 64);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + L::OFF_MISC + 1024);   // [2] TMA
  uint64_t *s_empty = full + 2;                                             // [2] count STATS_THREADS
  float2 *half = reinterpret_cast<float2 *>(smem + L::OFF_MISC + 1024 + 64);  // [128] second half's (m, l)
  const int ck = blockIdx.x, rt = blockIdx.y, h = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int row = tid & (BM - 1), hc = tid >> 7;  // column half
  float2 *ps = p.pstats + ((static_cast<int64_t>(h) * p.n_rt + rt) * p.n_chunks + ck) * BM;
  // chunk bounds against this row tile's causal extent
  const int r_last = min(p.n_s, (rt + 1) * BM) - 1;
  const int g_last = p.row_offset + p.rows[static_cast<int64_t>(h) * p.n_s + r_last];
  const int c_begin = ck * CHUNK;
  if (c_begin > g_last) {
    if (tid < BM) ps[tid] = make_float2(-INFINITY, 0.f);
    return;
  }
  const int c_end = min(c_begin + CHUNK, g_last + 1);
  const int kv = h / p.group;
  const int n_tiles = (c_end - c_begin + BN - 1) / BN;
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&full[b], 1);
      tc::mbar_init(&s_empty[b], STATS_THREADS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tc::prefetch_tmap(&tm_k);
    for (int t = 0; t < 2 && t < n_tiles; ++t) tma_k<D>(&tm_k, smem, L::OFF_K, t, &full[t], c_begin + t * BN, kv);
  }
  int nr;
  setup<D>(p, smem, L::OFF_MISC, h, rt, nr, gs, mbar, tmem_sh);  // Q rows (cp.async), TMEM, s_full barriers
  tc::cp_async_wait<0>();
  cta_sync_tc();
  const uint32_t tmem = *tmem_sh;
  if (tid == 0) {
    tc::mbar_wait(&full[0], 0);
    issue_s<D>(smem, L::OFF_K, tmem, 0, mbar);
  }
  const int my_g = gs[row];
  const bool row_ok = row < nr;
  const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
  float m = -INFINITY, l = 0.f;
  for (int t = 0; t < n_tiles; ++t) {
    const int buf = t & 1;
    const int c0 = c_begin + t * BN;
    if (tid == 0 && t + 1 < n_tiles) {  // S(t+1) behind S(t): its buffer was read by every thread at t-1
      tc::mbar_wait(&full[buf ^ 1], ((t + 1) >> 1) & 1);
      if (t >= 1) tc::mbar_wait(&s_empty[buf ^ 1], ((t - 1) >> 1) & 1);
      tc::fence_after_sync();
      issue_s<D>(smem, L::OFF_K, tmem, buf ^ 1, mbar);
    }
    tc::mbar_wait(&mbar[buf], (t >> 1) & 1);
    tc::fence_after_sync();
    if (tid == 0 && t + 2 < n_tiles)  // S(t) is done with K stage `buf`
      tma_k<D>(&tm_k, smem, L::OFF_K, buf, &full[buf], c0 + 2 * BN, kv);
    const int lim = min(my_g, c_end - 1) - c0 - 64 * hc;  // last valid column of this thread's 64
    float sv[64];
    tc::tmem_ld32(tmem + buf * 128 + lane_base + 64 * hc, sv);
    tc::tmem_ld32(tmem + buf * 128 + lane_base + 64 * hc + 32, sv + 32);
    tc::tmem_wait_ld();
    tc::fence_before_sync();
    tc::mbar_arrive(&s_empty[buf]);
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
  }
  // merge the two column halves of each row (half 0 + half 1, fixed order)
  if (hc == 1) half[row] = make_float2(m, l);
  __syncthreads();
  if (hc == 0) {
    const float2 o = half[row];
    const float mn = fmaxf(m, o.x);
    float lt = 0.f;
    if (m != -INFINITY) lt += l * fast_exp2(m - mn);
    if (o.x != -INFINITY) lt += o.y * fast_exp2(o.x - mn);
    ps[row] = make_float2(row_ok ? mn : -INFINITY, row_ok ? lt : 0.f);
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 256);
}

// ------------------------------------------------------------- pass 2
// 16 warps. Per 128-key tile: P = exp2(s - m) / l (fp32) from TMEM into
// shared memory (warp w: TMEM lanes of quadrant w % 4, 32 columns of block
// w / 4); vertical partials by 4 threads per column (32 rows each, fp64, in
// row order); slash partials by thread-owns-diagonal, rows ascending, with
// the first contributing row read from a position -> row table instead of a
// binary search; per-tile slash sums (<= ~13 cells) in fp32, accumulated per
// chunk in fp64 shared memory.
template <int D>
__global__ void __launch_bounds__(LINES_THREADS, 1) k1_lines_kernel(const __grid_constant__ CUtensorMap tm_k, Params p) {
  extern __shared__ unsigned char smem_dyn[];
  using L = LinesSmem<D>;
  unsigned char *smem =
      reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + L::OFF_MISC);
  uint32_t *tmem_sh = reinterpret_cast<uint32_t *>(smem + L::OFF_MISC + 16);
  int *gs = reinterpret_cast<int *>(smem + L::OFF_MISC + 64);              // [128]
  float *m_sh = reinterpret_cast<float *>(smem + L::OFF_MISC + 64 + 512);  // [128]
  float *li_sh = m_sh + BM;                                                 // [128]
  double *colp = reinterpret_cast<double *>(smem + L::OFF_MISC + 2048);         // [4][128]
  float *colm = reinterpret_cast<float *>(smem + L::OFF_MISC + 2048 + 4096);    // [4][128]
  float *Pf = reinterpret_cast<float *>(smem + L::OFF_P);
  double *acc = reinterpret_cast<double *>(smem + L::OFF_ACC);
  float *accm = reinterpret_cast<float *>(smem + L::OFF_ACCM);
  int *rp = reinterpret_cast<int *>(smem + L::OFF_RP);
  const int ck = blockIdx.x, rt = blockIdx.y, h = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r_last = min(p.n_s, (rt + 1) * BM) - 1;
  const int g_last = p.row_offset + p.rows[static_cast<int64_t>(h) * p.n_s + r_last];
  const int c_begin = ck * CHUNK;
  if (c_begin > g_last) return;
  const int c_end = min(c_begin + CHUNK, g_last + 1);
  int nr;
  setup<D>(p, smem, L::OFF_MISC, h, rt, nr, gs, mbar, tmem_sh);
  const uint16_t *kbase = p.k + static_cast<int64_t>(h / p.group) * p.kv_head_stride;
  // combine the chunk statistics of this CTA's rows (chunk order: deterministic)
  if (tid < BM) {
    float m = -INFINITY, l = 0.f;
    const float2 *ps = p.pstats + (static_cast<int64_t>(h) * p.n_rt + rt) * p.n_chunks * BM + tid;
    for (int c = 0; c < p.n_chunks; ++c) {
      const float2 v = ps[static_cast<int64_t>(c) * BM];
      if (v.x == -INFINITY) continue;
      const float mn = fmaxf(m, v.x);
      l = (m == -INFINITY ? 0.f : l * fast_exp2(m - mn)) + v.y * fast_exp2(v.x - mn);
      m = mn;
    }
    m_sh[tid] = m;
    li_sh[tid] = l > 0.f ? 1.f / l : 0.f;
    if (ck == 0 && tid < nr) {
      float *rs = p.row_stats + (static_cast<int64_t>(h) * p.n_s + rt * BM + tid) * 2;
      rs[0] = m;
      rs[1] = l > 0.f ? 1.f / l : 0.f;
    }
  }
  const int n_tiles = (c_end - c_begin + BN - 1) / BN;
  uint64_t *kfull = reinterpret_cast<uint64_t *>(smem + L::OFF_MISC + 32);  // [2] TMA K stages
  const int kvh = h / p.group;
  if (tid == 0) {
    tc::mbar_init(&kfull[0], 1);
    tc::mbar_init(&kfull[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tc::prefetch_tmap(&tm_k);
    tma_k<D>(&tm_k, smem, L::OFF_K, 0, &kfull[0], c_begin, kvh);
  }
  (void)kbase;
  tc::cp_async_wait<0>();
  cta_sync_tc();
  const uint32_t tmem = *tmem_sh;
  if (tid == 0) {
    tc::mbar_wait(&kfull[0], 0);
    issue_s<D>(smem, L::OFF_K, tmem, 0, mbar);
  }
  const int g_first = gs[0];
  const int g_hi = gs[nr - 1];
  // position -> first sampled row at or after it, for positions [g_first, g_hi]
  const int rp_span = g_hi - g_first + 1;
  const bool use_rp = rp_span <= RP_CAP;
  if (use_rp)
    for (int x = tid; x < rp_span; x += LINES_THREADS) rp[x] = lower_bound_dev(gs, nr, g_first + x);
  // slash accumulator window of the chunk: d in [d_base, d_base + width)
  const int d_base = max(0, g_first - (c_end - 1));
  const int width = g_hi - c_begin - d_base + 1;
  const bool smem_acc = width <= ACC_CAP;
  if (smem_acc)
    for (int i = tid; i < width; i += LINES_THREADS) {
      acc[i] = 0.0;
      accm[i] = 0.f;
    }
  __syncthreads();
  // TMEM reads: warp w -> lanes 32*(w%4), columns [32*(w/4), +32)
  const int row = (warp & 3) * 32 + lane;
  const int cblk = (warp >> 2) * 32;
  const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
  const int my_g = gs[row];
  const bool row_ok = row < nr;
  // P = exp2(s * scale - m) / l = exp2(s * scale - (m + log2 l))
  const float mr = li_sh[row] > 0.f ? m_sh[row] - __log2f(li_sh[row]) : INFINITY;
  uint32_t ph0 = 0, ph1 = 0;
  unsigned long long *sfix = p.sfix + static_cast<int64_t>(h) * p.n_total;
  unsigned int *smaxb = p.smaxb + static_cast<int64_t>(h) * p.n_total;
  for (int t = 0; t < n_tiles; ++t) {
    const int buf = t & 1;
    const int c0 = c_begin + t * BN;
    if (t + 1 < n_tiles && tid == 0)  // stage buf^1 held K(t-1), consumed by S(t-1)
      tma_k<D>(&tm_k, smem, L::OFF_K, buf ^ 1, &kfull[buf ^ 1], c0 + BN, kvh);
    tc::mbar_wait(&mbar[buf], buf ? ph1 : ph0);
    if (buf) ph1 ^= 1; else ph0 ^= 1;
    tc::fence_after_sync();
    {
      const int lim = min(my_g, c_end - 1) - c0 - cblk;  // last valid column of this thread's 32
      float sv[32];
      tc::tmem_ld32(tmem + buf * 128 + lane_base + cblk, sv);
      tc::tmem_wait_ld();
      float4 *prow = reinterpret_cast<float4 *>(Pf + row * LDP + cblk);
      if (row_ok && lim >= 31) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          prow[j / 4] = make_float4(fast_exp2(fmaf(sv[j], p.scale_log2, -mr)), fast_exp2(fmaf(sv[j + 1], p.scale_log2, -mr)),
                                    fast_exp2(fmaf(sv[j + 2], p.scale_log2, -mr)), fast_exp2(fmaf(sv[j + 3], p.scale_log2, -mr)));
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
    }
    // P lives in generic-proxy shared memory only (the MMAs read Q and K): no
    // proxy fence here, just the TMEM read -> next-MMA ordering around the barrier
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (t + 1 < n_tiles && tid == 0) {
      tc::mbar_wait(&kfull[buf ^ 1], ((t + 1) >> 1) & 1);
      issue_s<D>(smem, L::OFF_K, tmem, buf ^ 1, mbar);
    }
    // vertical partials: four threads per column (32-row quarters)
    {
      const int j = tid & (BN - 1), qq = tid >> 7;
      double sw = 0.0;
      float mx = 0.f;
      const int r0 = qq * 32, r1 = min(nr, r0 + 32);
      for (int r = r0; r < r1; ++r) {
        const float v = Pf[r * LDP + j];
        sw += static_cast<double>(v);
        mx = fmaxf(mx, v);
      }
      colp[qq * BN + j] = sw;
      colm[qq * BN + j] = mx;
    }
    // slash partials: thread owns diagonal d, rows ascending
    {
      const int d_lo = max(d_base, g_first - (c0 + BN - 1));
      const int d_hi = g_hi - c0;
      for (int dd = d_lo + tid; dd <= d_hi; dd += LINES_THREADS) {
        const int glo = c0 + dd, ghi = min(c0 + dd + BN - 1, g_hi);
        int r, r_end;
        if (use_rp) {
          r = rp[max(glo, g_first) - g_first];
          r_end = ghi + 1 <= g_hi ? rp[ghi + 1 - g_first] : nr;
        } else {
          r = lower_bound_dev(gs, nr, glo);
          r_end = lower_bound_dev(gs, nr, ghi + 1);
        }
        float sw = 0.f, mx = 0.f;
        const float *pcol = Pf - dd - c0;
#pragma unroll 4
        for (; r < r_end; ++r) {
          const float v = pcol[r * LDP + gs[r]];
          sw += v;
          mx = fmaxf(mx, v);
        }
        if (smem_acc) {
          acc[dd - d_base] += static_cast<double>(sw);
          accm[dd - d_base] = fmaxf(accm[dd - d_base], mx);
        } else if (sw > 0.f) {
          atomicAdd(sfix + dd, to_fix(static_cast<double>(sw)));
          atomicMax(smaxb + dd, __float_as_uint(mx));
        }
      }
    }
    __syncthreads();
    if (tid < BN) {
      const int c = c0 + tid;
      if (c < c_end) {
        const double sw = ((colp[tid] + colp[BN + tid]) + colp[2 * BN + tid]) + colp[3 * BN + tid];
        const float mx = fmaxf(fmaxf(colm[tid], colm[BN + tid]), fmaxf(colm[2 * BN + tid], colm[3 * BN + tid]));
        if (sw > 0.0) atomicAdd(p.vfix + static_cast<int64_t>(h) * p.n_total + c, to_fix(sw));
        if (mx > 0.f) atomicMax(p.vmaxb + static_cast<int64_t>(h) * p.n_total + c, __float_as_uint(mx));
      }
    }
    // (no barrier here: every read of Pf precedes the barrier above, and the next
    // tile writes colp / the slash accumulator only after its own first barrier)
  }
  if (smem_acc)
    for (int i = tid; i < width; i += LINES_THREADS) {
      if (acc[i] > 0.0) atomicAdd(sfix + d_base + i, to_fix(acc[i]));
      if (accm[i] > 0.f) atomicMax(smaxb + d_base + i, __float_as_uint(accm[i]));
    }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 256);
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
__global__ void row_lse_kernel(const float2 *pstats, int n_s, int n_rt, int n_chunks, float *lse) {
  const int h = blockIdx.y, r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_s) return;
  const float2 *ps = pstats + (static_cast<int64_t>(h) * n_rt + r / BM) * n_chunks * BM + (r % BM);
  float m = -INFINITY, l = 0.f;
  for (int c = 0; c < n_chunks; ++c) {
    const float2 v = ps[static_cast<int64_t>(c) * BM];
    if (v.x == -INFINITY) continue;
    const float mn = fmaxf(m, v.x);
    l = (m == -INFINITY ? 0.f : l * fast_exp2(m - mn)) + v.y * fast_exp2(v.x - mn);
    m = mn;
  }
  lse[static_cast<int64_t>(h) * n_s + r] = l > 0.f ? m + __log2f(l) : -INFINITY;
}

}  // namespace k1tc

size_t score_lines_tc_workspace(const ls_layer_desc *L, int32_t n_s) {
  const size_t n_rt = (n_s + k1tc::BM - 1) / k1tc::BM;
  const size_t n_ch = (L->n_total + k1tc::CHUNK - 1) / k1tc::CHUNK;
  const size_t H = L->n_heads;
  return H * n_rt * n_ch * k1tc::BM * sizeof(float2) + H * L->n_total * (8 + 8 + 4 + 4) + H * 24 + 8 * 256 + 4096;
}

int score_lines_tc(const ls_layer_desc *L, int32_t n_s, const uint16_t *q, const uint16_t *k, const int32_t *rows,
                   double *v_w, float *v_max, double *s_w, float *s_max, float *row_stats, double *total,
                   int64_t *score_count, void *ws, size_t ws_bytes, cudaStream_t st) {
  LS_REQUIRE(ws_bytes >= score_lines_tc_workspace(L, n_s), LS_ERR_WORKSPACE, "score_lines workspace too small");
  k1tc::Params p;
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
  Carver c(ws, ws_bytes);
  const size_t H = L->n_heads;
  p.pstats = c.take<float2>(H * p.n_rt * p.n_chunks * k1tc::BM);
  p.vfix = c.take<unsigned long long>(H * L->n_total);
  p.sfix = c.take<unsigned long long>(H * L->n_total);
  p.vmaxb = c.take<unsigned int>(H * L->n_total);
  p.smaxb = c.take<unsigned int>(H * L->n_total);
  unsigned long long *fin_tot = c.take<unsigned long long>(H);
  unsigned long long *fin_cnt = c.take<unsigned long long>(H);
  unsigned int *fin_tick = c.take<unsigned int>(H);
  // line accumulators and finish counters are consecutive in the workspace (shared
  // with other entries, so zeroed per call): one memset
  LS_CUDA(cudaMemsetAsync(p.vfix, 0, reinterpret_cast<char *>(fin_tick + H) - reinterpret_cast<char *>(p.vfix), st));
  dim3 grid(p.n_chunks, p.n_rt, L->n_heads);
  CUtensorMap tmk;
  int st_map = make_tmap_bf16_3d(&tmk, k, L->head_dim, L->n_total, L->n_kv_heads, L->head_dim, L->kv_head_stride);
  if (st_map) return st_map;
  if (L->head_dim == 128) {
    const int s1 = k1tc::StatsSmem<128>::TOTAL, s2 = k1tc::LinesSmem<128>::TOTAL;
    LS_CUDA(cudaFuncSetAttribute(k1tc::k1_stats_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, s1));
    LS_CUDA(cudaFuncSetAttribute(k1tc::k1_lines_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, s2));
    k1tc::k1_stats_kernel<128><<<grid, k1tc::STATS_THREADS, s1, st>>>(tmk, p);
    LS_LAUNCH_CHECK("k1_stats_kernel");
    k1tc::k1_lines_kernel<128><<<grid, k1tc::LINES_THREADS, s2, st>>>(tmk, p);
  } else {
    const int s1 = k1tc::StatsSmem<64>::TOTAL, s2 = k1tc::LinesSmem<64>::TOTAL;
    LS_CUDA(cudaFuncSetAttribute(k1tc::k1_stats_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, s1));
    LS_CUDA(cudaFuncSetAttribute(k1tc::k1_lines_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, s2));
    k1tc::k1_stats_kernel<64><<<grid, k1tc::STATS_THREADS, s1, st>>>(tmk, p);
    LS_LAUNCH_CHECK("k1_stats_kernel");
    k1tc::k1_lines_kernel<64><<<grid, k1tc::LINES_THREADS, s2, st>>>(tmk, p);
  }
  LS_LAUNCH_CHECK("k1_lines_kernel");
  {
    const dim3 fg((L->n_total + k1tc::FIN_CHUNK - 1) / k1tc::FIN_CHUNK, L->n_heads);
    k1tc::k1_finish_kernel<<<fg, k1tc::FIN_THREADS, 0, st>>>(p.vfix, p.vmaxb, p.sfix, p.smaxb, rows, n_s, L->n_total,
                                                           L->row_offset, v_w, v_max, s_w, s_max, total, score_count,
                                                           fin_tot, fin_cnt, fin_tick);
  }
  LS_LAUNCH_CHECK("k1_finish_kernel");
  return LS_OK;
}

// K1 pass 1 only, for the rows given: log2-sum-exp2 of every row over all its
// causal columns (the dense softmax normaliser), [H][n_s]
int score_row_lse(const ls_layer_desc *L, int32_t n_s, const uint16_t *q, const uint16_t *k, const int32_t *rows,
                  float *lse, void *ws, size_t ws_bytes, cudaStream_t st) {
  LS_REQUIRE(ws_bytes >= score_lines_tc_workspace(L, n_s), LS_ERR_WORKSPACE, "row_lse workspace too small");
  k1tc::Params p{};
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
  Carver c(ws, ws_bytes);
  p.pstats = c.take<float2>(static_cast<size_t>(L->n_heads) * p.n_rt * p.n_chunks * k1tc::BM);
  dim3 grid(p.n_chunks, p.n_rt, L->n_heads);
  CUtensorMap tmk;
  int st_map = make_tmap_bf16_3d(&tmk, k, L->head_dim, L->n_total, L->n_kv_heads, L->head_dim, L->kv_head_stride);
  if (st_map) return st_map;
  if (L->head_dim == 128) {
    const int s1 = k1tc::StatsSmem<128>::TOTAL;
    LS_CUDA(cudaFuncSetAttribute(k1tc::k1_stats_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, s1));
    k1tc::k1_stats_kernel<128><<<grid, k1tc::STATS_THREADS, s1, st>>>(tmk, p);
  } else {
    const int s1 = k1tc::StatsSmem<64>::TOTAL;
    LS_CUDA(cudaFuncSetAttribute(k1tc::k1_stats_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, s1));
    k1tc::k1_stats_kernel<64><<<grid, k1tc::STATS_THREADS, s1, st>>>(tmk, p);
  }
  LS_LAUNCH_CHECK("k1_stats_kernel");
  k1tc::row_lse_kernel<<<dim3((n_s + 255) / 256, L->n_heads), 256, 0, st>>>(p.pstats, n_s, p.n_rt, p.n_chunks, lse);
  LS_LAUNCH_CHECK("row_lse_kernel");
  return LS_OK;
}

}  // namespace ls
