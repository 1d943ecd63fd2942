// K5 (production path) -- warp-specialized vertical/slash sparse attention.
//
// Contract: reference masked_sparse_attention (tensor_ops.py:141-183) with the
// exact `_row_columns` cell set (tensor_ops.py:130-138) and the diagonal
// fallback, for every q-head of a layer; per-row cell counts = OpCounter
// increments (tensor_ops.py:172-174).
//
// One CTA per (head, 128-row q tile), 10 warps:
//   warp 8  (1 thread) TMA producer: every operand tile arrives by
//           cp.async.bulk.tensor (128B swizzle, zero fill out of range) into a
//           3-stage K ring (a stage is free once S(i) has read it) and a
//           2-stage V ring (free once PV(i) has read it); K runs one tile
//           ahead of V, so S(i+1)'s operand is resident while P(i) is made.
//   warp 9  (1 thread) MMA issuer: S(i) = Q K(i)^T into a double-buffered
//           TMEM S, then O += P(i-1) V(i-1) into a TMEM O accumulator
//           (tcgen05.mma kind::f16, bf16 -> fp32), commits to mbarriers.
//   warps 0-7 softmax: thread (row, half) owns one TMEM lane and 64 of the
//           128 S columns; masked online softmax in the log2 domain with lazy
//           rescaling of the TMEM O (only when the running max grows by 2^8),
//           P to shared memory in the UMMA K-major layout.
// Tile kinds, in order:
//   dense    : key block [128b, 128b+128) crossed by >= DENSE_SLASHES selected
//              slashes; mask causal & (vbit | sbit)              (tensor cores)
//   gathered : 128 consecutive entries of the head's compacted selected
//              verticals (K/V rows gathered once per call by a pre-kernel);
//              mask causal & column not in a dense block          (tensor cores)
//   window   : the key ranges [g0-d, g_hi-d] of selected slashes whose cells
//              fall outside dense blocks, merged and covered by disjoint
//              128-key windows at unaligned starts (tensor cores); mask
//              causal & sbit & !vbit & column not in a dense block.
// No cell is counted twice (windows are disjoint and skip dense-block and
// vertical columns); every cell of every row is covered.

#include <cuda.h>

#include <cstdlib>

#include "ls_common.cuh"
#include "tc_common.cuh"

namespace ls {
namespace k5ws {

constexpr int BM = 128, BN = 128;
constexpr int N_SOFT = 256;           // softmax threads (8 warps)
constexpr int THREADS = N_SOFT + 128;  // + warpgroup 2: producer warp, MMA warp, two idle warps
constexpr int REGS_SOFT = 224, REGS_CTRL = 56;  // setmaxnreg split: 8 x 232 + 4 x 40 warps' registers <= 64K
constexpr int MAX_KB = 2048;
constexpr int DENSE_SLASHES = 3;
constexpr float RESCALE_LOG2 = 8.f;  // lazy rescale threshold (factor 256)
constexpr int KST = 3, VST = 2;      // K / V ring stages
constexpr int NSB = 3;               // TMEM S / P buffers (+ one O accumulator: 512 columns)
#ifndef LS_K5_POLY
#define LS_K5_POLY 0
#endif

struct Params {
  const int32_t *slash_ids, *vert_ids, *counts;
  const uint32_t *vbits, *rsbits;
  int32_t *diag_ws;  // [H * n_qtiles][n_total]
  const uint16_t *v;  // archive V (diagonal fallback reads)
  int n_heads, group, n_new, n_total, row_offset, words, n_qtiles, dense;
  int64_t kv_head_stride;
  int64_t out_row_stride;  // elements between output rows
  float scale_log2;
  void *out;
  int out_bf16;
  long long *cells;
  long long *tiles;  // optional: tensor-core tiles executed per head (NULL: not counted)
  float *row_lse;    // optional [H][n_new]: log2-sum-exp2 of each row's plan cells (-inf: diagonal fallback)
  int *dbg;  // optional host-mapped progress record [CTA][16] (ls_debug_set_buffer)
  int32_t *status;  // device validation word (EmptyPlan)
};

// progress note of a role (0 producer, 1 MMA, 2 softmax, 3 tile counts) before a wait
#define KDBG(role, tile, code)                                                          \
  do {                                                                                  \
    if (p.dbg) {                                                                        \
      volatile int *d_ = p.dbg + (blockIdx.y * gridDim.x + blockIdx.x) * 16 + (role)*4; \
      d_[0] = (tile);                                                                   \
      d_[1] = (code);                                                                   \
      __threadfence_system();                                                           \
    }                                                                                   \
  } while (0)

template <int D>
struct Smem {
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int KV_BYTES = BN * D * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = Q_BYTES;                   // KST stages
  static constexpr int OFF_V = OFF_K + KST * KV_BYTES;    // VST stages
  static constexpr int OFF_MISC = OFF_V + VST * KV_BYTES;  // (P lives in TMEM, aliasing its S buffer)
  // misc: barriers 256 | ints 256 | kb_bits 256 | pmax 1024 | pd 1024 | lx 512 | gcols 1024 | dense_list 4096 | blk_cnt 8192
  static constexpr int MISC_BYTES = 256 + 256 + 256 + 1024 + 1024 + 512 + 1024 + MAX_KB * 2 + MAX_KB * 4;
  static constexpr int TOTAL = OFF_MISC + MISC_BYTES + 1024;
};

struct Bars {
  uint64_t kfull[KST], kempty[KST], vfull[VST], vempty[VST], s_full[NSB], p_full[NSB], pv_done[2], q_full;
};

__device__ __forceinline__ bool bit_of(const uint32_t *b, int i) { return (b[i >> 5] >> (i & 31)) & 1u; }

__device__ __forceinline__ void bit_window(const uint32_t *bits, int s, uint32_t *w, int n) {
  const int w0 = s >> 5, sh = s & 31;
  uint32_t x[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) x[i] = __ldg(bits + w0 + i);
#pragma unroll
  for (int i = 0; i < 2; ++i) w[i] = __funnelshift_r(x[i], x[i + 1], sh);
  (void)n;
}

// 128 bits of `bits` starting at bit s (s >= 0)
__device__ __forceinline__ void bit_window4(const uint32_t *bits, int s, uint32_t *w) {
  const int w0 = s >> 5, sh = s & 31;
  uint32_t x[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) x[i] = __ldg(bits + w0 + i);
#pragma unroll
  for (int i = 0; i < 4; ++i) w[i] = __funnelshift_r(x[i], x[i + 1], sh);
}

template <int D>
__global__ void __launch_bounds__(THREADS, 1)
    vs_attention_ws_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                           const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_kc,
                           const __grid_constant__ CUtensorMap tm_vc, Params p) {
  extern __shared__ unsigned char smem_dyn[];
  using L = Smem<D>;
  constexpr int DH = D / 2;
  unsigned char *smem = tc::align1024(smem_dyn);
  unsigned char *misc = smem + L::OFF_MISC;
  Bars *bars = reinterpret_cast<Bars *>(misc);
  int *sh_int = reinterpret_cast<int *>(misc + 256);                   // [64]
  uint32_t *kb_bits = reinterpret_cast<uint32_t *>(misc + 512);        // [64]
  float *pmax = reinterpret_cast<float *>(misc + 768);                 // [2][128]
  float *pd = reinterpret_cast<float *>(misc + 1792);                  // [2][128]
  float *lx = reinterpret_cast<float *>(misc + 2816);                  // [128]
  int *gcols = reinterpret_cast<int *>(misc + 3328);                   // [2][128]
  int16_t *dense_list = reinterpret_cast<int16_t *>(misc + 4352);      // [MAX_KB]
  int *blk_cnt = reinterpret_cast<int *>(misc + 4352 + MAX_KB * 2);   // [MAX_KB] slash counts, then window starts
  int *wins = blk_cnt;
  uint32_t *tmem_sh = reinterpret_cast<uint32_t *>(misc + 256 + 252);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = blockIdx.y, qt = blockIdx.x;
  const int r0 = qt * BM;
  const int nr = min(BM, p.n_new - r0);
  const int g0 = p.row_offset + r0;
  const int g_hi = g0 + nr - 1;
  const int kv = h / p.group;
  const uint32_t *vbits = p.vbits + static_cast<int64_t>(h) * (p.words + 8);
  const uint32_t *rsbits = p.rsbits + static_cast<int64_t>(h) * (p.words + 8);
  int32_t *sl = p.diag_ws + (static_cast<int64_t>(h) * p.n_qtiles + qt) * p.n_total;

  if (warp == 0) tc::tmem_alloc(tmem_sh, 512);
  if (tid == 0) {
    for (int s = 0; s < KST; ++s) {
      tc::mbar_init(&bars->kfull[s], 1);
      tc::mbar_init(&bars->kempty[s], 1);
    }
    for (int s = 0; s < VST; ++s) {
      tc::mbar_init(&bars->vfull[s], 1);
      tc::mbar_init(&bars->vempty[s], 1);
    }
    for (int s = 0; s < NSB; ++s) {
      tc::mbar_init(&bars->s_full[s], 1);
      tc::mbar_init(&bars->p_full[s], 4);  // one arrival per softmax warp of the tile's warpgroup
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&bars->pv_done[s], 1);
    }
    tc::mbar_init(&bars->q_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < 64; i += THREADS) kb_bits[i] = 0u;
  for (int i = tid; i < MAX_KB; i += THREADS) blk_cnt[i] = 0;
  __syncthreads();

  // ---- tile lists (all threads)
  const int n_kb = g_hi / BN + 1;
  const int n_sl = p.dense ? 0 : p.counts[h * 2 + 0];
  const int n_vt = p.dense ? 0 : p.counts[h * 2 + 1];
  // masked_sparse_attention raises EmptyPlan for a plan with no lines (tensor_ops.py:165-166)
  if (!p.dense && qt == 0 && tid == 0 && n_sl == 0 && n_vt == 0) report_status(p.status, LS_ERR_EMPTY_PLAN);
  const int32_t *S = p.slash_ids + static_cast<int64_t>(h) * p.n_total;
  const int32_t *Vl = p.vert_ids + static_cast<int64_t>(h) * p.n_total;
  if (p.dense) {
    for (int b = tid; b < n_kb; b += THREADS) atomicOr(&kb_bits[b >> 5], 1u << (b & 31));
  } else {
    for (int i = tid; i < n_sl; i += THREADS) {
      const int dd = S[i];
      if (dd > g_hi) break;
      const int c_lo = max(0, g0 - dd), c_hi = g_hi - dd;
      for (int b = c_lo / BN; b <= c_hi / BN; ++b) atomicAdd(&blk_cnt[b], 1);
    }
    __syncthreads();
    for (int b = tid; b < n_kb; b += THREADS)
      if (blk_cnt[b] >= DENSE_SLASHES) atomicOr(&kb_bits[b >> 5], 1u << (b & 31));
  }
  __syncthreads();
  if (tid == 0) {
    int n = 0;
    for (int w = 0; w < (n_kb + 31) / 32; ++w) {
      uint32_t x = kb_bits[w];
      while (x) {
        const int b = __ffs(x) - 1;
        x &= x - 1;
        if (w * 32 + b < n_kb) dense_list[n++] = static_cast<int16_t>(w * 32 + b);
      }
    }
    sh_int[0] = n;
    int lo = 0, hi = n_vt;  // verticals <= g_hi
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (Vl[mid] <= g_hi)
        lo = mid + 1;
      else
        hi = mid;
    }
    sh_int[1] = lo;
  }
  int n_diag = 0;
  if (!p.dense) {
    for (int base = 0; base < n_sl; base += THREADS) {
      const int i = base + tid;
      bool take = false;
      int dd = 0;
      if (i < n_sl) {
        dd = S[i];
        if (dd <= g_hi) {
          const int c_lo = max(0, g0 - dd), c_hi = g_hi - dd;
          for (int b = c_lo / BN; b <= c_hi / BN; ++b) take |= !bit_of(kb_bits, b);
        }
      }
      const unsigned ball = __ballot_sync(0xffffffffu, take);
      __syncthreads();
      if (lane == 0) sh_int[8 + warp] = __popc(ball);
      __syncthreads();
      int before = 0, tot = 0;
      for (int w = 0; w < THREADS / 32; ++w) {
        if (w < warp) before += sh_int[8 + w];
        tot += sh_int[8 + w];
      }
      if (take) sl[n_diag + before + __popc(ball & ((1u << lane) - 1u))] = dd;
      n_diag += tot;
    }
  }
  __syncthreads();  // (blk_cnt is free from here: it becomes the window list)
  if (tid == 0) {
    // isolated slashes in descending d = ascending key start; merge their key
    // ranges and cover them with disjoint 128-key windows
    int n_win = 0, covered = -1;
    for (int i = n_diag - 1; i >= 0; --i) {
      const int dd = sl[i];
      const int lo = max(0, g0 - dd), hi = g_hi - dd;
      if (hi <= covered) continue;
      for (int w = max(lo, covered + 1); w <= hi && n_win < MAX_KB; w += BN) {
        wins[n_win++] = w;
        covered = w + BN - 1;
      }
    }
    sh_int[2] = n_win;
  }
  __syncthreads();
  const int n_dense = sh_int[0];
  const int v_end = sh_int[1];
  const int n_gt = (v_end + BN - 1) / BN;
  const int n_tc = n_dense + n_gt;
  const int n_win = sh_int[2];
  const int n_all = n_tc + n_win;
  if (tid == 0 && p.dbg) {
    volatile int *d_ = p.dbg + (blockIdx.y * gridDim.x + blockIdx.x) * 16 + 12;
    d_[0] = n_dense;
    d_[1] = n_gt;
    d_[2] = n_win;
    d_[3] = 1;
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_sh;
  const uint32_t tmem_o = tmem + NSB * 128;  // S / P buffers in columns [0, 384), O after them

  if (warp >= 8) {
  tc::setmaxnreg_dec<REGS_CTRL>();
  if (warp == 8) {
    // =================================================== TMA producer
    if (lane == 0) {
      tc::prefetch_tmap(&tm_q);
      tc::prefetch_tmap(&tm_k);
      tc::prefetch_tmap(&tm_v);
      tc::prefetch_tmap(&tm_kc);
      tc::prefetch_tmap(&tm_vc);
      tc::mbar_expect_tx(&bars->q_full, L::Q_BYTES);
#pragma unroll
      for (int a = 0; a < D / 64; ++a)
        tc::tma_load_3d(tc::smem_u32(smem + L::OFF_Q + a * BM * 128), &tm_q, &bars->q_full, a * 64, r0, h);
      // tile t's operand rows: (tensor map, row, head)
      auto src = [&](int t, bool v, const CUtensorMap *&m, int &row, int &hh) {
        if (t < n_dense) {
          m = v ? &tm_v : &tm_k, row = dense_list[t] * BN, hh = kv;
        } else if (t < n_tc) {
          m = v ? &tm_vc : &tm_kc, row = (t - n_dense) * BN, hh = h;
        } else {  // window start (>= 0)
          m = v ? &tm_v : &tm_k, row = wins[t - n_tc], hh = kv;
        }
      };
      auto load = [&](int t, bool v) {
        const int st = v ? t % VST : t % KST, nst = v ? VST : KST;
        uint64_t *fullb = v ? &bars->vfull[st] : &bars->kfull[st];
        KDBG(0, t, v ? 11 : 1);
        tc::mbar_wait(v ? &bars->vempty[st] : &bars->kempty[st], ((t / nst) & 1) ^ 1);
        tc::mbar_expect_tx(fullb, L::KV_BYTES);
        const CUtensorMap *m;
        int row, hh;
        src(t, v, m, row, hh);
        const uint32_t dst = tc::smem_u32(smem + (v ? L::OFF_V : L::OFF_K) + st * L::KV_BYTES);
#pragma unroll
        for (int a = 0; a < D / 64; ++a) tc::tma_load_3d(dst + a * BN * 128, m, fullb, a * 64, row, hh);
      };
      if (n_all > 0) load(0, false);
      for (int t = 0; t < n_all; ++t) {
        if (t + 1 < n_all) load(t + 1, false);  // K one tile ahead of V
        load(t, true);
      }
    }
  } else if (warp == 9) {
    // =================================================== MMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC_S = tc::make_idesc(BM, BN, false, false);
      constexpr uint32_t IDESC_O = tc::make_idesc(BM, D, false, true);
      const uint32_t qs = tc::smem_u32(smem + L::OFF_Q);
      KDBG(1, -1, 2);
      tc::mbar_wait(&bars->q_full, 0);
      auto issue_pv = [&](int j) {  // O += P(j) V(j), P(j) bf16 in TMEM over S(j)
        KDBG(1, j, 3);
        tc::mbar_wait(&bars->p_full[j % NSB], (j / NSB) & 1);
        tc::mbar_wait(&bars->vfull[j % VST], (j / VST) & 1);
        tc::fence_after_sync();
        const uint32_t vs = tc::smem_u32(smem + L::OFF_V + (j % VST) * L::KV_BYTES);
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
          const uint64_t bd = tc::make_desc(vs + kk * 2048, BN * 128, 1024);
          tc::mma_bf16_ts(tmem_o, tmem + (j % NSB) * 128 + kk * 8, bd, IDESC_O, (j > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit(&bars->pv_done[j & 1]);
        tc::mma_commit(&bars->vempty[j % VST]);
      };
      // order S(0) S(1) S(2) PV(0) S(3) PV(1) S(4) ...: S(i) overwrites P(i - 3),
      // whose PV was issued before it (the tensor pipe executes one thread's MMAs
      // in order), and a warpgroup's next S(i + 2) is issued before its PV(i)
      for (int i = 0; i < n_all; ++i) {
        const int s = i % NSB;
        KDBG(1, i, 4);
        tc::mbar_wait(&bars->kfull[i % KST], (i / KST) & 1);
        KDBG(1, i, 5);
        tc::fence_after_sync();
        const uint32_t ks = tc::smem_u32(smem + L::OFF_K + (i % KST) * L::KV_BYTES);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t ad = tc::make_desc(qs + (kk >> 2) * (BM * 128) + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = tc::make_desc(ks + (kk >> 2) * (BN * 128) + (kk & 3) * 32, 16, 1024);
          tc::mma_bf16(tmem + s * 128, ad, bd, IDESC_S, kk > 0 ? 1u : 0u);
        }
        tc::mma_commit(&bars->s_full[s]);
        tc::mma_commit(&bars->kempty[i % KST]);
        if (i >= 2) issue_pv(i - 2);
      }
      for (int j = max(0, n_all - 2); j < n_all; ++j) issue_pv(j);
    }
  }
  } else {
    tc::setmaxnreg_inc<REGS_SOFT>();
    // =================================================== softmax warps
    // Warpgroup wg (warps 4 wg .. 4 wg + 3) works on the tiles i with i % 2 ==
    // wg, one thread per row over all 128 columns, so the two groups overlap
    // two tiles. S / P rotate through three TMEM buffers and PV(i) accumulates
    // into one shared O, so a group's next S(i + 2) is issued before its PV(i)
    // and is usually ready when P(i) is done. The lazy-rescale reference of a
    // row (m_ref_sh) is decided tile by tile in tile order: the group of tile i
    // takes the decision of tile i - 1 from the other group (a named barrier
    // per TMEM lane quadrant), raises the reference if its tile max exceeds it
    // by 2^8, and rescales O itself after PV(i - 1) has landed; each group keeps
    // its row-sum partial relative to the last reference it used.
    const int wg = warp >> 2, quad = warp & 3;
    const int row = quad * 32 + lane;
    const int my_g = g0 + row;
    const bool row_ok = row < nr;
    const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
    float *m_ref_sh = lx;  // [128] the row's current reference (log2 units)
    float m_seen = -INFINITY, l = 0.f;  // this group's row-sum partial, relative to m_seen
    int my_cells = 0;
    auto dec_bar = [&](int dst_wg) { return static_cast<uint32_t>(4 + quad * 2 + dst_wg); };
    for (int i = wg; i < n_all; i += 2) {
      const int s = i % NSB;
      const bool gathered = i >= n_dense && i < n_tc;
      uint32_t mk[4];
      if (i >= n_tc) {  // window: slash cells outside dense blocks and verticals
        const int c0 = wins[i - n_tc];
        if (!row_ok) {
          mk[0] = mk[1] = mk[2] = mk[3] = 0u;
        } else {
          uint32_t sw[4], vw[4];
          bit_window4(rsbits, p.n_total - 1 - my_g + c0, sw);
          bit_window4(vbits, c0, vw);
          // columns of the window in dense blocks: [0, split) in block b1, the rest in b1 + 1
          const int b1 = c0 / BN, split = (b1 + 1) * BN - c0;
          const bool d1 = bit_of(kb_bits, b1), d2 = split < BN && b1 + 1 < MAX_KB && bit_of(kb_bits, b1 + 1);
          const int lim = my_g - c0;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int sp = split - 32 * t;
            const uint32_t below = sp >= 32 ? 0xffffffffu : (sp <= 0 ? 0u : ((1u << sp) - 1u));
            const uint32_t dm = (d1 ? below : 0u) | (d2 ? ~below : 0u);
            const int hi = lim - 32 * t;
            const uint32_t causal = hi >= 31 ? 0xffffffffu : (hi < 0 ? 0u : ((2u << hi) - 1u));
            mk[t] = sw[t] & ~vw[t] & ~dm & causal;
          }
        }
      } else if (gathered) {
        // stage this tile's 128 vertical columns (sorted ascending) and the
        // tile-wide mask of columns outside dense blocks; a row's causal part
        // is then a prefix: columns <= g
        uint32_t *cm = reinterpret_cast<uint32_t *>(pd) + wg * 4;
        int *gc = gcols + wg * BN;
        tc::named_sync(2 + wg, 128);  // the previous gathered tile's reads are done
        {
          const int idx = (i - n_dense) * BN + row;
          const int c = idx < v_end ? Vl[idx] : 0x7fffffff;
          gc[row] = c;
          const unsigned b = __ballot_sync(0xffffffffu, c != 0x7fffffff && !bit_of(kb_bits, c / BN));
          if (lane == 0) cm[warp & 3] = b;
        }
        tc::named_sync(2 + wg, 128);
        int n_le;  // gathered columns <= my_g
        if (gc[BN - 1] <= g0) {
          n_le = BN;
        } else {
          int lo = 0, hi = BN;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (gc[mid] <= my_g) lo = mid + 1; else hi = mid;
          }
          n_le = lo;
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int hi = n_le - 32 * t;  // columns of this word below n_le
          const uint32_t causal = hi >= 32 ? 0xffffffffu : (hi <= 0 ? 0u : ((1u << hi) - 1u));
          mk[t] = row_ok ? (cm[t] & causal) : 0u;
        }
      } else {
        const int c0 = dense_list[i] * BN;
        const int lim = my_g - c0;
        if (p.dense || !row_ok) {
          mk[0] = mk[1] = mk[2] = mk[3] = 0xffffffffu;  // (rows past the block are cleared below)
        } else {
          uint32_t sw[4];
          bit_window4(rsbits, p.n_total - 1 - my_g + c0, sw);
#pragma unroll
          for (int t = 0; t < 4; ++t) mk[t] = ((c0 / 32 + t < p.words) ? __ldg(vbits + c0 / 32 + t) : 0u) | sw[t];
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int hi = lim - 32 * t;
          mk[t] &= (!row_ok) ? 0u : (hi >= 31 ? 0xffffffffu : (hi < 0 ? 0u : ((2u << hi) - 1u)));
        }
      }
      my_cells += __popc(mk[0]) + __popc(mk[1]) + __popc(mk[2]) + __popc(mk[3]);
      if (tid == 0) KDBG(2, i, 6);
      tc::mbar_wait(&bars->s_full[s], (i / NSB) & 1);
      tc::fence_after_sync();
      const uint32_t s_addr = tmem + s * 128 + lane_base;
      float sv[4][32];
      bool live[4];
#pragma unroll
      for (int cch = 0; cch < 4; ++cch) {
        live[cch] = __any_sync(0xffffffffu, mk[cch] != 0u);  // warp-uniform: TMEM loads are .sync.aligned
        if (live[cch]) tc::tmem_ld32(s_addr + cch * 32, sv[cch]);
      }
      tc::tmem_wait_ld();
      float tmax = -INFINITY;
#pragma unroll
      for (int cch = 0; cch < 4; ++cch) {
        if (live[cch]) {
          // masked cells become -inf once; max and exp then run unmasked
          // (exp2(-inf) = 0); whole-chunk-valid rows skip the masking
          const uint32_t m = mk[cch];
          if (m != 0xffffffffu) {
#pragma unroll
            for (int j = 0; j < 32; ++j) sv[cch][j] = ((m >> j) & 1u) ? sv[cch][j] : -INFINITY;
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) tmax = fmaxf(tmax, sv[cch][j]);
        }
      }
      const float m_tile = tmax == -INFINITY ? -INFINITY : tmax * p.scale_log2;
      // reference decision of tile i (after the other group's decision of tile i - 1)
      if (i >= 1) tc::named_sync(dec_bar(wg), 64);
      const float m_cur = i >= 1 ? m_ref_sh[row] : -INFINITY;
      const bool need = m_tile > m_cur + RESCALE_LOG2;
      const float m_ref = need ? m_tile : m_cur;
      m_ref_sh[row] = m_ref;
      if (i + 1 < n_all) asm volatile("bar.arrive %0, 64;" ::"r"(dec_bar(1 - wg)) : "memory");
      if (m_ref != m_seen) {  // this group's partial sum follows the reference
        if (m_seen != -INFINITY) l *= fast_exp2(m_seen - m_ref);
        m_seen = m_ref;
      }
      float2 lsum2 = make_float2(0.f, 0.f);
      const float2 sc2 = make_float2(p.scale_log2, p.scale_log2), nm2 = make_float2(-m_ref, -m_ref);
#pragma unroll
      for (int cch = 0; cch < 4; ++cch) {
        uint32_t pk[16];  // P(i) columns [32 cch, +32) as bf16 pairs: TMEM columns s * 128 + 16 cch + [0, 16)
        // a row with no valid cell so far (m_ref = -inf) has P = 0 (and no NaN)
        if (live[cch] && m_ref != -INFINITY) {
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float2 x = ffma2(make_float2(sv[cch][j], sv[cch][j + 1]), sc2, nm2);  // (s * scale - m) per pair
            const float a = fast_exp2(x.x);
            // LS_K5_POLY: share of the exponentials on the FMA pipe (FA4 split): 1 = every 8th, 2 = every 4th
            const bool poly = (LS_K5_POLY == 1 && (j & 14) == 14) || (LS_K5_POLY == 2 && (j & 6) == 6);
            const float b = poly ? poly_exp2(x.y) : fast_exp2(x.y);
            lsum2 = fadd2(lsum2, make_float2(a, b));
            pk[j >> 1] = tc::pack_bf16(a, b);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) pk[j] = 0u;
        }
        // (every S read of this tile finished at the wait::ld above)
        tc::tmem_st16(s_addr + cch * 16, pk);
      }
      tc::tmem_wait_st();
      l += lsum2.x + lsum2.y;
      // a raised reference: O (everything up to PV(i - 1)) to the new reference
      // before PV(i) adds P(i) (TMEM ld/st are .sync.aligned: the whole warp
      // rescales if any of its rows needs it)
      if (__any_sync(0xffffffffu, need && m_cur != -INFINITY)) {
        if (tid == 0) KDBG(2, i, 7);
        tc::mbar_wait(&bars->pv_done[(i - 1) & 1], ((i - 1) >> 1) & 1);
        tc::fence_after_sync();
        const float corr = (need && m_cur != -INFINITY) ? fast_exp2(m_cur - m_tile) : 1.f;
#pragma unroll
        for (int cch = 0; cch < D / 32; ++cch) {
          float ov[32];
          tc::tmem_ld32(tmem_o + lane_base + cch * 32, ov);
          tc::tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) ov[j] *= corr;
          tc::tmem_st32(tmem_o + lane_base + cch * 32, ov);
        }
        tc::tmem_wait_st();
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&bars->p_full[s]);  // one arrival per warp of the group
    }
    // ---- epilogue: O is relative to the final reference; row sums of both groups
    float *lx2 = pd;  // [2][128] (the gathered-tile staging is done)
    tc::named_sync(1, N_SOFT);  // every decision and staging read is done
    const float mm = n_all > 0 ? m_ref_sh[row] : -INFINITY;
    lx2[wg * BM + row] = (m_seen == -INFINITY || mm == -INFINITY) ? 0.f : l * fast_exp2(m_seen - mm);
    // the last PV has landed. (A parity wait on PV(j) needs PV(j - 2) complete: S(n_all - 1),
    // seen complete by its group, follows PV(n_all - 4); PV(n_all - 2) then implies PV(n_all - 3).)
    if (n_all > 1) tc::mbar_wait(&bars->pv_done[(n_all - 2) & 1], ((n_all - 2) >> 1) & 1);
    if (n_all > 0) tc::mbar_wait(&bars->pv_done[(n_all - 1) & 1], ((n_all - 1) >> 1) & 1);
    tc::fence_after_sync();
    tc::named_sync(1, N_SOFT);
    const float l_all = lx2[row] + lx2[BM + row];
    // this thread writes output columns [wg * DH, wg * DH + DH) of its row
    float o[DH];
    if (n_all > 0) {
#pragma unroll
      for (int cch = 0; cch < DH / 32; ++cch) {
        float ov[32];
        tc::tmem_ld32(tmem_o + lane_base + wg * DH + cch * 32, ov);
        tc::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) o[cch * 32 + j] = ov[j];
      }
    } else {
#pragma unroll
      for (int j = 0; j < DH; ++j) o[j] = 0.f;
    }
    if (row_ok && wg == 0 && p.row_lse)  // plan-cell mass of the row on the log2 scale (ls_plan_coverage)
      p.row_lse[static_cast<int64_t>(h) * p.n_new + r0 + row] = l_all > 0.f ? mm + __log2f(l_all) : -INFINITY;
    if (row_ok) {
      const int64_t orow = static_cast<int64_t>(r0 + row) * p.out_row_stride + static_cast<int64_t>(h) * D + wg * DH;
      if (l_all > 0.f) {
        const float inv = 1.f / l_all;
        if (p.out_bf16) {
          uint16_t *dst = reinterpret_cast<uint16_t *>(p.out) + orow;
#pragma unroll
          for (int j = 0; j < DH; j += 8)
            *reinterpret_cast<uint4 *>(dst + j) =
                make_uint4(tc::pack_bf16(o[j] * inv, o[j + 1] * inv), tc::pack_bf16(o[j + 2] * inv, o[j + 3] * inv),
                           tc::pack_bf16(o[j + 4] * inv, o[j + 5] * inv), tc::pack_bf16(o[j + 6] * inv, o[j + 7] * inv));
        } else {
          float *dst = reinterpret_cast<float *>(p.out) + orow;
#pragma unroll
          for (int j = 0; j < DH; j += 4)
            *reinterpret_cast<float4 *>(dst + j) = make_float4(o[j] * inv, o[j + 1] * inv, o[j + 2] * inv, o[j + 3] * inv);
        }
      } else {  // diagonal fallback (tensor_ops.py:136-137)
        const uint16_t *vrow = p.v + static_cast<int64_t>(kv) * p.kv_head_stride + static_cast<int64_t>(my_g) * D + wg * DH;
        for (int j = 0; j < DH; ++j) {
          const float val = bf2f(vrow[j]);
          if (p.out_bf16)
            reinterpret_cast<uint16_t *>(p.out)[orow + j] = f2bf(val);
          else
            reinterpret_cast<float *>(p.out)[orow + j] = val;
        }
        if (wg == 0) my_cells += 1;
      }
    }
    const long long cs = warp_sum_ll(static_cast<long long>(my_cells));
    if (lane == 0 && cs)
      atomicAdd(reinterpret_cast<unsigned long long *>(p.cells + h), static_cast<unsigned long long>(cs));
    if (tid == 0 && p.tiles && n_all)
      atomicAdd(reinterpret_cast<unsigned long long *>(p.tiles + h), static_cast<unsigned long long>(n_all));
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

// compacted selected verticals: kc/vc[h][j] = K/V[kv(h)][vert_ids[h][j]], rows
// [n_vt, round_up(n_vt, 128)) zeroed so that padded tile rows are finite
__global__ void gather_verticals_kernel(const uint16_t *k, const uint16_t *v, const int32_t *vert_ids,
                                        const int32_t *counts, int n_total, int vcap, int group,
                                        int64_t kv_head_stride, int d, uint16_t *kc, uint16_t *vc) {
  const int h = blockIdx.y;
  const int n = counts[h * 2 + 1];
  const int n_pad = min((n + 127) / 128 * 128, vcap);
  const int vec = d / 8;
  const uint4 *ks = reinterpret_cast<const uint4 *>(k + static_cast<int64_t>(h / group) * kv_head_stride);
  const uint4 *vs = reinterpret_cast<const uint4 *>(v + static_cast<int64_t>(h / group) * kv_head_stride);
  uint4 *kd = reinterpret_cast<uint4 *>(kc + static_cast<int64_t>(h) * vcap * d);
  uint4 *vd = reinterpret_cast<uint4 *>(vc + static_cast<int64_t>(h) * vcap * d);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_pad * vec; i += gridDim.x * blockDim.x) {
    const int j = i / vec, e = i % vec;
    if (j < n) {
      const int64_t src = static_cast<int64_t>(vert_ids[static_cast<int64_t>(h) * n_total + j]) * vec + e;
      kd[i] = ks[src];
      vd[i] = vs[src];
    } else {
      kd[i] = make_uint4(0, 0, 0, 0);
      vd[i] = make_uint4(0, 0, 0, 0);
    }
  }
}

__global__ void vert_bits_kernel(const int32_t *vert_ids, const int32_t *counts, int n_total, int words,
                                 uint32_t *vbits) {
  const int h = blockIdx.y;
  const int n = counts[h * 2 + 1];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int c = vert_ids[static_cast<int64_t>(h) * n_total + i];
    atomicOr(vbits + static_cast<int64_t>(h) * (words + 8) + (c >> 5), 1u << (c & 31));
  }
}

__global__ void reverse_bits_kernel(const int32_t *slash_ids, const int32_t *counts, int n_total, int words,
                                    uint32_t *rsbits) {
  const int h = blockIdx.y;
  const int n = counts[h * 2];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int d = slash_ids[static_cast<int64_t>(h) * n_total + i];
    const int x = n_total - 1 - d;
    atomicOr(rsbits + static_cast<int64_t>(h) * (words + 8) + (x >> 5), 1u << (x & 31));
  }
}

}  // namespace k5ws

// ------------------------------------------------------------------ host
int *g_debug_buffer = nullptr;  // ls_debug_set_buffer (host-mapped), read by the pipelined kernels

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

// bf16 [heads][rows][d] with explicit strides; box = 64 columns x 128 rows
int make_tmap_bf16_3d_box(CUtensorMap *m, const void *base, int d, int64_t rows, int heads, int64_t row_stride_el,
                          int64_t head_stride_el, int box_rows);
int make_tmap_bf16_3d(CUtensorMap *m, const void *base, int d, int64_t rows, int heads, int64_t row_stride_el,
                      int64_t head_stride_el) {
  return make_tmap_bf16_3d_box(m, base, d, rows, heads, row_stride_el, head_stride_el, 128);
}

int make_tmap_bf16_3d_box(CUtensorMap *m, const void *base, int d, int64_t rows, int heads, int64_t row_stride_el,
                          int64_t head_stride_el, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  LS_REQUIRE(fn != nullptr, LS_ERR_CUDA, "cuTensorMapEncodeTiled is unavailable");
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(heads)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(row_stride_el * 2), static_cast<cuuint64_t>(head_stride_el * 2)};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  LS_REQUIRE(r == CUDA_SUCCESS, LS_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return LS_OK;
}

size_t vs_attention_ws_workspace(const ls_layer_desc *L) {
  const size_t words = (L->n_total + 31) / 32;
  const size_t nqt = (L->n_new + k5ws::BM - 1) / k5ws::BM;
  const size_t H = L->n_heads;
  return H * ((words + 8) * 4 + (words + 8) * 4) + nqt * H * L->n_total * 4 +
         2 * H * (static_cast<size_t>(L->n_total) + 128) * L->head_dim * 2 + 8 * 256;
}

int vs_attention_ws(const ls_layer_desc *L, const uint16_t *q, const uint16_t *k, const uint16_t *v,
                    const int32_t *slash_ids, const int32_t *vert_ids, const int32_t *counts, void *out,
                    int32_t out_bf16, int64_t *cells, int64_t *tiles, int dense, void *ws, size_t ws_bytes,
                    cudaStream_t st, float *row_lse) {
  LS_REQUIRE(L->head_dim == 64 || L->head_dim == 128, LS_ERR_UNSUPPORTED, "head_dim must be 64 or 128");
  LS_REQUIRE((L->n_total + k5ws::BN - 1) / k5ws::BN <= k5ws::MAX_KB, LS_ERR_UNSUPPORTED, "n_total too large");
  LS_REQUIRE(dense || ws_bytes >= vs_attention_ws_workspace(L), LS_ERR_WORKSPACE, "vs_attention workspace too small");
  const int H = L->n_heads, d = L->head_dim;
  const int words = (L->n_total + 31) / 32;
  const int nqt = (L->n_new + k5ws::BM - 1) / k5ws::BM;
  Carver c(ws, ws_bytes);
  uint32_t *vbits = c.take<uint32_t>(static_cast<size_t>(H) * (words + 8));
  uint32_t *rsbits = c.take<uint32_t>(static_cast<size_t>(H) * (words + 8));
  int32_t *diag = c.take<int32_t>(static_cast<size_t>(nqt) * H * L->n_total);
  const size_t vcap = static_cast<size_t>(L->n_total) + 128;
  uint16_t *kc = c.take<uint16_t>(static_cast<size_t>(H) * vcap * d);
  uint16_t *vc = c.take<uint16_t>(static_cast<size_t>(H) * vcap * d);
  if (!dense) {
    // vbits and rsbits are consecutive in the workspace: one memset
    LS_CUDA(cudaMemsetAsync(vbits, 0, reinterpret_cast<char *>(rsbits + static_cast<size_t>(H) * (words + 8)) -
                                          reinterpret_cast<char *>(vbits), st));
    k5ws::vert_bits_kernel<<<dim3(4, H), 256, 0, st>>>(vert_ids, counts, L->n_total, words, vbits);
    k5ws::reverse_bits_kernel<<<dim3(4, H), 256, 0, st>>>(slash_ids, counts, L->n_total, words, rsbits);
    k5ws::gather_verticals_kernel<<<dim3(32, H), 256, 0, st>>>(k, v, vert_ids, counts, L->n_total,
                                                               static_cast<int>(vcap), H / L->n_kv_heads,
                                                               L->kv_head_stride, d, kc, vc);
    LS_LAUNCH_CHECK("vs_attention_ws prep");
  }
  CUtensorMap tq, tk, tv, tkc, tvc;
  int s;
  if ((s = make_tmap_bf16_3d(&tq, q, d, L->n_new, H, d, L->q_head_stride))) return s;
  if ((s = make_tmap_bf16_3d(&tk, k, d, L->n_total, L->n_kv_heads, d, L->kv_head_stride))) return s;
  if ((s = make_tmap_bf16_3d(&tv, v, d, L->n_total, L->n_kv_heads, d, L->kv_head_stride))) return s;
  if (dense) {  // no gathered tiles: any valid map will do
    tkc = tk;
    tvc = tv;
  } else {
    if ((s = make_tmap_bf16_3d(&tkc, kc, d, static_cast<int64_t>(vcap), H, d, static_cast<int64_t>(vcap) * d)))
      return s;
    if ((s = make_tmap_bf16_3d(&tvc, vc, d, static_cast<int64_t>(vcap), H, d, static_cast<int64_t>(vcap) * d)))
      return s;
  }
  k5ws::Params p;
  p.slash_ids = slash_ids;
  p.vert_ids = vert_ids;
  p.counts = counts;
  p.vbits = vbits;
  p.rsbits = rsbits;
  p.diag_ws = diag;
  p.v = v;
  p.n_heads = H;
  p.out_row_stride = L->out_row_stride ? L->out_row_stride : static_cast<int64_t>(H) * d;
  p.group = H / L->n_kv_heads;
  p.n_new = L->n_new;
  p.n_total = L->n_total;
  p.row_offset = L->row_offset;
  p.words = words;
  p.n_qtiles = nqt;
  p.dense = dense;
  p.kv_head_stride = L->kv_head_stride;
  p.scale_log2 = kLog2e / sqrtf(static_cast<float>(d));
  p.out = out;
  p.out_bf16 = out_bf16;
  p.cells = reinterpret_cast<long long *>(cells);
  p.tiles = reinterpret_cast<long long *>(tiles);
  p.row_lse = row_lse;
  p.dbg = g_debug_buffer;
  p.status = device_status_ptr();
  LS_CUDA(cudaMemsetAsync(cells, 0, sizeof(int64_t) * H, st));
  if (tiles) LS_CUDA(cudaMemsetAsync(tiles, 0, sizeof(int64_t) * H, st));
  dim3 grid(nqt, H);
  if (d == 128) {
    const int smem = k5ws::Smem<128>::TOTAL;
    LS_CUDA(cudaFuncSetAttribute(k5ws::vs_attention_ws_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k5ws::vs_attention_ws_kernel<128><<<grid, k5ws::THREADS, smem, st>>>(tq, tk, tv, tkc, tvc, p);
  } else {
    const int smem = k5ws::Smem<64>::TOTAL;
    LS_CUDA(cudaFuncSetAttribute(k5ws::vs_attention_ws_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k5ws::vs_attention_ws_kernel<64><<<grid, k5ws::THREADS, smem, st>>>(tq, tk, tv, tkc, tvc, p);
  }
  LS_LAUNCH_CHECK("vs_attention_ws_kernel");
  return LS_OK;
}

}  // namespace ls

extern "C" int ls_debug_set_buffer(void *host_mapped) {
  ls::g_debug_buffer = static_cast<int *>(host_mapped);
  return LS_OK;
}
