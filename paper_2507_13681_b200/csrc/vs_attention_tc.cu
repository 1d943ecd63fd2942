// K5 (tensor-core path) -- vertical/slash sparse attention on tcgen05 / TMEM.
//
// Same contract as the CUDA-core kernel in vs_attention.cu (reference
// masked_sparse_attention, tensor_ops.py:141-183 with `_row_columns`,
// tensor_ops.py:130-138): per (head, 128-row q tile) the CTA walks
//   * key blocks (BN = 128) touched by a selected slash, mask
//     causal & (vbit[c] | sbit[g - c]), and
//   * gathered tiles of selected verticals outside those blocks, mask causal,
// with S = Q K^T and O_tile = P V on the 5th-gen tensor cores:
//   Q, K, V, P staged in shared memory in the 128B-swizzled UMMA layouts
//   (tc_common.cuh), K/V tiles double-buffered with cp.async (gathers are
//   row-granular, so TMA tiled copies do not apply), accumulators in TMEM
//   (S: 128 columns, O_tile: D columns), one elected thread issues
//   tcgen05.mma and commits to an mbarrier; 128 softmax threads own one TMEM
//   lane (= one q row) each: masked online softmax in fp32 (log2 domain),
//   P rounded to bf16 into shared memory, O accumulated in registers.
// Rows with no selected cell fall back to the diagonal (out = V[g]).
// The per-row popcount of the mask is the OpCounter increment
// (tensor_ops.py:172-174).

#include "ls_common.cuh"
#include "tc_common.cuh"

namespace ls {
namespace k5tc {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int THREADS = 256;  // two warpgroups split S / O columns of the same 128 rows
constexpr int MAX_KB = 2048;  // key blocks per head (n_total <= 262144)
constexpr int DENSE_SLASHES = 3;  // slashes crossing a key block before it goes to the tensor cores

struct Params {
  const uint16_t *q, *k, *v;
  const int32_t *slash_ids, *vert_ids, *counts;
  const uint32_t *vbits;   // [H][words]
  const uint32_t *rsbits;  // [H][words + 8] reversed slash bits: bit i = sbit[n_total-1-i]
  int32_t *gather_ws;      // [n_qtiles * H][n_total]
  int n_heads, group, n_new, n_total, row_offset, words, n_qtiles;
  int64_t q_head_stride, kv_head_stride;
  float scale_log2;
  void *out;
  int out_bf16;
  long long *cells;
  int dense;
};

template <int D>
struct Smem {
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int KV_BYTES = BN * D * 2;
  static constexpr int P_BYTES = BM * BN * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K0 = OFF_Q + Q_BYTES;
  static constexpr int OFF_V0 = OFF_K0 + 2 * KV_BYTES;
  static constexpr int OFF_P = OFF_V0 + 2 * KV_BYTES;
  static constexpr int OFF_MISC = OFF_P + P_BYTES;
  static constexpr int MISC_BYTES = 1536 + MAX_KB * 2 + 2 * BN * 4 + BM * 4 + MAX_KB * 4 + 64;
  static constexpr int TOTAL = OFF_MISC + MISC_BYTES + 1024;  // + alignment slack
};

__device__ __forceinline__ void cp_async16_zfill(uint32_t saddr, const void *gptr, bool valid) {
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(gptr), "r"(n) : "memory");
}

// 128-bit window of a bit array starting at bit `s` (bits beyond the array read as 0 if padded)
__device__ __forceinline__ void bit_window(const uint32_t *bits, int s, uint32_t *w) {
  const int w0 = s >> 5, sh = s & 31;
  uint32_t x[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) x[i] = __ldg(bits + w0 + i);
#pragma unroll
  for (int i = 0; i < 4; ++i) w[i] = __funnelshift_r(x[i], x[i + 1], sh);
}

template <int D>
__global__ void __launch_bounds__(THREADS, 1) vs_attention_tc_kernel(Params p) {
  extern __shared__ unsigned char smem_dyn[];
  using L = Smem<D>;
  constexpr int DH = D / 2;  // O columns per warpgroup
  unsigned char *smem =
      reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  unsigned char *misc = smem + L::OFF_MISC;
  uint64_t *mbar = reinterpret_cast<uint64_t *>(misc);          // [0,1] S buffers, [2] O
  uint32_t *tmem_base_sh = reinterpret_cast<uint32_t *>(misc + 32);
  int *sh_int = reinterpret_cast<int *>(misc + 64);              // scratch ints [32]
  uint32_t *kb_bits = reinterpret_cast<uint32_t *>(misc + 256);  // [64] bitmap of touched key blocks
  float *pmax = reinterpret_cast<float *>(misc + 512);           // [2][128] partial row maxima
  int16_t *dense_list = reinterpret_cast<int16_t *>(misc + 1536);
  int *gcols = reinterpret_cast<int *>(misc + 1536 + MAX_KB * 2);  // [2][BN] columns per buffer
  float *lsum_sh = reinterpret_cast<float *>(misc + 1536 + MAX_KB * 2 + 2 * BN * 4);  // [128]
  int *blk_cnt = reinterpret_cast<int *>(misc + 1536 + MAX_KB * 2 + 2 * BN * 4 + BM * 4);  // [MAX_KB]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wg = warp >> 2;          // column half of S / O handled by this thread
  const int row = (warp & 3) * 32 + lane;  // TMEM lane = q row
  const int h = blockIdx.y, qt = blockIdx.x;
  const int r0 = qt * BM;
  const int nr = min(BM, p.n_new - r0);
  const int g0 = p.row_offset + r0;
  const int g_hi = g0 + nr - 1;
  const int kv = h / p.group;
  const uint16_t *qb = p.q + static_cast<int64_t>(h) * p.q_head_stride;
  const uint16_t *kb = p.k + static_cast<int64_t>(kv) * p.kv_head_stride;
  const uint16_t *vb = p.v + static_cast<int64_t>(kv) * p.kv_head_stride;
  const uint32_t *vbits = p.vbits + static_cast<int64_t>(h) * p.words;
  const uint32_t *rsbits = p.rsbits + static_cast<int64_t>(h) * (p.words + 8);
  int32_t *gl = p.gather_ws + (static_cast<int64_t>(h) * p.n_qtiles + qt) * 2 * p.n_total;

  // ---- TMEM (S double buffer + O tile), barriers, Q tile
  if (warp == 0) tc::tmem_alloc(tmem_base_sh, 512);
  if (tid == 0) {
    tc::mbar_init(&mbar[0], 1);
    tc::mbar_init(&mbar[1], 1);
    tc::mbar_init(&mbar[2], 1);
  }
  for (int i = tid; i < 64; i += THREADS) kb_bits[i] = 0u;
  for (int i = tid; i < MAX_KB; i += THREADS) blk_cnt[i] = 0;
  {
    const uint32_t qs = tc::smem_u32(smem + L::OFF_Q);
    constexpr int CH = D / 8;
    for (int i = tid; i < BM * CH; i += THREADS) {
      const int r = i / CH, c = i % CH;
      const bool ok = r < nr;
      cp_async16_zfill(qs + tc::sw128_offset(r, c, BM), qb + static_cast<int64_t>(ok ? r0 + r : 0) * D + c * 8, ok);
    }
    tc::cp_async_commit();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_base_sh;
  const uint32_t tmem_o = tmem + 256;  // columns [256, 256 + D)

  // ---- tile list: touched key blocks, then gathered verticals
  const int n_kb = g_hi / BN + 1;
  const int n_sl = p.dense ? 0 : p.counts[h * 2 + 0];
  const int n_vt = p.dense ? 0 : p.counts[h * 2 + 1];
  const int32_t *S = p.slash_ids + static_cast<int64_t>(h) * p.n_total;
  const int32_t *V = p.vert_ids + static_cast<int64_t>(h) * p.n_total;
  if (p.dense) {
    for (int b = tid; b < n_kb; b += THREADS) atomicOr(&kb_bits[b >> 5], 1u << (b & 31));
  } else {
    // a key block goes to the tensor cores when >= DENSE_SLASHES slashes cross it;
    // the other slash cells take the CUDA-core diagonal path below
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
  }
  int n_g = 0;  // gathered verticals (ascending): V entries <= g_hi whose block is untouched
  if (!p.dense && n_vt > 0) {
    int lo = 0, hi = n_vt;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (V[mid] <= g_hi)
        lo = mid + 1;
      else
        hi = mid;
    }
    const int v_end = lo;
    for (int base = 0; base < v_end; base += THREADS) {
      const int i = base + tid;
      const int c = i < v_end ? V[i] : 0;
      const bool take = i < v_end && !((kb_bits[(c / BN) >> 5] >> ((c / BN) & 31)) & 1u);
      const unsigned ball = __ballot_sync(0xffffffffu, take);
      __syncthreads();
      if (lane == 0) sh_int[8 + warp] = __popc(ball);
      __syncthreads();
      int before = 0, tot = 0;
      for (int w = 0; w < THREADS / 32; ++w) {
        if (w < warp) before += sh_int[8 + w];
        tot += sh_int[8 + w];
      }
      if (take) gl[n_g + before + __popc(ball & ((1u << lane) - 1u))] = c;
      n_g += tot;
    }
  }
  // diagonal slashes: selected slashes crossing at least one non-tensor block
  int32_t *sl = gl + p.n_total;
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
          for (int b = c_lo / BN; b <= c_hi / BN; ++b) take |= !((kb_bits[b >> 5] >> (b & 31)) & 1u);
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
  __syncthreads();
  const int n_dense = sh_int[0];
  const int n_tiles = n_dense + (n_g + BN - 1) / BN;

  const int my_g = g0 + row;
  const bool row_ok = row < nr;
  float m = -INFINITY, l = 0.f;
  float o[DH];
#pragma unroll
  for (int i = 0; i < DH; ++i) o[i] = 0.f;
  long long my_cells = 0;

  constexpr uint32_t IDESC_S = tc::make_idesc(BM, BN, false, false);
  constexpr uint32_t IDESC_O = tc::make_idesc(BM, D, false, true);
  const uint32_t q_s = tc::smem_u32(smem + L::OFF_Q);
  const uint32_t p_s = tc::smem_u32(smem + L::OFF_P);
  const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;

  // K / V rows of tile i into buffer `buf` (two threads per key row: K and V)
  auto issue_load = [&](int i, int buf) {
    const int r = tid & (BN - 1);
    const bool is_v = tid >= BN;
    int c;
    bool ok;
    if (i < n_dense) {
      c = dense_list[i] * BN + r;
      ok = c < p.n_total;
    } else {
      const int j = (i - n_dense) * BN + r;
      ok = j < n_g;
      c = ok ? gl[j] : 0x7fffffff;
    }
    if (!is_v) gcols[buf * BN + r] = c;
    const int cc = ok ? c : 0;
    const uint32_t dst = tc::smem_u32(smem + (is_v ? L::OFF_V0 : L::OFF_K0) + buf * L::KV_BYTES);
    const uint16_t *src = (is_v ? vb : kb) + static_cast<int64_t>(cc) * D;
    constexpr int CH = D / 8;
#pragma unroll
    for (int ch = 0; ch < CH; ++ch) cp_async16_zfill(dst + tc::sw128_offset(r, ch, BN), src + ch * 8, ok);
    tc::cp_async_commit();
  };
  auto issue_s = [&](int buf) {  // S[buf] = Q K[buf]^T (thread 0)
    const uint32_t ks = tc::smem_u32(smem + L::OFF_K0 + buf * L::KV_BYTES);
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      const uint64_t ad = tc::make_desc(q_s + (kk >> 2) * (BM * 128) + (kk & 3) * 32, 16, 1024);
      const uint64_t bd = tc::make_desc(ks + (kk >> 2) * (BN * 128) + (kk & 3) * 32, 16, 1024);
      tc::mma_bf16(tmem + buf * 128, ad, bd, IDESC_S, kk > 0);
    }
    tc::mma_commit(&mbar[buf]);
  };

  uint32_t ph_s0 = 0, ph_s1 = 0, ph_o = 0;
  if (n_tiles > 0) {
    issue_load(0, 0);
    tc::cp_async_wait<0>();
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (tid == 0) issue_s(0);
    if (n_tiles > 1) issue_load(1, 1);
  }
  for (int i = 0; i < n_tiles; ++i) {
    const int buf = i & 1;
    // ---- mask of (row, this thread's 64 columns) -- overlaps the S MMA
    const bool gathered = i >= n_dense;
    uint32_t mk[2];
    if (!row_ok) {
      mk[0] = mk[1] = 0u;
    } else if (!gathered) {
      const int c0 = dense_list[i] * BN + wg * 64;
      const int lim = my_g - c0;
      if (p.dense) {
        mk[0] = mk[1] = 0xffffffffu;
      } else {
        uint32_t sw[4];
        bit_window(rsbits, p.n_total - 1 - my_g + c0, sw);
#pragma unroll
        for (int t = 0; t < 2; ++t) mk[t] = ((c0 / 32 + t < p.words) ? __ldg(vbits + c0 / 32 + t) : 0u) | sw[t];
      }
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int hi = lim - 32 * t;
        mk[t] &= hi >= 31 ? 0xffffffffu : (hi < 0 ? 0u : ((2u << hi) - 1u));
      }
    } else {
      const int *gc = gcols + buf * BN;
      int lo = 0, hi = BN;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (gc[mid] <= my_g)
          lo = mid + 1;
        else
          hi = mid;
      }
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int nb = lo - wg * 64 - 32 * t;
        mk[t] = nb >= 32 ? 0xffffffffu : (nb <= 0 ? 0u : ((1u << nb) - 1u));
      }
    }
    my_cells += __popc(mk[0]) + __popc(mk[1]);
    // ---- S ready
    if (buf) {
      tc::mbar_wait(&mbar[1], ph_s1);
      ph_s1 ^= 1;
    } else {
      tc::mbar_wait(&mbar[0], ph_s0);
      ph_s0 ^= 1;
    }
    tc::fence_after_sync();
    const uint32_t s_addr = tmem + buf * 128 + lane_base + wg * 64;
    float tmax = -INFINITY;
#pragma unroll
    for (int cch = 0; cch < 2; ++cch) {
      float sv[32];
      tc::tmem_ld32(s_addr + cch * 32, sv);
      tc::tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) tmax = fmaxf(tmax, ((mk[cch] >> j) & 1u) ? sv[j] : -INFINITY);
    }
    pmax[wg * BM + row] = tmax;
    __syncthreads();
    const float tm = fmaxf(pmax[row], pmax[BM + row]);
    const float m_new = fmaxf(m, tm == -INFINITY ? -INFINITY : tm * p.scale_log2);
    const float corr = (m_new == -INFINITY) ? 1.f : fast_exp2(m - m_new);
    float lsum = 0.f;
#pragma unroll
    for (int cch = 0; cch < 2; ++cch) {
      float sv[32];
      tc::tmem_ld32(s_addr + cch * 32, sv);
      tc::tmem_wait_ld();
      uint32_t pk[16];
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const float a = ((mk[cch] >> j) & 1u) ? fast_exp2(fmaf(sv[j], p.scale_log2, -m_new)) : 0.f;
        const float b = ((mk[cch] >> (j + 1)) & 1u) ? fast_exp2(fmaf(sv[j + 1], p.scale_log2, -m_new)) : 0.f;
        lsum += a + b;
        pk[j >> 1] = tc::pack_bf16(a, b);
      }
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const int chunk = wg * 8 + cch * 4 + q4;  // 16-byte chunk along keys
        *reinterpret_cast<uint4 *>(smem + L::OFF_P + tc::sw128_offset(row, chunk, BM)) =
            make_uint4(pk[q4 * 4 + 0], pk[q4 * 4 + 1], pk[q4 * 4 + 2], pk[q4 * 4 + 3]);
      }
    }
    l = l * corr + lsum;
    m = m_new;
    // next tile's K/V must have landed before its S MMA is issued
    if (i + 1 < n_tiles) tc::cp_async_wait<0>();
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (tid == 0) {
      const uint32_t vs = tc::smem_u32(smem + L::OFF_V0 + buf * L::KV_BYTES);
#pragma unroll
      for (int kk = 0; kk < BN / 16; ++kk) {
        const uint64_t ad = tc::make_desc(p_s + (kk >> 2) * (BM * 128) + (kk & 3) * 32, 16, 1024);
        const uint64_t bd = tc::make_desc(vs + kk * 2048, BN * 128, 1024);
        tc::mma_bf16(tmem_o, ad, bd, IDESC_O, kk > 0);
      }
      tc::mma_commit(&mbar[2]);
      if (i + 1 < n_tiles) issue_s(buf ^ 1);  // queued behind PV: overlaps the O update below
    }
    tc::mbar_wait(&mbar[2], ph_o);
    ph_o ^= 1;
    tc::fence_after_sync();
#pragma unroll
    for (int cch = 0; cch < DH / 32; ++cch) {
      float ov[32];
      tc::tmem_ld32(tmem_o + lane_base + wg * DH + cch * 32, ov);
      tc::tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) o[cch * 32 + j] = fmaf(o[cch * 32 + j], corr, ov[j]);
    }
    tc::fence_before_sync();
    // K/V buffer `buf` is free (S(i) and PV(i) done): prefetch tile i + 2
    if (i + 2 < n_tiles) issue_load(i + 2, buf);
  }
  tc::cp_async_wait<0>();

  // ---- diagonal slash cells on CUDA cores: cells of `sl` slashes whose column
  // is in a non-tensor block and is not a selected vertical (those cells were
  // covered above). Thread (row, wg) owns half of the head dim; the partial
  // dot products of a batch of DB slashes are exchanged through shared memory.
  if (n_diag > 0) {
    constexpr int DB = 8;
    float *part = reinterpret_cast<float *>(smem + L::OFF_P);  // [2][DB][BM] (P buffer is free now)
    float qf[DH];
#pragma unroll
    for (int c8 = 0; c8 < DH / 8; ++c8) {
      const uint4 u =
          *reinterpret_cast<const uint4 *>(smem + L::OFF_Q + tc::sw128_offset(row, wg * (DH / 8) + c8, BM));
      bf16x8_to_f32(u, qf + c8 * 8);
    }
    for (int base = 0; base < n_diag; base += DB) {
      int cj[DB];
      bool vj[DB];
#pragma unroll
      for (int j = 0; j < DB; ++j) {
        const int idx = base + j;
        const int c = my_g - (idx < n_diag ? sl[idx] : 0x3fffffff);
        bool v = row_ok && idx < n_diag && c >= 0;
        if (v) {
          const int b = c / BN;
          v = !((kb_bits[b >> 5] >> (b & 31)) & 1u) && !((__ldg(vbits + (c >> 5)) >> (c & 31)) & 1u);
        }
        cj[j] = c;
        vj[j] = v;
        float acc = 0.f;
        if (v) {
          const uint16_t *kr = kb + static_cast<int64_t>(c) * D + wg * DH;
#pragma unroll
          for (int c8 = 0; c8 < DH / 8; ++c8) {
            float f[8];
            bf16x8_to_f32(*reinterpret_cast<const uint4 *>(kr + c8 * 8), f);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc = fmaf(qf[c8 * 8 + e], f[e], acc);
          }
        }
        part[(wg * DB + j) * BM + row] = acc;
      }
      __syncthreads();
      float sc[DB];
      float bmax = -INFINITY;
#pragma unroll
      for (int j = 0; j < DB; ++j) {
        sc[j] = vj[j] ? (part[j * BM + row] + part[(DB + j) * BM + row]) * p.scale_log2 : -INFINITY;
        bmax = fmaxf(bmax, sc[j]);
      }
      __syncthreads();  // `part` is rewritten by the next batch
      if (bmax != -INFINITY) {
        const float m_new = fmaxf(m, bmax);
        const float corr = fast_exp2(m - m_new);  // 0 when m == -inf
        float lsum = 0.f;
#pragma unroll
        for (int i = 0; i < DH; ++i) o[i] *= corr;
#pragma unroll
        for (int j = 0; j < DB; ++j) {
          if (!vj[j]) continue;
          const float pj = fast_exp2(sc[j] - m_new);
          lsum += pj;
          const uint16_t *vr = vb + static_cast<int64_t>(cj[j]) * D + wg * DH;
#pragma unroll
          for (int c8 = 0; c8 < DH / 8; ++c8) {
            float f[8];
            bf16x8_to_f32(*reinterpret_cast<const uint4 *>(vr + c8 * 8), f);
#pragma unroll
            for (int e = 0; e < 8; ++e) o[c8 * 8 + e] = fmaf(pj, f[e], o[c8 * 8 + e]);
          }
          if (wg == 0) my_cells += 1;
        }
        l = l * corr + (wg == 0 ? lsum : 0.f);  // each cell's p is counted once (warpgroup 0)
        m = m_new;
      }
    }
  }

  // ---- epilogue: l = sum of both halves
  lsum_sh[row] = 0.f;
  __syncthreads();
  if (wg == 1) lsum_sh[row] = l;
  __syncthreads();
  const float l_tot = l + (wg == 0 ? lsum_sh[row] : 0.f);
  __syncthreads();
  if (wg == 0) lsum_sh[row] = l_tot;
  __syncthreads();
  const float l_all = lsum_sh[row];
  if (row_ok) {
    const int64_t orow = (static_cast<int64_t>(r0 + row) * p.n_heads + h) * D + wg * DH;
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
      for (int j = 0; j < DH; ++j) {
        const float val = bf2f(vb[static_cast<int64_t>(my_g) * D + wg * DH + j]);
        if (p.out_bf16)
          reinterpret_cast<uint16_t *>(p.out)[orow + j] = f2bf(val);
        else
          reinterpret_cast<float *>(p.out)[orow + j] = val;
      }
      if (wg == 0) my_cells += 1;
    }
  }
  const long long cs = warp_sum_ll(my_cells);
  if (lane == 0 && cs)
    atomicAdd(reinterpret_cast<unsigned long long *>(p.cells + h), static_cast<unsigned long long>(cs));
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

__global__ void vert_bits_kernel(const int32_t *vert_ids, const int32_t *counts, int n_total, int words,
                                 uint32_t *vbits) {
  const int h = blockIdx.y;
  const int n = counts[h * 2 + 1];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int c = vert_ids[static_cast<int64_t>(h) * n_total + i];
    atomicOr(vbits + static_cast<int64_t>(h) * words + (c >> 5), 1u << (c & 31));
  }
}

// reversed slash bitmap: bit i = sbit[n_total - 1 - i]
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

}  // namespace k5tc
}  // namespace ls

using namespace ls;

namespace ls {
size_t vs_attention_tc_workspace(const ls_layer_desc *L) {
  const size_t words = (L->n_total + 31) / 32;
  const size_t nqt = (L->n_new + k5tc::BM - 1) / k5tc::BM;
  return static_cast<size_t>(L->n_heads) * (words * 4 + (words + 8) * 4) + 2 * nqt * L->n_heads * L->n_total * 4 + 4096;
}

int vs_attention_tc(const ls_layer_desc *L, const uint16_t *q, const uint16_t *k, const uint16_t *v,
                    const int32_t *slash_ids, const int32_t *vert_ids, const int32_t *counts, void *out,
                    int32_t out_bf16, int64_t *cells, int dense, void *ws, size_t ws_bytes, cudaStream_t st) {
  LS_REQUIRE(L->head_dim == 64 || L->head_dim == 128, LS_ERR_UNSUPPORTED, "head_dim must be 64 or 128");
  LS_REQUIRE((L->n_total + k5tc::BN - 1) / k5tc::BN <= k5tc::MAX_KB, LS_ERR_UNSUPPORTED, "n_total too large");
  LS_REQUIRE(dense || ws_bytes >= vs_attention_tc_workspace(L), LS_ERR_WORKSPACE, "vs_attention workspace too small");
  const int words = (L->n_total + 31) / 32;
  const int nqt = (L->n_new + k5tc::BM - 1) / k5tc::BM;
  Carver c(dense ? nullptr : ws, ws_bytes);  // dense mode reads no plan buffers
  uint32_t *vbits = c.take<uint32_t>(static_cast<size_t>(L->n_heads) * words);
  uint32_t *rsbits = c.take<uint32_t>(static_cast<size_t>(L->n_heads) * (words + 8));
  int32_t *gather = c.take<int32_t>(2 * static_cast<size_t>(nqt) * L->n_heads * L->n_total);
  if (!dense) {
    LS_CUDA(cudaMemsetAsync(vbits, 0, sizeof(uint32_t) * L->n_heads * words, st));
    LS_CUDA(cudaMemsetAsync(rsbits, 0, sizeof(uint32_t) * L->n_heads * (words + 8), st));
    k5tc::vert_bits_kernel<<<dim3(4, L->n_heads), 256, 0, st>>>(vert_ids, counts, L->n_total, words, vbits);
    k5tc::reverse_bits_kernel<<<dim3(4, L->n_heads), 256, 0, st>>>(slash_ids, counts, L->n_total, words, rsbits);
    LS_LAUNCH_CHECK("reverse_bits_kernel");
  }
  k5tc::Params p;
  p.q = q;
  p.k = k;
  p.v = v;
  p.slash_ids = slash_ids;
  p.vert_ids = vert_ids;
  p.counts = counts;
  p.vbits = vbits;
  p.rsbits = rsbits;
  p.gather_ws = gather;
  p.n_heads = L->n_heads;
  p.group = L->n_heads / L->n_kv_heads;
  p.n_new = L->n_new;
  p.n_total = L->n_total;
  p.row_offset = L->row_offset;
  p.words = words;
  p.n_qtiles = nqt;
  p.q_head_stride = L->q_head_stride;
  p.kv_head_stride = L->kv_head_stride;
  p.scale_log2 = kLog2e / sqrtf(static_cast<float>(L->head_dim));
  p.out = out;
  p.out_bf16 = out_bf16;
  p.cells = reinterpret_cast<long long *>(cells);
  p.dense = dense;
  LS_CUDA(cudaMemsetAsync(cells, 0, sizeof(int64_t) * L->n_heads, st));
  dim3 grid(nqt, L->n_heads);
  if (L->head_dim == 128) {
    const int smem = k5tc::Smem<128>::TOTAL;
    LS_CUDA(cudaFuncSetAttribute(k5tc::vs_attention_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k5tc::vs_attention_tc_kernel<128><<<grid, k5tc::THREADS, smem, st>>>(p);
  } else {
    const int smem = k5tc::Smem<64>::TOTAL;
    LS_CUDA(cudaFuncSetAttribute(k5tc::vs_attention_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k5tc::vs_attention_tc_kernel<64><<<grid, k5tc::THREADS, smem, st>>>(p);
  }
  LS_LAUNCH_CHECK("vs_attention_tc_kernel");
  return LS_OK;
}
}  // namespace ls
