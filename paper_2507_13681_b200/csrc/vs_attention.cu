// K4 + K5 -- vertical/slash sparse attention with exact cell semantics.
//
// Replaces masked_sparse_attention (reference tensor_ops.py:141-183) and the
// per-row cell set `_row_columns` (tensor_ops.py:130-138):
//   cells(g) = {c in V : c <= g} U {g - d : d in S, d <= g},  {g} if empty,
// softmax over exactly those cells. Layout of the work per (head, q-tile of
// BM rows [g0, g_hi]):
//   * key blocks touched by a selected slash (each slash d covers columns
//     [max(0, g0-d), g_hi-d]) are processed densely with the cell mask
//     causal & (vbit[c] | sbit[g-c]);
//   * selected verticals outside those blocks are gathered into tiles of
//     BN columns (mask: causal only) -- so no cell is counted twice;
//   * online softmax in fp32 (log2 domain), rows with no cell fall back to
//     the diagonal (out = V[g]).
// The per-row cell count is the OpCounter increment of tensor_ops.py:172-174.
// `dense` mode (scaled_dot_attention, tensor_ops.py:104-127) touches every
// causal block with the causal mask only.
//
// This is the CUDA-core path; the tcgen05 path keeps this tiling.

#include "ls_common.cuh"

namespace ls {
namespace k5 {

constexpr int BM = 64;
constexpr int BN = 64;
constexpr int THREADS = 256;  // 4 threads per q row
constexpr int MAX_KB_WORDS = 64;  // key-block bitmap: up to 2048 * BN keys

struct Params {
  const uint16_t *q, *k, *v;
  const int32_t *slash_ids, *vert_ids, *counts;
  const uint32_t *sbits, *vbits;  // [H][words]
  int n_heads, group, d, n_new, n_total, row_offset, words;
  int64_t out_row_stride;
  int64_t q_head_stride, kv_head_stride;
  float scale_log2;
  void *out;
  int out_bf16;
  long long *cells;
  int dense;
};

__device__ __forceinline__ bool bit(const uint32_t *b, int i) { return (b[i >> 5] >> (i & 31)) & 1u; }

__global__ void __launch_bounds__(THREADS) vs_attention_kernel(Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int d = p.d, ld = d + 1;
  float *Qs = reinterpret_cast<float *>(smem_raw);  // [BM][ld]
  float *Ks = Qs + BM * ld;                          // [BN][ld]
  float *Vs = Ks + BN * ld;                          // [BN][d]
  float *Ps = Vs + BN * d;                           // [BM][BN+1]
  uint32_t *kb_bits = reinterpret_cast<uint32_t *>(Ps + BM * (BN + 1));  // [MAX_KB_WORDS]
  int *gcols = reinterpret_cast<int *>(kb_bits + MAX_KB_WORDS);           // [BN] gathered columns
  int *scratch = gcols + BN;                                              // misc

  const int h = blockIdx.y;
  const int r0 = blockIdx.x * BM;
  const int nr = min(BM, p.n_new - r0);
  const int g0 = p.row_offset + r0;
  const int g_hi = g0 + nr - 1;
  const int kv = h / p.group;
  const uint16_t *qb = p.q + static_cast<int64_t>(h) * p.q_head_stride;
  const uint16_t *kb = p.k + static_cast<int64_t>(kv) * p.kv_head_stride;
  const uint16_t *vb = p.v + static_cast<int64_t>(kv) * p.kv_head_stride;
  const uint32_t *sb = p.sbits + static_cast<int64_t>(h) * p.words;
  const uint32_t *vbits = p.vbits + static_cast<int64_t>(h) * p.words;
  const int n_sl = p.dense ? 0 : p.counts[h * 2 + 0];
  const int n_vt = p.dense ? 0 : p.counts[h * 2 + 1];
  const int32_t *S = p.slash_ids + static_cast<int64_t>(h) * p.n_total;
  const int32_t *V = p.vert_ids + static_cast<int64_t>(h) * p.n_total;

  // Q tile
  for (int i = threadIdx.x; i < BM * (d / 8); i += blockDim.x) {
    int r = i / (d / 8), vv = i % (d / 8);
    float f[8];
    if (r < nr) {
      uint4 u = *reinterpret_cast<const uint4 *>(qb + static_cast<int64_t>(r0 + r) * d + vv * 8);
      bf16x8_to_f32(u, f);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) Qs[r * ld + vv * 8 + j] = f[j];
  }
  // touched key blocks
  const int n_kb = g_hi / BN + 1;
  for (int i = threadIdx.x; i < MAX_KB_WORDS; i += blockDim.x) kb_bits[i] = 0u;
  __syncthreads();
  if (p.dense) {
    for (int b = threadIdx.x; b < n_kb; b += blockDim.x) atomicOr(&kb_bits[b >> 5], 1u << (b & 31));
  } else {
    for (int i = threadIdx.x; i < n_sl; i += blockDim.x) {
      const int dd = S[i];
      if (dd > g_hi) break;  // sorted ascending
      const int c_lo = max(0, g0 - dd), c_hi = g_hi - dd;
      for (int b = c_lo / BN; b <= c_hi / BN; ++b) atomicOr(&kb_bits[b >> 5], 1u << (b & 31));
    }
  }
  __syncthreads();

  const int row = threadIdx.x / 4, cq = threadIdx.x % 4;
  const int my_g = g0 + row;
  const bool row_ok = row < nr;
  float m = -INFINITY, l = 0.f;
  float o[32];  // dims cq + 4*i (d = 128) / cq + 4*i, i < 16 (d = 64)
  const int n_od = d / 4;
#pragma unroll
  for (int i = 0; i < 32; ++i) o[i] = 0.f;
  long long my_cells = 0;

  // process one tile whose columns are cols(j) = base + j (gathered == nullptr) or gcols[j]
  auto process_tile = [&](int base, bool gathered, int n_cols) {
    // load K, V rows
    for (int i = threadIdx.x; i < BN * (d / 8); i += blockDim.x) {
      int j = i / (d / 8), vv = i % (d / 8);
      float fk[8], fv[8];
      int c = gathered ? (j < n_cols ? gcols[j] : -1) : base + j;
      if (c >= 0 && c < p.n_total) {
        uint4 uk = *reinterpret_cast<const uint4 *>(kb + static_cast<int64_t>(c) * d + vv * 8);
        uint4 uv = *reinterpret_cast<const uint4 *>(vb + static_cast<int64_t>(c) * d + vv * 8);
        bf16x8_to_f32(uk, fk);
        bf16x8_to_f32(uv, fv);
      } else {
#pragma unroll
        for (int t = 0; t < 8; ++t) fk[t] = fv[t] = 0.f;
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        Ks[j * ld + vv * 8 + t] = fk[t];
        Vs[j * d + vv * 8 + t] = fv[t];
      }
    }
    __syncthreads();
    float s[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) s[i] = 0.f;
    const float *qr = Qs + row * ld;
    for (int kk = 0; kk < d; ++kk) {
      float qv = qr[kk];
#pragma unroll
      for (int i = 0; i < 16; ++i) s[i] = fmaf(qv, Ks[(cq + 4 * i) * ld + kk], s[i]);
    }
    float tmax = -INFINITY;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int j = cq + 4 * i;
      const int c = gathered ? (j < n_cols ? gcols[j] : 0x7fffffff) : base + j;
      bool keep = row_ok && c <= my_g;
      if (keep && !gathered && !p.dense) keep = bit(vbits, c) || bit(sb, my_g - c);
      s[i] = keep ? s[i] * p.scale_log2 : -INFINITY;
      my_cells += keep ? 1 : 0;
      tmax = fmaxf(tmax, s[i]);
    }
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
    const float m_new = fmaxf(m, tmax);
    const float corr = (m_new == -INFINITY) ? 1.f : fast_exp2(m - m_new);
    float lsum = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float pv = (s[i] == -INFINITY) ? 0.f : fast_exp2(s[i] - m_new);
      lsum += pv;
      Ps[row * (BN + 1) + cq + 4 * i] = pv;
    }
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 1);
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
    l = l * corr + lsum;
    m = m_new;
#pragma unroll
    for (int i = 0; i < 32; ++i) o[i] *= corr;
    __syncthreads();
    // O[row][cq + 4i] += sum_j P[row][j] V[j][cq + 4i]
    for (int j = 0; j < BN; ++j) {
      const float pv = Ps[row * (BN + 1) + j];
      const float *vr = Vs + j * d + cq;
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < n_od) o[i] = fmaf(pv, vr[4 * i], o[i]);
    }
    __syncthreads();
  };

  // dense blocks touched by slashes (or all causal blocks in dense mode)
  for (int b = 0; b < n_kb; ++b) {
    if (!((kb_bits[b >> 5] >> (b & 31)) & 1u)) continue;
    process_tile(b * BN, false, BN);
  }
  // gathered verticals outside touched blocks
  if (!p.dense && n_vt > 0) {
    const int v_end = [&] {  // verticals with c <= g_hi
      int lo = 0, hi = n_vt;
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (V[mid] <= g_hi)
          lo = mid + 1;
        else
          hi = mid;
      }
      return lo;
    }();
    int nbuf = 0;  // uniform across the CTA (kept in registers, synced via smem)
    for (int v0 = 0; v0 < v_end; v0 += 32) {
      if (threadIdx.x < 32) {
        const int vi = v0 + threadIdx.x;
        int c = vi < v_end ? V[vi] : -1;
        bool take = c >= 0 && !((kb_bits[(c / BN) >> 5] >> ((c / BN) & 31)) & 1u);
        unsigned ball = __ballot_sync(0xffffffffu, take);
        int rank = __popc(ball & ((1u << threadIdx.x) - 1u));
        int total = __popc(ball);
        // append; if it overflows BN the remainder goes to scratch first
        if (take) {
          int slot = nbuf + rank;
          if (slot < BN)
            gcols[slot] = c;
          else
            scratch[slot - BN] = c;
        }
        if (threadIdx.x == 0) scratch[63] = nbuf + total;
      }
      __syncthreads();
      nbuf = scratch[63];
      if (nbuf >= BN) {
        process_tile(0, true, BN);
        // move overflow back
        __syncthreads();
        const int rest = nbuf - BN;
        if (threadIdx.x < rest) gcols[threadIdx.x] = scratch[threadIdx.x];
        nbuf = rest;
        __syncthreads();
      }
    }
    if (nbuf > 0) process_tile(0, true, nbuf);
  }

  // epilogue
  if (row_ok) {
    const int64_t orow = static_cast<int64_t>(r0 + row) * p.out_row_stride + static_cast<int64_t>(h) * d;
    if (l > 0.f) {
      const float inv = 1.f / l;
      for (int i = 0; i < n_od; ++i) {
        const int dd = cq + 4 * i;
        float val = o[i] * inv;
        if (p.out_bf16)
          reinterpret_cast<uint16_t *>(p.out)[orow + dd] = f2bf(val);
        else
          reinterpret_cast<float *>(p.out)[orow + dd] = val;
      }
    } else {  // diagonal fallback, tensor_ops.py:136-137
      for (int i = 0; i < n_od; ++i) {
        const int dd = cq + 4 * i;
        float val = bf2f(vb[static_cast<int64_t>(my_g) * d + dd]);
        if (p.out_bf16)
          reinterpret_cast<uint16_t *>(p.out)[orow + dd] = f2bf(val);
        else
          reinterpret_cast<float *>(p.out)[orow + dd] = val;
      }
      if (cq == 0) my_cells += 1;
    }
  }
  // cell count
  long long cs = warp_sum_ll(my_cells);
  if ((threadIdx.x & 31) == 0 && cs) atomicAdd(reinterpret_cast<unsigned long long *>(p.cells + h),
                                               static_cast<unsigned long long>(cs));
}

__global__ void set_bits_kernel(const int32_t *ids, const int32_t *counts, int which, int n_total, int words,
                                uint32_t *bits) {
  const int h = blockIdx.y;
  const int n = counts[h * 2 + which];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int x = ids[static_cast<int64_t>(h) * n_total + i];
    atomicOr(bits + static_cast<int64_t>(h) * words + (x >> 5), 1u << (x & 31));
  }
}

// Seed rows: full probability rows of block rows [n_new - n_rows, n_new)
// (the decode observation seeds, session.py:89-95), in two parallel passes:
//  plan_scores_kernel  grid (column chunks of 256, row, head), one warp per 32
//                      columns: the selected cells (vertical bit or slash bit of
//                      g - c, tensor_ops.py:130-138) get q.k * log2(e)/sqrt(d)
//                      by a coalesced warp dot product, the others -inf; each
//                      CTA writes its chunk's (max, sum of exp2) partial.
//  plan_norm_kernel    grid (row, head): combines the partials in chunk order
//                      and normalises the row in place (zeros off-plan); an
//                      empty row becomes the diagonal fallback (tensor_ops.py:136-137).
constexpr int PR_CHUNK = 256;

__global__ void __launch_bounds__(PR_CHUNK) plan_scores_kernel(Params p, int n_rows, float *out, int64_t out_stride,
                                                               int64_t out_head_stride, float2 *part, int n_chunks) {
  __shared__ float wmax[PR_CHUNK / 32], wsum[PR_CHUNK / 32];
  const int ch = blockIdx.x, i = blockIdx.y, h = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = p.n_new - n_rows + i;
  const int g = p.row_offset + r;
  const int d = p.d;
  const int c = ch * PR_CHUNK + threadIdx.x;  // this thread's column
  const uint32_t *sb = p.sbits + static_cast<int64_t>(h) * p.words;
  const uint32_t *vbits = p.vbits + static_cast<int64_t>(h) * p.words;
  const bool sel = c <= g && c < p.n_total && (bit(vbits, c) || bit(sb, g - c));
  // q: lane owns dims [4 lane, 4 lane + 4) (d = 128) or [2 lane, +2) (d = 64)
  const uint16_t *qr = p.q + static_cast<int64_t>(h) * p.q_head_stride + static_cast<int64_t>(r) * d;
  const uint16_t *kb = p.k + static_cast<int64_t>(h / p.group) * p.kv_head_stride;
  const int dpl = d / 32;
  float qv[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) qv[e] = e < dpl ? bf2f(qr[lane * dpl + e]) : 0.f;
  float my = -INFINITY;
  unsigned m = __ballot_sync(0xffffffffu, sel);
  while (m) {
    const int src = __ffs(m) - 1;
    m &= m - 1;
    const int cc = ch * PR_CHUNK + warp * 32 + src;
    const uint16_t *kr = kb + static_cast<int64_t>(cc) * d + lane * dpl;
    float acc;
    if (dpl == 4) {
      const uint2 u = *reinterpret_cast<const uint2 *>(kr);
      acc = qv[0] * __uint_as_float(u.x << 16) + qv[1] * __uint_as_float(u.x & 0xffff0000u) +
            qv[2] * __uint_as_float(u.y << 16) + qv[3] * __uint_as_float(u.y & 0xffff0000u);
    } else {
      const uint32_t u = *reinterpret_cast<const uint32_t *>(kr);
      acc = qv[0] * __uint_as_float(u << 16) + qv[1] * __uint_as_float(u & 0xffff0000u);
    }
    acc = warp_sum(acc) * p.scale_log2;
    if (lane == src) my = acc;
  }
  float *orow = out + static_cast<int64_t>(h) * out_head_stride + static_cast<int64_t>(i) * out_stride;
  if (c < p.n_total) orow[c] = my;
  // chunk partial (max, sum exp2(s - max))
  const float wm = warp_max(my);
  const float we = warp_sum(my == -INFINITY ? 0.f : fast_exp2(my - wm));
  if (lane == 0) {
    wmax[warp] = wm;
    wsum[warp] = we;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = -INFINITY, S = 0.f;
    for (int w = 0; w < PR_CHUNK / 32; ++w) M = fmaxf(M, wmax[w]);
    for (int w = 0; w < PR_CHUNK / 32; ++w)
      if (wmax[w] != -INFINITY) S += wsum[w] * fast_exp2(wmax[w] - M);
    part[(static_cast<int64_t>(h) * n_rows + i) * n_chunks + ch] = make_float2(M, S);
  }
}

__global__ void __launch_bounds__(256) plan_norm_kernel(Params p, int n_rows, float *out, int64_t out_stride,
                                                        int64_t out_head_stride, const float2 *part, int n_chunks) {
  __shared__ float stats[2];
  __shared__ float red[256 / 32];
  const int i = blockIdx.x, h = blockIdx.y;
  const int g = p.row_offset + p.n_new - n_rows + i;
  const float2 *pp = part + (static_cast<int64_t>(h) * n_rows + i) * n_chunks;
  // the chunk partials combined by the whole block (fixed-order reductions:
  // deterministic), not by one thread walking them serially
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float m = -INFINITY;
  for (int c = threadIdx.x; c < n_chunks; c += blockDim.x) m = fmaxf(m, pp[c].x);
  m = warp_max(m);
  if (lane == 0) red[wid] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = -INFINITY;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) M = fmaxf(M, red[w]);
    stats[0] = M;
  }
  __syncthreads();
  const float Mb = stats[0];
  float sacc = 0.f;
  for (int c = threadIdx.x; c < n_chunks; c += blockDim.x) {
    const float2 v = pp[c];
    if (v.x != -INFINITY) sacc += v.y * fast_exp2(v.x - Mb);
  }
  sacc = warp_sum(sacc);
  __syncthreads();  // red reused
  if (lane == 0) red[wid] = sacc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float S = 0.f;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) S += red[w];
    stats[1] = S > 0.f ? 1.f / S : 0.f;
  }
  __syncthreads();
  const float M = stats[0], inv = stats[1];
  float *orow = out + static_cast<int64_t>(h) * out_head_stride + static_cast<int64_t>(i) * out_stride;
  // this CTA's column slice (grid.z): every slice recomputes the row statistics
  const int per = (p.n_total + gridDim.z - 1) / gridDim.z;
  const int c_lo = blockIdx.z * per, c_hi = min(p.n_total, c_lo + per);
  for (int c = c_lo + threadIdx.x; c < c_hi; c += blockDim.x) {
    if (M == -INFINITY) {
      orow[c] = (c == g) ? 1.f : 0.f;
    } else {
      const float s = orow[c];
      orow[c] = s == -INFINITY ? 0.f : fast_exp2(s - M) * inv;
    }
  }
}

inline size_t smem_bytes(int d) {
  const int ld = d + 1;
  return static_cast<size_t>(BM * ld + BN * ld + BN * d + BM * (BN + 1)) * 4 + MAX_KB_WORDS * 4 + BN * 4 +
         64 * 4 + 64;
}

inline void fill(Params &p, const ls_layer_desc *L) {
  p.n_heads = L->n_heads;
  p.out_row_stride = L->out_row_stride ? L->out_row_stride : static_cast<int64_t>(L->n_heads) * L->head_dim;
  p.group = L->n_heads / L->n_kv_heads;
  p.d = L->head_dim;
  p.n_new = L->n_new;
  p.n_total = L->n_total;
  p.row_offset = L->row_offset;
  p.words = (L->n_total + 31) / 32;
  p.q_head_stride = L->q_head_stride;
  p.kv_head_stride = L->kv_head_stride;
  p.scale_log2 = kLog2e / sqrtf(static_cast<float>(L->head_dim));
}

int check_desc(const ls_layer_desc *L) {
  LS_REQUIRE(L->head_dim == 64 || L->head_dim == 128, LS_ERR_UNSUPPORTED, "head_dim must be 64 or 128");
  LS_REQUIRE(L->n_heads > 0 && L->n_kv_heads > 0 && L->n_heads % L->n_kv_heads == 0, LS_ERR_DIMENSION_MISMATCH,
             "n_heads must be a multiple of n_kv_heads");
  LS_REQUIRE(L->n_new > 0 && L->row_offset == L->n_total - L->n_new, LS_ERR_DIMENSION_MISMATCH,
             "row_offset=%d must equal K rows - Q rows >= 0", L->row_offset);
  LS_REQUIRE((L->n_total + BN - 1) / BN <= MAX_KB_WORDS * 32, LS_ERR_UNSUPPORTED, "n_total too large");
  return LS_OK;
}

}  // namespace k5
}  // namespace ls

using namespace ls;

namespace ls {
size_t vs_attention_ws_workspace(const ls_layer_desc *L);
int vs_attention_ws(const ls_layer_desc *L, const uint16_t *q, const uint16_t *k, const uint16_t *v,
                    const int32_t *slash_ids, const int32_t *vert_ids, const int32_t *counts, void *out,
                    int32_t out_bf16, int64_t *cells, int64_t *tiles, int dense, void *ws, size_t ws_bytes,
                    cudaStream_t st, float *row_lse = nullptr);
size_t score_lines_tc_workspace(const ls_layer_desc *L, int32_t n_s);
int score_row_lse(const ls_layer_desc *L, int32_t n_s, const uint16_t *q, const uint16_t *k, const int32_t *rows,
                  float *lse, void *ws, size_t ws_bytes, cudaStream_t st);

namespace cov {
__global__ void iota_rows_kernel(int32_t *rows, int n) {
  const int h = blockIdx.y;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    rows[static_cast<int64_t>(h) * n + r] = r;
}
// coverage[h] = (1/n) sum_r 2^(lse_plan[r] - lse_full[r]): the full-softmax mass
// of each row's plan cells, averaged over the block's rows (every row sums to 1)
__global__ void coverage_kernel(const float *lse_plan, const float *lse_full, int n, double *coverage) {
  __shared__ double red[32];
  const int h = blockIdx.x;
  double sum = 0.0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    const float lp = lse_plan[static_cast<int64_t>(h) * n + r], lf = lse_full[static_cast<int64_t>(h) * n + r];
    if (lp != -INFINITY) sum += static_cast<double>(exp2f(fminf(lp - lf, 0.f)));
  }
  sum = warp_sum_d(sum);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
    coverage[h] = n > 0 ? t / n : 0.0;
  }
}
}  // namespace cov
}  // namespace ls

extern "C" size_t ls_vs_attention_workspace(const ls_layer_desc *L) {
  const size_t words = (L->n_total + 31) / 32;
  const size_t simt = 2 * static_cast<size_t>(L->n_heads) * words * 4 + 1024;
  const size_t tcw = vs_attention_ws_workspace(L);
  return simt > tcw ? simt : tcw;
}

extern "C" int ls_vs_attention(const ls_layer_desc *L, const uint16_t *q, const uint16_t *k, const uint16_t *v,
                               const int32_t *slash_ids, const int32_t *vert_ids, const int32_t *counts, void *out,
                               int32_t out_bf16, int64_t *cells, void *ws, size_t ws_bytes, ls_stream_t stream) {
  int stc = k5::check_desc(L);
  if (stc) return stc;
  return vs_attention_ws(L, q, k, v, slash_ids, vert_ids, counts, out, out_bf16, cells, nullptr, 0, ws, ws_bytes,
                         static_cast<cudaStream_t>(stream));
}

extern "C" int ls_vs_attention_ex(const ls_layer_desc *L, const uint16_t *q, const uint16_t *k, const uint16_t *v,
                                  const int32_t *slash_ids, const int32_t *vert_ids, const int32_t *counts,
                                  void *out, int32_t out_bf16, int64_t *cells, int64_t *tiles, void *ws,
                                  size_t ws_bytes, ls_stream_t stream) {
  int stc = k5::check_desc(L);
  if (stc) return stc;
  return vs_attention_ws(L, q, k, v, slash_ids, vert_ids, counts, out, out_bf16, cells, tiles, 0, ws, ws_bytes,
                         static_cast<cudaStream_t>(stream));
}

static int build_bits(const ls_layer_desc *L, const int32_t *slash_ids, const int32_t *vert_ids,
                      const int32_t *counts, uint32_t *sbits, uint32_t *vbits, cudaStream_t st) {
  const int words = (L->n_total + 31) / 32;
  LS_CUDA(cudaMemsetAsync(sbits, 0, sizeof(uint32_t) * L->n_heads * words, st));
  LS_CUDA(cudaMemsetAsync(vbits, 0, sizeof(uint32_t) * L->n_heads * words, st));
  k5::set_bits_kernel<<<dim3(4, L->n_heads), 256, 0, st>>>(slash_ids, counts, 0, L->n_total, words, sbits);
  k5::set_bits_kernel<<<dim3(4, L->n_heads), 256, 0, st>>>(vert_ids, counts, 1, L->n_total, words, vbits);
  LS_LAUNCH_CHECK("set_bits_kernel");
  return LS_OK;
}

extern "C" int ls_vs_attention_simt(const ls_layer_desc *L, const uint16_t *q, const uint16_t *k,
                                    const uint16_t *v, const int32_t *slash_ids, const int32_t *vert_ids,
                                    const int32_t *counts, void *out, int32_t out_bf16, int64_t *cells, void *ws,
                                    size_t ws_bytes, ls_stream_t stream) {
  int stc = k5::check_desc(L);
  if (stc) return stc;
  LS_REQUIRE(ws_bytes >= ls_vs_attention_workspace(L), LS_ERR_WORKSPACE, "vs_attention workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int words = (L->n_total + 31) / 32;
  Carver c(ws, ws_bytes);
  uint32_t *sbits = c.take<uint32_t>(static_cast<size_t>(L->n_heads) * words);
  uint32_t *vbits = c.take<uint32_t>(static_cast<size_t>(L->n_heads) * words);
  int s = build_bits(L, slash_ids, vert_ids, counts, sbits, vbits, st);
  if (s) return s;
  k5::Params p;
  k5::fill(p, L);
  p.q = q;
  p.k = k;
  p.v = v;
  p.slash_ids = slash_ids;
  p.vert_ids = vert_ids;
  p.counts = counts;
  p.sbits = sbits;
  p.vbits = vbits;
  p.out = out;
  p.out_bf16 = out_bf16;
  p.cells = reinterpret_cast<long long *>(cells);
  p.dense = 0;
  LS_CUDA(cudaMemsetAsync(cells, 0, sizeof(int64_t) * L->n_heads, st));
  const size_t smem = k5::smem_bytes(L->head_dim);
  LS_CUDA(cudaFuncSetAttribute(k5::vs_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  k5::vs_attention_kernel<<<dim3(ceil_div(L->n_new, k5::BM), L->n_heads), k5::THREADS, smem, st>>>(p);
  LS_LAUNCH_CHECK("vs_attention_kernel");
  return LS_OK;
}

// stream-ordered scratch: keep the default pool's memory across syncs so the
// per-call cudaMallocAsync is a pool hit, not a fresh mapping
static void keep_pool_memory() {
  static bool done = false;
  if (done) return;
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done = true;
}

extern "C" int ls_plan_rows(const ls_layer_desc *L, int32_t n_rows, const uint16_t *q, const uint16_t *k,
                            const int32_t *slash_ids, const int32_t *vert_ids, const int32_t *counts, float *out,
                            int64_t out_row_stride, int64_t out_head_stride, ls_stream_t stream) {
  int stc = k5::check_desc(L);
  if (stc) return stc;
  LS_REQUIRE(n_rows >= 0 && n_rows <= L->n_new, LS_ERR_DIMENSION_MISMATCH, "n_rows outside [0, n_new]");
  if (n_rows == 0) return LS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int words = (L->n_total + 31) / 32;
  uint32_t *bits = nullptr;
  keep_pool_memory();
  const int n_chunks = ceil_div(L->n_total, k5::PR_CHUNK);
  const size_t bits_bytes = (sizeof(uint32_t) * 2 * L->n_heads * words + 255) / 256 * 256;
  LS_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&bits),
                          bits_bytes + sizeof(float2) * static_cast<size_t>(L->n_heads) * n_rows * n_chunks, st));
  float2 *part = reinterpret_cast<float2 *>(reinterpret_cast<char *>(bits) + bits_bytes);
  uint32_t *sbits = bits, *vbits = bits + static_cast<size_t>(L->n_heads) * words;
  int s = build_bits(L, slash_ids, vert_ids, counts, sbits, vbits, st);
  if (s) return s;
  k5::Params p;
  k5::fill(p, L);
  p.q = q;
  p.k = k;
  p.sbits = sbits;
  p.vbits = vbits;
  k5::plan_scores_kernel<<<dim3(n_chunks, n_rows, L->n_heads), k5::PR_CHUNK, 0, st>>>(p, n_rows, out, out_row_stride,
                                                                                     out_head_stride, part, n_chunks);
  LS_LAUNCH_CHECK("plan_scores_kernel");
  k5::plan_norm_kernel<<<dim3(n_rows, L->n_heads, (L->n_total + 2047) / 2048), 256, 0, st>>>(
      p, n_rows, out, out_row_stride, out_head_stride, part,
                                                                 n_chunks);
  LS_LAUNCH_CHECK("plan_norm_kernel");
  LS_CUDA(cudaFreeAsync(bits, st));
  return LS_OK;
}

extern "C" int ls_dense_attention(const ls_layer_desc *L, const uint16_t *q, const uint16_t *k, const uint16_t *v,
                                  void *out, int32_t out_bf16, ls_stream_t stream) {
  int stc = k5::check_desc(L);
  if (stc) return stc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t *cells = nullptr;
  keep_pool_memory();
  LS_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&cells), sizeof(int64_t) * L->n_heads, st));
  // dense mode touches every causal key block with the causal mask only (tensor-core path)
  int s = vs_attention_ws(L, q, k, v, nullptr, nullptr, nullptr, out, out_bf16, cells, nullptr, 1, nullptr, 0, st);
  LS_CUDA(cudaFreeAsync(cells, st));
  return s;
}

// ------------------------------------------------------------ plan coverage
// coverage_ratio (reference prefill.py:254-281) for every head of a layer: the
// fraction of the block's full (dense, causal) attention mass that the plan's
// lines cover, by inclusion-exclusion == the mass of the union of plan cells.
// Per row: dense normaliser from K1's statistics pass over all rows, plan-cell
// normaliser from K5 (row_lse), mass = 2^(lse_plan - lse_full).
static size_t cov_align(size_t x) { return (x + 255) / 256 * 256; }

extern "C" size_t ls_plan_coverage_workspace(const ls_layer_desc *L) {
  const size_t H = L->n_heads, n = L->n_new;
  return 3 * cov_align(H * n * 4) + cov_align(n * H * L->head_dim * 2) + cov_align(H * 8) +
         cov_align(score_lines_tc_workspace(L, L->n_new)) + cov_align(ls_vs_attention_workspace(L)) + 1024;
}

extern "C" int ls_plan_coverage(const ls_layer_desc *L, const uint16_t *q, const uint16_t *k, const uint16_t *v,
                                const int32_t *slash_ids, const int32_t *vert_ids, const int32_t *counts,
                                double *coverage, void *ws, size_t ws_bytes, ls_stream_t stream) {
  int stc = k5::check_desc(L);
  if (stc) return stc;
  LS_REQUIRE(ws_bytes >= ls_plan_coverage_workspace(L), LS_ERR_WORKSPACE, "plan coverage workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int H = L->n_heads, n = L->n_new;
  char *b = static_cast<char *>(ws);
  int32_t *rows = reinterpret_cast<int32_t *>(b);
  b += cov_align(static_cast<size_t>(H) * n * 4);
  float *lse_full = reinterpret_cast<float *>(b);
  b += cov_align(static_cast<size_t>(H) * n * 4);
  float *lse_plan = reinterpret_cast<float *>(b);
  b += cov_align(static_cast<size_t>(H) * n * 4);
  void *out = b;
  b += cov_align(static_cast<size_t>(n) * H * L->head_dim * 2);
  int64_t *cells = reinterpret_cast<int64_t *>(b);
  b += cov_align(static_cast<size_t>(H) * 8);
  const size_t w1 = cov_align(score_lines_tc_workspace(L, n));
  void *ws1 = b;
  b += w1;
  const size_t w2 = ls_vs_attention_workspace(L);
  cov::iota_rows_kernel<<<dim3(8, H), 256, 0, st>>>(rows, n);
  LS_LAUNCH_CHECK("iota_rows_kernel");
  int r = score_row_lse(L, n, q, k, rows, lse_full, ws1, w1, st);
  if (r) return r;
  r = vs_attention_ws(L, q, k, v, slash_ids, vert_ids, counts, out, 1, cells, nullptr, 0, b, w2, st, lse_plan);
  if (r) return r;
  cov::coverage_kernel<<<H, 256, 0, st>>>(lse_plan, lse_full, n, coverage);
  LS_LAUNCH_CHECK("coverage_kernel");
  return LS_OK;
}
