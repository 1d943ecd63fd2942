// K6 + K7 + K8 -- progressive decode with periodic KV compression.
//
// Device-resident decode state for ALL layers of a session (ls_decode_stack),
// with the step counters in device memory so that one decode step (every
// layer) and one compression event (every layer) are fixed launch sequences
// that the host captures into CUDA graphs.
//
// K6 decode attention replaces the working-set branch of forward_extend
// (reference model.py:232-241) inside decode_step (model.py:289-311): per
// q-head, cols = working set U {new position}, softmax(K[cols] q / sqrt(d)),
// out = w V[cols]; the observation row (cols, w) (kvcompress.py:233) goes to
// the head's ring slot as raw log2-domain logits plus the row's (max, sum), so
// it is normalised only when an event reads it. Working set:
//   before the first event: [0, length)                        (kvcompress.py:194, 237)
//   after it: selected U [length - W, length)                  (kvcompress.py:235)
// Dense steps are computed per KV head for its q-head group (each K/V row is
// read once for the group); compressed steps per q-head from the compacted
// cache (segment A: selected ids < length - W) plus the archive window
// (segment B). One kernel: split-K CTAs write partials, the last CTA of a head
// combines them (threadfence + ticket).
//
// K7 (event, all layers in one launch) replaces accumulate_scores +
// _top_by_score + retained_union (kvcompress.py:67-90, 126-130, 210-224):
// buffered rows are accumulated oldest -> newest in fp64 (rows have distinct
// ids: a row is added in parallel with no races, the per-id order is the
// reference's), candidates are the touched ids only (kvcompress.py:73-83),
// an 8-pass radix select on the fp64 bits finds the B-th largest by (score
// desc, id asc), picked ids are emitted in id order.
//
// K8 (all layers) replaces compact_cache (kvcompress.py:133-147): coalesced
// 16-byte gather of the picked K/V rows into the contiguous per-head cache.

#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#include "ls_common.cuh"
#include "tc_common.cuh"

namespace ls {
extern int *g_debug_buffer;  // ls_debug_set_buffer (host-mapped): per-CTA timeline records
namespace dec {

constexpr int K6_THREADS = 128;
constexpr int K7_THREADS = 1024;
constexpr int K7_SMEM_CAP = 24 * 1024;  // ids accumulated in shared memory (fp64) up to this length
constexpr int K7_CAND_CAP = 4096;       // touched ids listed in shared memory (radix + ranking over the list)
constexpr int K7_BITONIC = 2048;        // candidate lists up to this size are ranked by one bitonic sort
constexpr int K7_RB = 8, K7_PF = 2;     // rows fetched per round, columns per thread per row
constexpr int K7_DMAX = 64, K7_DCH = 16;  // dense-window fast path: rows, rows loaded per batch

__device__ __forceinline__ int64_t head_row(const ls_decode_stack &S, int layer, int h) {
  return static_cast<int64_t>(layer) * S.n_heads + h;
}

struct Geo {
  int n_a, lo, n_cols;
};

// first index i in [0, n) with a[i] >= x, all threads of the block together:
// two dependent global round trips (128 strided samples, then one bucket)
// instead of log2(n) for a single-thread binary search
__device__ __forceinline__ int block_lower_bound(const int32_t *a, int n, int x) {
  const int nt = blockDim.x;
  const int stride = (n + nt - 1) / nt;
  const int t = threadIdx.x;
  const int c1 = __syncthreads_count(t * stride < n && __ldg(a + t * stride) < x);
  if (c1 == 0) return 0;
  const int start = (c1 - 1) * stride;
  const int c2 = __syncthreads_count(t < stride && start + t < n && __ldg(a + start + t) < x);
  return start + c2;
}

// geometry of a q-head's working set at this step (called by every thread)
__device__ __forceinline__ Geo geometry(const ls_decode_stack &S, int layer, int h, int length, int compressed) {
  Geo g;
  if (compressed) {
    g.lo = max(0, length - S.window);
    g.n_a = S.n_a[head_row(S, layer, h)];  // kept current by the event and advance kernels
  } else {
    g.lo = 0;
    g.n_a = 0;
  }
  g.n_cols = g.n_a + (length - g.lo + 1);
  return g;
}

// ------------------------------------------------------------------ K6
// Split-K over columns: CTA (split, unit) owns a contiguous column range and
// streams it in tiles of K6_TILE rows. K and V tiles are staged in shared
// memory with cp.async (16-B chunks, double-buffered, zero-filled past the
// range), so every HBM byte is requested once, coalesced, with two tiles in
// flight per CTA and several CTAs per SM. Scores: 8 lanes per row (16 B
// chunks, conflict-free quarter-warp phases), q in registers, shuffle
// reduction; the raw log2 logits go to the ring (coalesced, 64 per head).
// Online softmax per CTA across its tiles; PV: warp w owns 16 rows of a tile,
// lane owns D/32 dims. The last CTA of a unit combines the splits in split
// order (deterministic).
constexpr int K6_TILE = 64;
constexpr int K6_STAGES = 2;
constexpr int K6_MAX_CLUSTER = 16;  // splits of a unit = one thread-block cluster
// G <= 4: 16-CTA clusters (non-portable); larger q-groups: 8 (the gather
// area + cross-warp buffers must fit in the tile buffers)
__host__ __device__ constexpr int k6_max_cluster(int G) { return G > 4 ? 8 : K6_MAX_CLUSTER; }

__device__ __forceinline__ void cp_async16_zfill(uint32_t saddr, const void *g, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(valid ? 16 : 0) : "memory");
}

template <int D>
constexpr int k6_smem_bytes(int G) {
  return 2 * K6_STAGES * K6_TILE * D * 2 + 2 * G * K6_TILE * 4 + (G * K6_MAX_CLUSTER + 2 * G) * 4;
}

template <int D, int G>
__global__ void __launch_bounds__(K6_THREADS) decode_kernel(ls_decode_stack S, int layer, const uint16_t *q,
                                                            int64_t q_head_stride, int q_from_archive,
                                                            const uint16_t *k, const uint16_t *v, int compressed,
                                                            float scale_log2, void *out, int out_bf16, int pdl) {
  constexpr int ROW_B = D * 2;
  constexpr int CH = D / 8;                 // 16-B chunks per row
  constexpr int CPL = CH / 8;               // chunks per lane in the score phase (8 lanes per row)
  constexpr int TILE_B = K6_TILE * ROW_B;
  constexpr int DPL = D / 32;               // dims per lane in the PV phase
  constexpr int GS = G < 4 ? G : 4;         // heads per score pass (register bound)
  constexpr int NSUB = (G + GS - 1) / GS;
  extern __shared__ __align__(16) unsigned char dsm[];
  unsigned char *kt = dsm;
  unsigned char *vt = dsm + K6_STAGES * TILE_B;
  float *ps = reinterpret_cast<float *>(dsm + 2 * K6_STAGES * TILE_B);  // [G][TILE] raw log2 scores
  float *pp = ps + G * K6_TILE;                                        // [G][TILE] probabilities
  // [4][G][D] cross-warp reduction, in the tile buffers after the gather area
  float *ored = reinterpret_cast<float *>(dsm) + k6_max_cluster(G) * G * (D + 2);
  const int split = blockIdx.x, unit = blockIdx.y, n_split = gridDim.x;  // cluster = the unit's splits
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, seg = lane & 7;
  const int length = S.step[0];
  const int slot = S.step[1] % S.window;
  const int group = S.n_heads / S.n_kv_heads;
  // units: q-heads when G == 1 (compressed steps, and dense steps split per
  // q-head for parallelism), else kv-heads with their G q-heads
  const int kv = G == 1 ? unit / group : unit;
  const int h0 = G == 1 ? unit : unit * G;
  const Geo geo = geometry(S, layer, h0, length, compressed);
  const int per = ((geo.n_cols + n_split - 1) / n_split + K6_TILE - 1) / K6_TILE * K6_TILE;
  const int c_begin = min(geo.n_cols, split * per);
  const int c_end = min(geo.n_cols, c_begin + per);
  const int n_tiles = (c_end - c_begin + K6_TILE - 1) / K6_TILE;
  const uint16_t *kb = k + static_cast<int64_t>(kv) * S.kv_head_stride;
  const uint16_t *vb = v + static_cast<int64_t>(kv) * S.kv_head_stride;
  const int64_t hr0 = head_row(S, layer, h0);
  const uint16_t *ckb = S.ck + hr0 * S.budget_cap * D;
  const uint16_t *cvb = S.cv + hr0 * S.budget_cap * D;
  const int32_t *sel = S.sel_ids + hr0 * S.budget_cap;

  auto issue = [&](int t) {
    const int st = t % K6_STAGES;
    const int c0 = c_begin + t * K6_TILE;
    const uint32_t ks = tc::smem_u32(kt + st * TILE_B), vs = tc::smem_u32(vt + st * TILE_B);
#pragma unroll
    for (int it = 0; it < K6_TILE * CH / K6_THREADS; ++it) {
      const int i = tid + it * K6_THREADS;
      const int r = i / CH, c = i % CH;
      const int j = c0 + r;
      const bool ok = j < c_end;
      int64_t off;
      const uint16_t *kbase, *vbase;
      if (j < geo.n_a) {
        off = static_cast<int64_t>(j) * D;
        kbase = ckb, vbase = cvb;
      } else {
        off = static_cast<int64_t>(ok ? geo.lo + (j - geo.n_a) : 0) * D;
        kbase = kb, vbase = vb;
      }
      cp_async16_zfill(ks + r * ROW_B + c * 16, kbase + off + c * 8, ok);
      cp_async16_zfill(vs + r * ROW_B + c * 16, vbase + off + c * 8, ok);
    }
    tc::cp_async_commit();
  };

  if (n_tiles > 0) issue(0);
  // programmatic dependent launch: the archive / compacted-cache tiles above
  // do not depend on the previous kernel; q (the previous layer's output in a
  // full model) and every write below do
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  // q of this step: [H][D] buffer, or the Q archive at position `length`
  const uint16_t *qbase = q_from_archive ? q + static_cast<int64_t>(length) * D : q;

  // q of the first head sub-group stays in registers (dims of this lane's chunks)
  float qr[GS][CPL * 8];
  auto load_q = [&](int gb) {
#pragma unroll
    for (int g = 0; g < GS; ++g)
#pragma unroll
      for (int m = 0; m < CPL; ++m) {
        const int hh = min(h0 + gb + g, h0 + G - 1);
        bf16x8_to_f32(__ldg(reinterpret_cast<const uint4 *>(qbase + static_cast<int64_t>(hh) * q_head_stride +
                                                            (seg + 8 * m) * 8)),
                      &qr[g][m * 8]);
      }
  };
  if (NSUB == 1) load_q(0);

  float m_run[G], l_run[G], o[G][DPL];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m_run[g] = -INFINITY;
    l_run[g] = 0.f;
#pragma unroll
    for (int e = 0; e < DPL; ++e) o[g][e] = 0.f;
  }

  for (int t = 0; t < n_tiles; ++t) {
    const int st = t % K6_STAGES;
    const int c0 = c_begin + t * K6_TILE;
    if (t + 1 < n_tiles) {
      issue(t + 1);
      tc::cp_async_wait<1>();
    } else {
      tc::cp_async_wait<0>();
    }
    __syncthreads();
    const unsigned char *ktile = kt + st * TILE_B;
    // ---- scores
#pragma unroll
    for (int sb = 0; sb < NSUB; ++sb) {
      if (NSUB > 1) load_q(sb * GS);
#pragma unroll
      for (int it = 0; it < K6_TILE / 16; ++it) {
        const int r = warp * (K6_TILE / 4) + it * 4 + (lane >> 3);
        float acc[GS];
#pragma unroll
        for (int g = 0; g < GS; ++g) acc[g] = 0.f;
#pragma unroll
        for (int m = 0; m < CPL; ++m) {
          float f[8];
          bf16x8_to_f32(*reinterpret_cast<const uint4 *>(ktile + r * ROW_B + (seg + 8 * m) * 16), f);
#pragma unroll
          for (int g = 0; g < GS; ++g)
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[g] = fmaf(qr[g][m * 8 + e], f[e], acc[g]);
        }
#pragma unroll
        for (int g = 0; g < GS; ++g) {
          acc[g] += __shfl_xor_sync(0xffffffffu, acc[g], 1);
          acc[g] += __shfl_xor_sync(0xffffffffu, acc[g], 2);
          acc[g] += __shfl_xor_sync(0xffffffffu, acc[g], 4);
        }
        if (seg == 0) {
#pragma unroll
          for (int g = 0; g < GS; ++g)
            if (sb * GS + g < G) ps[(sb * GS + g) * K6_TILE + r] = (c0 + r < c_end) ? acc[g] * scale_log2 : -INFINITY;
        }
      }
    }
    __syncthreads();
    // ---- ring rows (raw log2 logits, normalised at events) + online softmax
    if (tid < K6_TILE && c0 + tid < c_end) {
      const int j = c0 + tid;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int64_t hr = head_row(S, layer, h0 + g);
        S.ring_s[(hr * S.window + slot) * S.row_cap + j] = ps[g * K6_TILE + tid];
        if (compressed) S.ring_ids[(hr * S.window + slot) * S.sparse_cap + j] = j < geo.n_a ? sel[j] : geo.lo + (j - geo.n_a);
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float a = ps[g * K6_TILE + lane], b = ps[g * K6_TILE + 32 + lane];
      const float m_new = fmaxf(m_run[g], warp_max(fmaxf(a, b)));
      const float corr = m_run[g] == -INFINITY ? 0.f : fast_exp2(m_run[g] - m_new);
      const float pa = a == -INFINITY ? 0.f : fast_exp2(a - m_new);
      const float pb = b == -INFINITY ? 0.f : fast_exp2(b - m_new);
      l_run[g] = l_run[g] * corr + warp_sum(pa + pb);
#pragma unroll
      for (int e = 0; e < DPL; ++e) o[g][e] *= corr;
      m_run[g] = m_new;
      // this warp's rows [16 warp, 16 warp + 16): row r < 32 sits in lane r of a, else lane r - 32 of b
      const int r = warp * 16 + (lane & 15);
      if ((lane >> 4) == (warp & 1)) pp[g * K6_TILE + r] = (warp < 2) ? pa : pb;
    }
    __syncwarp();
    // ---- PV over this warp's 16 rows
    const unsigned char *vtile = vt + st * TILE_B;
#pragma unroll 4
    for (int rr = 0; rr < 16; ++rr) {
      const int r = warp * 16 + rr;
      float f[DPL];
      if constexpr (DPL == 4) {
        const uint2 u = *reinterpret_cast<const uint2 *>(vtile + r * ROW_B + lane * 8);
        f[0] = __uint_as_float(u.x << 16);
        f[1] = __uint_as_float(u.x & 0xffff0000u);
        f[2] = __uint_as_float(u.y << 16);
        f[3] = __uint_as_float(u.y & 0xffff0000u);
      } else {
        const uint32_t u = *reinterpret_cast<const uint32_t *>(vtile + r * ROW_B + lane * 4);
        f[0] = __uint_as_float(u << 16);
        f[1] = __uint_as_float(u & 0xffff0000u);
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float pv = pp[g * K6_TILE + r];
#pragma unroll
        for (int e = 0; e < DPL; ++e) o[g][e] = fmaf(pv, f[e], o[g][e]);
      }
    }
    __syncthreads();  // stage st and ps/pp are reused by tile t + 2 / t + 1
  }

  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // next layer may start its prologue
  // ---- cross-warp reduce -> this split's partial, in this CTA's shared memory
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int e = 0; e < DPL; ++e) ored[(warp * G + g) * D + lane * DPL + e] = o[g][e];
  __syncthreads();
  // ---- the unit's splits form one thread-block cluster: every split pushes
  // its partial (max, sum, o) into rank 0's shared memory (fire-and-forget
  // DSMEM stores), rank 0 combines them in split order
  cg::cluster_group cluster = cg::this_cluster();
  cluster.sync();  // rank 0's tile buffers are free: its loop is done
  float *gather = reinterpret_cast<float *>(dsm);                       // [n_split][G][D + 2] in rank 0
  float *dst = cluster.map_shared_rank(gather, 0) + split * G * (D + 2);
  for (int i = tid; i < G * (D + 2); i += K6_THREADS) {
    const int g = i / (D + 2), e = i % (D + 2);
    float val;
    if (e == 0) {
      val = m_run[g];
    } else if (e == 1) {
      val = l_run[g];
    } else {
      val = 0.f;
#pragma unroll
      for (int w = 0; w < 4; ++w) val += ored[(w * G + g) * D + e - 2];
    }
    dst[i] = val;
  }
  cluster.sync();  // partials visible in rank 0
  if (split == 0) {
    float *wsc = reinterpret_cast<float *>(dsm + 2 * K6_STAGES * TILE_B) + 2 * G * K6_TILE;  // [G][n_split] weights
    float *mg = wsc + G * K6_MAX_CLUSTER;                                                   // [2G] max, total
    if (tid < G) {
      const int g = tid;
      float M = -INFINITY;
      for (int r = 0; r < n_split; ++r) M = fmaxf(M, gather[(r * G + g) * (D + 2)]);
      float Lsum = 0.f;
      for (int r = 0; r < n_split; ++r) {
        const float *pr = gather + (r * G + g) * (D + 2);
        const float w = pr[0] == -INFINITY ? 0.f : fast_exp2(pr[0] - M);
        wsc[g * K6_MAX_CLUSTER + r] = w;
        Lsum += pr[1] * w;
      }
      mg[g] = M;
      mg[G + g] = Lsum;
    }
    __syncthreads();
    for (int i = tid; i < G * D; i += K6_THREADS) {
      const int g = i / D, e = i % D;
      float acc = 0.f;
      for (int r = 0; r < n_split; ++r) acc = fmaf(wsc[g * K6_MAX_CLUSTER + r], gather[(r * G + g) * (D + 2) + 2 + e], acc);
      const float res = acc / mg[G + g];
      const int64_t oi = static_cast<int64_t>(h0 + g) * D + e;
      if (out_bf16)
        reinterpret_cast<uint16_t *>(out)[oi] = f2bf(res);
      else
        reinterpret_cast<float *>(out)[oi] = res;
    }
    if (tid < G) {
      const int64_t hr = head_row(S, layer, h0 + tid);
      S.ring_ml[(hr * S.window + slot) * 2 + 0] = mg[tid];
      S.ring_ml[(hr * S.window + slot) * 2 + 1] = mg[G + tid];
      S.ring_n[hr * S.window + slot] = geo.n_cols;
      S.ring_dense[hr * S.window + slot] = compressed ? 0 : 1;
    }
  }
}

// ------------------------------------------------------------------ K6 (tensor-core form)
// The same step on the tensor pipe: at decode shapes the CUDA-core form above
// spends ~0.25 warp-instructions per HBM byte (scalar dot products, shuffle
// reductions, per-row softmax) and is issue-bound at ~1.4 TB/s. Here a tile
// of 64 K/V rows arrives by TMA (128-B swizzle, one elected producer lane,
// NST-deep mbarrier ring) and each of the 4 consumer warps owns 16 rows:
//   S = Q K^T : mma.m16n8k16 bf16 -> fp32, A = the unit's q-heads (rows >= G
//               zero), B = K rows by ldmatrix (K row-major == B col-major);
//   online softmax per warp in registers (quad shuffles), raw log2 logits to
//   the ring; P (bf16) is reused as the A fragment of
//   O += P V    : mma.m16n8k16, B = V rows by ldmatrix.trans.
// ~0.02 warp-instructions per byte. mma.sync (not tcgen05) on purpose: M is
// the q-group (<= 8 rows), the kernel is HBM-bound and the tensor pipe idles.
// Warps merge in shared memory (fixed order), splits through global partials
// and a per-unit ticket (the last CTA combines in split order).
constexpr int KM_MAX_SPLIT = 64;  // splits of a unit (global partials)

struct KmMaps {
  CUtensorMap ck, cv, k, v;  // compacted cache [hr][budget_cap][D]; archive [kv][rows][D] (box 64 x 64)
};

// cluster combine: [n_split][G][D + 2] partials in rank 0 (dense variant: 16 splits x 8 heads)
__host__ __device__ constexpr int km_gather_b(int NG) { return NG == 2 ? 16 * 8 * 130 * 4 : 8192; }

// NW consumer warps x 16 rows = one tile of TILE K/V rows; NG such warp
// groups take alternate tiles (ping-pong); + one producer warp
template <int D, int NST, int NW, int NG, int RPW = 16>
struct KmSmem {
  static constexpr int TILE = RPW * NW;
  static constexpr int TILE_B = TILE * D * 2;  // one K or V tile, [D / 64][TILE rows][128 B] swizzled
  static constexpr int OFF_V = NST * TILE_B;
  static constexpr int OFF_BAR = 2 * NST * TILE_B;   // full[S], empty[S]
  static constexpr int OFF_MG = OFF_BAR + 16 * NST;  // [2][8] (M, L) of the CTA / combine weights
  static constexpr int OFF_W = OFF_MG + 2 * 8 * 4;   // [8][KM_MAX_SPLIT] split weights
  static constexpr int OFF_GATHER = (OFF_W + 8 * KM_MAX_SPLIT * 4 + 15) / 16 * 16;
  static constexpr int GATHER_B = km_gather_b(NG);
  static constexpr int TOTAL = OFF_GATHER + GATHER_B + 1024;  // + alignment slack
  // after the tile loop the stage buffers hold the warp merge: m[W][8], l[W][8], o[W][8][D]
  static_assert((3 * NW * NG * 8 + NW * NG * 8 * D + 8) * 4 <= 2 * NST * TILE_B, "merge area");
};

__device__ __forceinline__ void ldsm_x4(uint32_t *r, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t *r, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
// D += A B, m16n8k16 bf16 -> fp32; A rows 8-15 are zero here (a1 = a3 = 0)
__device__ __forceinline__ void mma_16816(float *d, uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
// D += A B, m16n8k16 bf16 -> fp32, all four A registers
__device__ __forceinline__ void mma_16816_a4(float *d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                             uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t *>(&h);
}
// byte offset of 16-B chunk c of tile row r in a [D / 64][TILE][128 B] 128-B-swizzled tile
template <int TILE>
__device__ __forceinline__ uint32_t km_off(int r, int c) {
  return static_cast<uint32_t>((c >> 3) * (TILE * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

struct KmTile {
  int seg_a;  // 1: compacted cache rows, 0: archive rows
  int row0;   // first source row (compacted index, or archive position)
  int valid;  // rows of the tile inside the working set
  int j0;     // working-set column of the tile's row 0
};
// working set = [compacted 0, n_a) ++ archive [lo, lo + n_cols - n_a); tiles never straddle the two
template <int KM_TILE>
__device__ __forceinline__ KmTile km_tile(int t, int t_a, const Geo &geo) {
  KmTile x;
  if (t < t_a) {
    x.seg_a = 1;
    x.row0 = t * KM_TILE;
    x.valid = min(KM_TILE, geo.n_a - x.row0);
    x.j0 = x.row0;
  } else {
    const int b = (t - t_a) * KM_TILE;
    x.seg_a = 0;
    x.row0 = geo.lo + b;
    x.valid = min(KM_TILE, geo.n_cols - geo.n_a - b);
    x.j0 = geo.n_a + b;
  }
  return x;
}

template <int D, int G, int NST, int NW, int NG, int RPW>
__global__ void __launch_bounds__((NW * NG + 1) * 32) decode_mma_kernel(const __grid_constant__ KmMaps maps, ls_decode_stack S,
                                                                int layer, const uint16_t *q, int64_t q_head_stride,
                                                                int q_from_archive, int compressed, float scale_log2,
                                                                void *out, int out_bf16, int pdl, int ccombine,
                                                                int *dbg) {
  static_assert(G <= 8, "q-group rows live in rows 0-7 of the m16 tile");
  auto gtime = []() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return static_cast<int>(t & 0x7fffffffull);
  };
  // the next layer's CTAs may launch at once: they only prefetch K/V before
  // their griddepcontrol.wait, which returns when this grid has completed
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  int *rec = dbg ? dbg + (static_cast<int64_t>(layer) * 256 + blockIdx.y * gridDim.x + blockIdx.x) * 16 : nullptr;
  if (rec && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    rec[0] = static_cast<int>(smid);
    rec[1] = gtime();
  }
  // a stage is only ever consumed by one warp group, so every group waits the
  // phases of its stages in order (a group running two phases ahead on a
  // shared barrier would see the older phase's parity as complete)
  static_assert(NST % NG == 0, "stages per warp group");
  static_assert(RPW == 16 || RPW == 8, "rows per consumer warp");
  constexpr int NTS = RPW / 8;  // n-tiles of 8 key rows per warp in S
  using L = KmSmem<D, NST, NW, NG, RPW>;
  constexpr int KM_TILE = L::TILE, KM_WARPS = NW * NG, KM_THREADS = (NW * NG + 1) * 32;
  constexpr int NT = D / 8;  // n-tiles of 8 dims in O
  constexpr bool SWAP = G == 1 && RPW == 16;  // one q-head: K / V as the A operands (see the tile loop)
  extern __shared__ unsigned char km_dyn[];
  unsigned char *sm = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(km_dyn) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + L::OFF_BAR);
  uint64_t *empty = full + NST;
  float *mg = reinterpret_cast<float *>(sm + L::OFF_MG);
  float *wsc = reinterpret_cast<float *>(sm + L::OFF_W);
  __shared__ int is_last;
  const int split = blockIdx.x, unit = blockIdx.y, n_split = gridDim.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int length = S.step[0];
  const int slot = S.step[1] % S.window;
  const int group = S.n_heads / S.n_kv_heads;
  const int kv = G == 1 ? unit / group : unit;
  const int h0 = G == 1 ? unit : unit * G;
  const Geo geo = geometry(S, layer, h0, length, compressed);
  const int t_a = (geo.n_a + KM_TILE - 1) / KM_TILE;
  const int t_all = t_a + (geo.n_cols - geo.n_a + KM_TILE - 1) / KM_TILE;
  const int t_begin = static_cast<int>(static_cast<int64_t>(t_all) * split / n_split);
  const int t_end = static_cast<int>(static_cast<int64_t>(t_all) * (split + 1) / n_split);
  const int n_my = t_end - t_begin;
  const int64_t hr0 = head_row(S, layer, h0);

  __shared__ __align__(8) uint64_t gbar;  // cluster combine: rank 0 receives the other splits' partials
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], NW);  // the warps of the group that consumes the stage
    }
    if (ccombine == 1 && split == 0) tc::mbar_init(&gbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (ccombine == 1 && split == 0)  // armed before any split can send (cluster barrier below)
      tc::mbar_expect_tx(&gbar, static_cast<uint32_t>((n_split - 1) * G * (D + 2) * 4));
  }
  __syncthreads();
  // cluster combine: this arrive (paired with the wait before the sends) orders
  // rank 0's armed mbarrier before every split's st.async
  if (ccombine == 1) asm volatile("barrier.cluster.arrive.aligned;" ::: "memory");

  if (warp == KM_WARPS) {
    // ---- producer: TMA K and V tiles of this split (independent of the previous kernel)
    if (lane == 0 && n_my > 0) {
      tc::prefetch_tmap(&maps.k);
      tc::prefetch_tmap(&maps.v);
      for (int i = 0; i < n_my; ++i) {
        const int st = i % NST;
        if (i >= NST) tc::mbar_wait(&empty[st], ((i / NST) - 1) & 1);
        const KmTile x = km_tile<KM_TILE>(t_begin + i, t_a, geo);
        tc::mbar_expect_tx(&full[st], 2 * L::TILE_B);
        const uint32_t ks = tc::smem_u32(sm + st * L::TILE_B), vs = tc::smem_u32(sm + L::OFF_V + st * L::TILE_B);
        const CUtensorMap *mk = x.seg_a ? &maps.ck : &maps.k;
        const CUtensorMap *mv = x.seg_a ? &maps.cv : &maps.v;
        const int z = x.seg_a ? static_cast<int>(hr0) : kv;
#pragma unroll
        for (int a = 0; a < D / 64; ++a) {
          tc::tma_load_3d(ks + a * KM_TILE * 128, mk, &full[st], a * 64, x.row0, z);
          tc::tma_load_3d(vs + a * KM_TILE * 128, mv, &full[st], a * 64, x.row0, z);
        }
      }
    }
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  } else {
    // ---- consumers
    const int wr0 = (warp % NW) * RPW, grp = warp / NW;
    // the working-set ids of this warp's rows in its first tiles (written by the
    // last compression event, not by the previous layer): loaded before the
    // dependency wait, so the per-tile ring-id stores never wait on L2
    constexpr int MAXPF = 4;
    int id_pf[MAXPF];
#pragma unroll
    for (int k = 0; k < MAXPF; ++k) {
      id_pf[k] = 0;
      const int i = grp + k * NG;
      if (compressed == 1 && i < n_my && lane < RPW) {
        const KmTile x = km_tile<KM_TILE>(t_begin + i, t_a, geo);
        if (wr0 + lane < x.valid)
          id_pf[k] = x.seg_a ? __ldg(S.sel_ids + hr0 * S.budget_cap + x.row0 + wr0 + lane) : x.row0 + wr0 + lane;
      }
    }
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    const int g = lane >> 2, t4 = lane & 3;
    const bool hv = g < G;
    const uint16_t *qbase = q_from_archive ? q + static_cast<int64_t>(length) * D : q;
    uint32_t qa[D / 16][2];
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      const uint16_t *qp = qbase + static_cast<int64_t>(h0 + (hv ? g : 0)) * q_head_stride + kk * 16 + 2 * t4;
      qa[kk][0] = hv ? __ldg(reinterpret_cast<const uint32_t *>(qp)) : 0u;
      qa[kk][1] = hv ? __ldg(reinterpret_cast<const uint32_t *>(qp + 8)) : 0u;
    }
    float o[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m_run = -INFINITY, l_part = 0.f;
    const int64_t hr_g = head_row(S, layer, h0 + (hv ? g : 0));
    float *ring_row = S.ring_s + (hr_g * S.window + slot) * S.row_cap;
    const int m8 = lane >> 3, r8 = lane & 7;
    for (int i = grp; i < n_my; i += NG) {
      const int st = i % NST;
      const KmTile x = km_tile<KM_TILE>(t_begin + i, t_a, geo);
      // this tile's working-set ids (ring_ids of compressed rows): prefetched for the
      // first MAXPF tiles, else fetched before the data wait
      const int kt = (i - grp) / NG;
      int id = kt == 0 ? id_pf[0] : kt == 1 ? id_pf[1] : kt == 2 ? id_pf[2] : id_pf[3];
      if (kt >= MAXPF && compressed == 1 && lane < RPW && wr0 + lane < x.valid)
        id = x.seg_a ? __ldg(S.sel_ids + hr0 * S.budget_cap + x.row0 + wr0 + lane) : x.row0 + wr0 + lane;
      tc::mbar_wait(&full[st], (i / NST) & 1);
      if (rec && tid == 0 && i == 0) rec[2] = gtime();
      const uint32_t ks = tc::smem_u32(sm + st * L::TILE_B), vs = tc::smem_u32(sm + L::OFF_V + st * L::TILE_B);
      if (x.valid < wr0 + RPW) {
        // rows past the working set hold other (finite or not) data: zero this warp's V rows (P = 0 there)
        unsigned char *vt = sm + L::OFF_V + st * L::TILE_B;
        for (int e = lane; e < RPW * (D / 8); e += 32) {
          const int r = wr0 + e / (D / 8), c = e % (D / 8);
          if (r >= x.valid) *reinterpret_cast<uint4 *>(vt + km_off<KM_TILE>(r, c)) = make_uint4(0, 0, 0, 0);
        }
        tc::fence_proxy_async();  // the stage is refilled by TMA (async proxy) later
        __syncwarp();
      }
      if constexpr (SWAP) {
        // one q-head: the K / V tiles are the A operands and q / P the B
        // column (n = 0), halving the MMAs of the m16 q-row form (15 of whose 16
        // A rows are zero). S^T = K q^T: C rows = this warp's 16 key rows;
        // column 0 (lanes t4 == 0) holds rows g (c0) and g + 8 (c2). The
        // B-operand ldmatrix fragments of the q-row form are the A fragments
        // here with the middle pair swapped; k-steps in the same two chains.
        uint32_t fb[D / 16][4];
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          ldsm_x4(fb[kk], ks + km_off<KM_TILE>(wr0 + (m8 >> 1) * 8 + r8, 2 * kk + (m8 & 1)));
        float cs[4] = {0.f, 0.f, 0.f, 0.f}, cd[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int kk = 0; kk < D / 16; kk += 2) {
          mma_16816_a4(cs, fb[kk][0], fb[kk][2], fb[kk][1], fb[kk][3], qa[kk][0], qa[kk][1]);
          mma_16816_a4(cd, fb[kk + 1][0], fb[kk + 1][2], fb[kk + 1][1], fb[kk + 1][3], qa[kk + 1][0], qa[kk + 1][1]);
        }
        cs[0] += cd[0];
        cs[2] += cd[2];
        // V^T fragments (ldmatrix.trans; A = dims x rows) in flight while the softmax runs
#pragma unroll
        for (int np = 0; np < D / 16; ++np)
          ldsm_x4_t(fb[np], vs + km_off<KM_TILE>(wr0 + (m8 & 1) * 8 + r8, 2 * np + (m8 >> 1)));
        const bool col0 = t4 == 0;
        const int ra = wr0 + g, rb = wr0 + g + 8;
        const float xa = col0 && ra < x.valid ? cs[0] * scale_log2 : -INFINITY;
        const float xb = col0 && rb < x.valid ? cs[2] * scale_log2 : -INFINITY;
        if (col0) {  // raw logits to the ring (columns j0 + r)
          if (ra < x.valid) ring_row[x.j0 + ra] = xa;
          if (rb < x.valid) ring_row[x.j0 + rb] = xb;
        }
        if (compressed == 1 && lane < RPW && wr0 + lane < x.valid)
          S.ring_ids[(head_row(S, layer, h0) * S.window + slot) * S.sparse_cap + x.j0 + wr0 + lane] = id;
        float tmax = fmaxf(xa, xb);
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 4));
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 8));
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 16));
        const float m_new = fmaxf(m_run, tmax);
        float pa = 0.f, pb = 0.f, corr = 1.f;
        if (m_new != -INFINITY) {
          corr = m_run == -INFINITY ? 0.f : fast_exp2(m_run - m_new);
          pa = xa == -INFINITY ? 0.f : fast_exp2(xa - m_new);
          pb = xb == -INFINITY ? 0.f : fast_exp2(xb - m_new);
          m_run = m_new;
        }
        l_part = l_part * corr + (pa + pb);
        if (corr != 1.f) {  // (uniform over the warp)
#pragma unroll
          for (int mt = 0; mt < D / 16; ++mt) {
            o[mt][0] *= corr;
            o[mt][2] *= corr;
          }
        }
        // P^T as the B column: lane t4 of row group 0 takes rows 2t4, 2t4+1 (b0)
        // and 8+2t4, 9+2t4 (b1) from the lanes 8 t4 and 8 t4 + 4 that hold them
        const float va = __shfl_sync(0xffffffffu, pa, 8 * t4), vb = __shfl_sync(0xffffffffu, pa, 8 * t4 + 4);
        const float vc = __shfl_sync(0xffffffffu, pb, 8 * t4), vd = __shfl_sync(0xffffffffu, pb, 8 * t4 + 4);
        const uint32_t b0 = g == 0 ? pack_bf16(va, vb) : 0u, b1 = g == 0 ? pack_bf16(vc, vd) : 0u;
        // O^T += V^T P^T: m-tile mt = dims [16 mt, +16); column 0 in lanes t4 == 0
#pragma unroll
        for (int mt = 0; mt < D / 16; ++mt) mma_16816_a4(o[mt], fb[mt][0], fb[mt][2], fb[mt][1], fb[mt][3], b0, b1);
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&empty[st]);
        if (rec && tid == 0 && i < 4) rec[11 + i] = gtime();
        continue;
      }
      // S = Q K^T over this warp's rows (n-tile n = rows wr0 + 8n .. +7)
      // (all fragment loads first, then the MMAs in two independent chains per n-tile)
      uint32_t fb[D / 16][4];
      float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      float sd[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      if constexpr (RPW == 16) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) ldsm_x4(fb[kk], ks + km_off<KM_TILE>(wr0 + (m8 >> 1) * 8 + r8, 2 * kk + (m8 & 1)));
#pragma unroll
        for (int kk = 0; kk < D / 16; kk += 2) {
          mma_16816(sc[0], qa[kk][0], qa[kk][1], fb[kk][0], fb[kk][1]);
          mma_16816(sc[1], qa[kk][0], qa[kk][1], fb[kk][2], fb[kk][3]);
          mma_16816(sd[0], qa[kk + 1][0], qa[kk + 1][1], fb[kk + 1][0], fb[kk + 1][1]);
          mma_16816(sd[1], qa[kk + 1][0], qa[kk + 1][1], fb[kk + 1][2], fb[kk + 1][3]);
        }
      } else {
        // 8 rows: one x4 load = the rows' chunks 4kp..4kp+3 = two k-steps of the one n-tile
#pragma unroll
        for (int kp = 0; kp < D / 32; ++kp) ldsm_x4(fb[kp], ks + km_off<KM_TILE>(wr0 + r8, 4 * kp + m8));
#pragma unroll
        for (int kp = 0; kp < D / 32; ++kp) {
          mma_16816(sc[0], qa[2 * kp][0], qa[2 * kp][1], fb[kp][0], fb[kp][1]);
          mma_16816(sd[0], qa[2 * kp + 1][0], qa[2 * kp + 1][1], fb[kp][2], fb[kp][3]);
        }
      }
#pragma unroll
      for (int n = 0; n < NTS; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) sc[n][e] += sd[n][e];
      // V fragments in flight while the softmax runs
      if constexpr (RPW == 16) {
#pragma unroll
        for (int np = 0; np < D / 16; ++np)
          ldsm_x4_t(fb[np], vs + km_off<KM_TILE>(wr0 + (m8 & 1) * 8 + r8, 2 * np + (m8 >> 1)));
      } else {
        // 8 rows (k 0-7; k 8-15 of the m16n8k16 step are zero): x4.trans = 4 dim n-tiles
#pragma unroll
        for (int nq = 0; nq < D / 32; ++nq) ldsm_x4_t(fb[nq], vs + km_off<KM_TILE>(wr0 + r8, 4 * nq + m8));
      }
      // logits (log2 units); rows past the working set -> -inf
      float xs[2][2] = {{-INFINITY, -INFINITY}, {-INFINITY, -INFINITY}};
      float tmax = -INFINITY;
#pragma unroll
      for (int n = 0; n < NTS; ++n)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = wr0 + n * 8 + 2 * t4 + e;
          xs[n][e] = r < x.valid ? sc[n][e] * scale_log2 : -INFINITY;
          tmax = fmaxf(tmax, xs[n][e]);
        }
      // raw logits to the ring (head g, columns j0 + r)
      if (hv) {
#pragma unroll
        for (int n = 0; n < NTS; ++n) {
          const int r = wr0 + n * 8 + 2 * t4;
          if (r < x.valid) ring_row[x.j0 + r] = xs[n][0];
          if (r + 1 < x.valid) ring_row[x.j0 + r + 1] = xs[n][1];
        }
      }
      if (compressed == 1 && lane < RPW && wr0 + lane < x.valid) {  // (2: ids derived by K7)
        const int r = wr0 + lane;
#pragma unroll
        for (int gg = 0; gg < G; ++gg)
          S.ring_ids[(head_row(S, layer, h0 + gg) * S.window + slot) * S.sparse_cap + x.j0 + r] = id;
      }
      // online softmax of this warp's rows (row g of the quad)
      tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
      tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
      const float m_new = fmaxf(m_run, tmax);
      float p[2][2];
      float corr = 1.f;
      if (m_new == -INFINITY || !hv) {
        p[0][0] = p[0][1] = p[1][0] = p[1][1] = 0.f;
      } else {
        corr = m_run == -INFINITY ? 0.f : fast_exp2(m_run - m_new);
#pragma unroll
        for (int n = 0; n < 2; ++n)
#pragma unroll
          for (int e = 0; e < 2; ++e) p[n][e] = (n >= NTS || xs[n][e] == -INFINITY) ? 0.f : fast_exp2(xs[n][e] - m_new);
        m_run = m_new;
      }
      l_part = l_part * corr + ((p[0][0] + p[0][1]) + (p[1][0] + p[1][1]));
      if (__any_sync(0xffffffffu, corr != 1.f)) {
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          o[n][0] *= corr;
          o[n][1] *= corr;
        }
      }
      const uint32_t pa0 = pack_bf16(p[0][0], p[0][1]), pa2 = pack_bf16(p[1][0], p[1][1]);
      // O += P V (B = this warp's V rows)
      if constexpr (RPW == 16) {
#pragma unroll
        for (int np = 0; np < D / 16; ++np) {
          mma_16816(o[2 * np], pa0, pa2, fb[np][0], fb[np][1]);
          mma_16816(o[2 * np + 1], pa0, pa2, fb[np][2], fb[np][3]);
        }
      } else {
#pragma unroll
        for (int nq = 0; nq < D / 32; ++nq)
#pragma unroll
          for (int m = 0; m < 4; ++m) mma_16816(o[4 * nq + m], pa0, 0u, fb[nq][m], 0u);
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&empty[st]);
      if (rec && tid == 0 && i < 4) rec[11 + i] = gtime();
    }
    if (rec && tid == 0) {
      rec[3] = gtime();
      rec[5] = n_my;
    }
    // quad sum of the row's softmax denominator (swapped form: the column-0 lanes)
    if constexpr (SWAP) {
      l_part += __shfl_xor_sync(0xffffffffu, l_part, 4);
      l_part += __shfl_xor_sync(0xffffffffu, l_part, 8);
      l_part += __shfl_xor_sync(0xffffffffu, l_part, 16);
    } else {
      l_part += __shfl_xor_sync(0xffffffffu, l_part, 1);
      l_part += __shfl_xor_sync(0xffffffffu, l_part, 2);
    }
    // (A) every consumer warp is done with the stage buffers (the producer warp
    // issued its last TMA long before; every tile was waited on by a consumer)
    tc::named_sync(1, 32 * KM_WARPS);
    float *wm = reinterpret_cast<float *>(sm);  // [W][8]
    float *wl = wm + KM_WARPS * 8;              // [W][8]
    float *wo = wl + KM_WARPS * 8;              // [W][8][D]
    if constexpr (SWAP) {  // O^T column 0: lane 4g holds dims 16 mt + g (c0) and 16 mt + 8 + g (c2)
      if (lane == 0) {
        wm[warp * 8] = m_run;
        wl[warp * 8] = l_part;
      }
      if (t4 == 0) {
#pragma unroll
        for (int mt = 0; mt < D / 16; ++mt) {
          wo[warp * 8 * D + 16 * mt + g] = o[mt][0];
          wo[warp * 8 * D + 16 * mt + 8 + g] = o[mt][2];
        }
      }
    } else if (hv) {
      if (t4 == 0) {
        wm[warp * 8 + g] = m_run;
        wl[warp * 8 + g] = l_part;
      }
#pragma unroll
      for (int n = 0; n < NT; ++n)
        *reinterpret_cast<float2 *>(wo + (warp * 8 + g) * D + n * 8 + 2 * t4) = make_float2(o[n][0], o[n][1]);
    }
  }
  __syncthreads();  // (B) warp partials written
  // ---- this CTA's partial (M, L, O) per head, warps merged in order -> global
  {
    float *wm = reinterpret_cast<float *>(sm);
    float *wl = wm + KM_WARPS * 8;
    float *wo = wl + KM_WARPS * 8;
    float *part = S.partials + static_cast<int64_t>(unit) * n_split * G * (D + 2);
    float *gl = reinterpret_cast<float *>(sm + L::OFF_GATHER);  // rank 0's gather area (cluster mode)
    const bool solo = n_split == 1;  // the unit's only CTA: its merged partial is the result
    float *dst = ccombine == 1 || solo ? gl : part + split * G * (D + 2);  // rank 0 keeps its own partial locally
    uint32_t rgl = 0, rbar = 0;
    if (ccombine == 1) {
      asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
      asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rgl) : "r"(tc::smem_u32(gl)));
      asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rbar) : "r"(tc::smem_u32(&gbar)));
    }
    // per-warp scale factors once per head, then every element is an unrolled
    // sum of independent shared loads
    float *wsw = wo + KM_WARPS * 8 * D;  // [W][8]
    float *wM = wsw + KM_WARPS * 8;      // [8]
    if (tid < G) {
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < KM_WARPS; ++w) M = fmaxf(M, wm[w * 8 + tid]);
#pragma unroll
      for (int w = 0; w < KM_WARPS; ++w) {
        const float mw = wm[w * 8 + tid];
        wsw[w * 8 + tid] = mw == -INFINITY ? 0.f : fast_exp2(mw - M);
      }
      wM[tid] = M;
    }
    __syncthreads();
    for (int i = tid; i < G * (D + 2); i += KM_THREADS) {
      const int gg = i / (D + 2), e = i % (D + 2);
      float acc = 0.f;
      if (e > 0) {
#pragma unroll
        for (int w = 0; w < KM_WARPS; ++w)
          acc = fmaf(wsw[w * 8 + gg], e == 1 ? wl[w * 8 + gg] : wo[(w * 8 + gg) * D + e - 2], acc);
      }
      const float val = e == 0 ? wM[gg] : acc;
      if (ccombine == 1 && split != 0)  // straight into rank 0's gather area, counted on its mbarrier
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                         rgl + 4u * static_cast<uint32_t>(split * G * (D + 2) + i)),
                     "r"(__float_as_uint(val)), "r"(rbar)
                     : "memory");
      else
        dst[i] = val;
    }
    if (rec && tid == 0) rec[4] = gtime();
    int o_begin = 0, o_end = G * D;  // output elements this CTA writes
    bool write_meta = true;
    if (solo) {
      __syncthreads();  // no other split: combine straight from shared memory
      part = gl;
    } else if (ccombine == 1) {
      // the other splits' partials arrive by st.async on rank 0's mbarrier: no
      // cluster barrier (whose release would wait for every CTA's global stores)
      if (split != 0) return;
      __syncthreads();  // rank 0's own partial
      if (tid == 0) tc::mbar_wait(&gbar, 0);
      __syncthreads();
      part = gl;
    } else if (ccombine == 2) {
      // every CTA of the grid is resident (checked at launch): all splits wait
      // for the unit's last partial, then each combines its own slice of the
      // outputs -- no single-CTA tail
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        atomicAdd(S.counters + unit, 1);
        const volatile int *arr = S.counters + unit;
        long long t0 = -1;
        unsigned n = 0;
        while (*arr < n_split) {
          __nanosleep(32);
          if ((++n & 1023u) == 0u) {  // a protocol bug traps instead of hanging the device
            const long long now = clock64();
            if (t0 < 0) t0 = now;
            else if (now - t0 > 20000000000LL) __trap();
          }
        }
      }
      __syncthreads();
      __threadfence();
      if (rec && tid == 0) rec[9] = gtime();
      const int per = (G * D + n_split - 1) / n_split;
      o_begin = min(G * D, split * per);
      o_end = min(G * D, o_begin + per);
      write_meta = split == 0;
    } else {
      __threadfence();
      if (rec && tid == 0) rec[8] = gtime();
      __syncthreads();
      if (tid == 0) is_last = atomicAdd(S.counters + unit, 1) == n_split - 1;
      if (rec && tid == 0) rec[9] = gtime();
      __syncthreads();
      if (!is_last) return;
      __threadfence();
      if (rec && tid == 0) rec[10] = gtime();
      // every split's partial into shared memory in one round of independent
      // L2 loads (the combine below would otherwise chain n_split round trips)
      const int n_el = n_split * G * (D + 2);
      if (n_el * 4 <= 2 * NST * L::TILE_B) {
        float *stg = reinterpret_cast<float *>(sm);
        constexpr int B = 16;  // independent loads in flight per thread
        if ((G * (D + 2)) % 4 == 0) {  // 16-B loads: every partial block is 16-B aligned
          const float4 *src4 = reinterpret_cast<const float4 *>(part);
          float4 *stg4 = reinterpret_cast<float4 *>(stg);
          const int n4 = n_el / 4;
          for (int i0 = tid; i0 < n4; i0 += KM_THREADS * B) {
            float4 v[B];
#pragma unroll
            for (int u = 0; u < B; ++u) {
              const int i = i0 + u * KM_THREADS;
              v[u] = i < n4 ? __ldcg(src4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < B; ++u) {
              const int i = i0 + u * KM_THREADS;
              if (i < n4) stg4[i] = v[u];
            }
          }
        } else
        for (int i0 = tid; i0 < n_el; i0 += KM_THREADS * B) {
          float v[B];
#pragma unroll
          for (int u = 0; u < B; ++u) {
            const int i = i0 + u * KM_THREADS;
            v[u] = i < n_el ? __ldcg(part + i) : 0.f;
          }
#pragma unroll
          for (int u = 0; u < B; ++u) {
            const int i = i0 + u * KM_THREADS;
            if (i < n_el) stg[i] = v[u];
          }
        }
        __syncthreads();
        part = stg;
      }
    }
    if (rec && tid == 0) rec[7] = gtime();
    // ---- last CTA of the unit (or cluster rank 0): combine the splits in split order
    const bool in_smem = __isShared(part);
    auto ldp = [&](const float *x) { return in_smem ? *x : __ldcg(x); };  // shared or L2
    for (int gg = warp; gg < G; gg += KM_WARPS + 1) {  // warp per head, lane r: splits r and r + 32
      float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
      if (lane < n_split) {
        m0 = ldp(part + (lane * G + gg) * (D + 2));
        l0 = ldp(part + (lane * G + gg) * (D + 2) + 1);
      }
      if (lane + 32 < n_split) {
        m1 = ldp(part + ((lane + 32) * G + gg) * (D + 2));
        l1 = ldp(part + ((lane + 32) * G + gg) * (D + 2) + 1);
      }
      const float M = warp_max(fmaxf(m0, m1));
      const float w0 = m0 == -INFINITY ? 0.f : fast_exp2(m0 - M);
      const float w1 = m1 == -INFINITY ? 0.f : fast_exp2(m1 - M);
      if (lane < n_split) wsc[gg * KM_MAX_SPLIT + lane] = w0;
      if (lane + 32 < n_split) wsc[gg * KM_MAX_SPLIT + lane + 32] = w1;
      const float Lsum = warp_sum(fmaf(l0, w0, l1 * w1));
      if (lane == 0) {
        mg[gg] = M;
        mg[8 + gg] = Lsum;
      }
    }
    __syncthreads();
    for (int i = o_begin + tid; i < o_end; i += KM_THREADS) {
      const int gg = i / D, e = i % D;
      float acc = 0.f;
#pragma unroll 8
      for (int r = 0; r < n_split; ++r)
        acc = fmaf(wsc[gg * KM_MAX_SPLIT + r], ldp(part + (r * G + gg) * (D + 2) + 2 + e), acc);
      const float res = acc / mg[8 + gg];
      const int64_t oi = static_cast<int64_t>(h0 + gg) * D + e;
      if (out_bf16)
        reinterpret_cast<uint16_t *>(out)[oi] = f2bf(res);
      else
        reinterpret_cast<float *>(out)[oi] = res;
    }
    if (write_meta && tid < G) {
      const int64_t hr = head_row(S, layer, h0 + tid);
      S.ring_ml[(hr * S.window + slot) * 2 + 0] = mg[tid];
      S.ring_ml[(hr * S.window + slot) * 2 + 1] = mg[8 + tid];
      S.ring_n[hr * S.window + slot] = geo.n_cols;
      S.ring_dense[hr * S.window + slot] = compressed == 2 ? LS_RING_WORKING_SET : compressed ? 0 : 1;
      if (compressed == 2) {  // the row's ids follow from the current selection: n_a and the window start
        S.ring_ids[(hr * S.window + slot) * S.sparse_cap + 0] = geo.n_a;
        S.ring_ids[(hr * S.window + slot) * S.sparse_cap + 1] = geo.lo;
      }
    }
    if (ccombine == 0 && !solo && tid == 0) S.counters[unit] = 0;  // ticket re-armed for the next launch
    if (ccombine == 2) {
      // departures: the last CTA to leave re-arms both counters (every CTA has
      // stopped polling the arrival count by then)
      __syncthreads();
      if (tid == 0 && atomicAdd(S.counters + S.n_heads + unit, 1) == n_split - 1) {
        S.counters[unit] = 0;
        S.counters[S.n_heads + unit] = 0;
      }
    }
    if (rec && tid == 0) rec[6] = gtime();
  }
}

// step[0] += 1, step[1] += rows; and the working-set split point n_a of every
// (layer, q-head) follows the window start lo = max(0, length - W) one up
// (an id equal to the old lo moves below the window)
__global__ void advance_kernel(ls_decode_stack S, int rows) {
  const int length = S.step[0];
  for (int hr = blockIdx.x * blockDim.x + threadIdx.x; hr < S.n_layers * S.n_heads; hr += gridDim.x * blockDim.x) {
    const int lo_old = max(0, length - S.window), lo_new = max(0, length + 1 - S.window);
    if (lo_new != lo_old) {
      const int na = S.n_a[hr];
      if (na < S.n_sel[hr] && S.sel_ids[static_cast<int64_t>(hr) * S.budget_cap + na] == lo_old) S.n_a[hr] = na + 1;
    }
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    S.step[0] = length + 1;
    S.step[1] += rows;
  }
}


// ------------------------------------------------------------------ K7
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
  for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) tot += sh[i];
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
  for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) tot += sh[i];
  __syncthreads();
  return tot;
}

// exclusive prefix of v over the block (thread order); *tot = block total
__device__ int block_excl_scan(int v, int *sh, int *tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
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
  for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) {
    if (i < wid) before += sh[i];
    all += sh[i];
  }
  *tot = all;
  return before + incl - v;
}

__device__ int block_rank(int flag, int *sh, int *tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned b = __ballot_sync(0xffffffffu, flag);
  __syncthreads();
  if (lane == 0) sh[wid] = __popc(b);
  __syncthreads();
  // every warp scans the (<= 32) warp counts with shuffles: one shared load per lane
  const int c = lane < static_cast<int>(blockDim.x >> 5) ? sh[lane] : 0;
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  *tot = __shfl_sync(0xffffffffu, incl, 31);
  return __shfl_sync(0xffffffffu, incl - c, wid) + __popc(b & ((1u << lane) - 1u));
}

__device__ __forceinline__ int gtime32() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return static_cast<int>(t & 0x7fffffffull);
}

// ------------------------------------------------------------------ K7, working-set events
// Every event after the first one buffers only rows that decode_mma_kernel wrote
// as LS_RING_WORKING_SET (interval >= window): row r covers the current picks
// below its window start, sel_ids[0, na_r), then the positions [lo_r, L_r]. The
// touched ids are then known without a bitmap: candidates c < n0 (= na of the
// oldest row) are sel_ids[c], the rest are the positions lo_0 + (c - n0) up to
// the newest row's end, and every one of them is touched (the windows overlap).
// A CTA (256 threads, ~cap * 12 B of shared memory) owns candidates, adds the
// rows' weights oldest -> newest in fp64 (the reference's order,
// kvcompress.py:75-79), finds the B-th (score desc, id asc) key by a radix select and
// writes the picks as select_kernel does (same scores and picks; the coverage
// masses summed over another thread partition). A (layer, head) whose rows are not all
// working-set rows, or with more than `cap` candidates, is left to
// select_kernel, which skips the heads handled here.
struct WsEvent {
  bool ok;
  int n_rows, n0, lo0, n_cand;
};
// called by every thread of the block (thread r reads row r's record; one round trip)
__device__ WsEvent ws_event(const ls_decode_stack &S, int64_t hr, int cap) {
  __shared__ int w_first[2], w_last_end;
  WsEvent e;
  const int appended = S.step[1];
  e.n_rows = min(S.window, appended);
  const int r = threadIdx.x;
  bool mine = true;
  if (r < e.n_rows) {
    const int64_t so = hr * S.window + (appended - e.n_rows + r) % S.window;
    const int kind = __ldg(S.ring_dense + so);
    const int na = __ldg(S.ring_ids + so * S.sparse_cap), lo = __ldg(S.ring_ids + so * S.sparse_cap + 1);
    const int n = __ldg(S.ring_n + so);
    mine = kind == LS_RING_WORKING_SET;
    if (r == 0) {
      w_first[0] = na;
      w_first[1] = lo;
    }
    if (r == e.n_rows - 1) w_last_end = lo + (n - na) - 1;  // the newest row's last position
  }
  e.ok = __syncthreads_and(mine) && e.n_rows > 0 && e.n_rows <= K7_DMAX;
  if (e.ok) {
    e.n0 = w_first[0];
    e.lo0 = w_first[1];
    e.n_cand = e.n0 + (w_last_end - e.lo0 + 1);
    e.ok = e.n_cand <= cap;
  }
  __syncthreads();  // the records may be reused by the next call
  return e;
}

// id of working-set column j of a LS_RING_WORKING_SET row (decode_mma_kernel's
// column order): the first n_a picked ids, then the archive window from lo
__device__ __forceinline__ int working_id(const ls_decode_stack &S, int64_t hr, int na, int lo, int j) {
  return j < na ? __ldg(S.sel_ids + hr * S.budget_cap + j) : lo + (j - na);
}

__global__ void __launch_bounds__(K7_THREADS) select_kernel(ls_decode_stack S, int budget, double *acc_ws,
                                                            uint32_t *touched_ws, int use_smem, int32_t *retained_n,
                                                            double *score_cov, int *dbg, int ws_cap) {
  extern __shared__ __align__(16) unsigned char smem7[];
  __shared__ int hist[256];
  __shared__ int shi[32];
  __shared__ double shd[32];
  __shared__ int s_digit, s_above;
  const int h = blockIdx.x, layer = blockIdx.y;
  const int64_t hr = head_row(S, layer, h);
  if (ws_cap > 0 && ws_event(S, hr, ws_cap).ok) return;  // handled by select_ws_kernel (same test)
  const int length = S.step[0];
  const int appended = S.step[1];
  const int n_rows = min(S.window, appended);
  const int words = (length + 31) / 32;
  double *acc = use_smem ? reinterpret_cast<double *>(smem7) : acc_ws + hr * S.row_cap;
  uint32_t *touched =
      use_smem ? reinterpret_cast<uint32_t *>(smem7 + static_cast<size_t>(K7_SMEM_CAP) * 8)
               : touched_ws + hr * ((S.row_cap + 31) / 32);
  int *rec = (dbg && threadIdx.x == 0) ? dbg + (static_cast<int64_t>(layer) * gridDim.x + h) * 16 : nullptr;
  if (rec) rec[0] = gtime32();
  for (int i = threadIdx.x; i < length; i += blockDim.x) acc[i] = 0.0;
  for (int i = threadIdx.x; i < words; i += blockDim.x) touched[i] = 0u;
  __syncthreads();
  if (rec) rec[1] = gtime32();
  // accumulate rows oldest -> newest (kvcompress.py:75-79). Rows of up to
  // K7_PF * blockDim columns (every compressed row) are fetched K7_RB rows at
  // a time into registers (one round of independent loads), then added in row
  // order; longer (dense) rows stream.
  auto row_weight = [](float sv, float M, float Lr, float inv) {
    return (Lr == 0.f) ? sv : fast_exp2(sv - M) * inv;  // Lr == 0: stored probabilities (seeds)
  };
  // every buffered row dense (the first event: seed rows + dense steps): id j is
  // owned by one thread, which adds the rows in order from registers -- all of
  // a chunk's row values are loaded at once and no block barrier runs per row
  __shared__ int64_t d_so[K7_DMAX];
  __shared__ int d_n[K7_DMAX], d_dense[K7_DMAX], d_na[K7_DMAX], d_lo[K7_DMAX];
  __shared__ float d_m[K7_DMAX], d_l[K7_DMAX], d_inv[K7_DMAX];
  __shared__ int d_all;
  if (threadIdx.x == 0) d_all = n_rows <= K7_DMAX;
  __syncthreads();
  if (threadIdx.x < n_rows && threadIdx.x < K7_DMAX) {
    const int64_t so = hr * S.window + (appended - n_rows + static_cast<int>(threadIdx.x)) % S.window;
    d_so[threadIdx.x] = so;
    d_n[threadIdx.x] = S.ring_n[so];
    d_m[threadIdx.x] = S.ring_ml[so * 2];
    d_l[threadIdx.x] = S.ring_ml[so * 2 + 1];
    d_inv[threadIdx.x] = d_l[threadIdx.x] > 0.f ? 1.f / d_l[threadIdx.x] : 0.f;
    d_dense[threadIdx.x] = S.ring_dense[so];
    if (d_dense[threadIdx.x] == LS_RING_WORKING_SET) {
      d_na[threadIdx.x] = S.ring_ids[so * S.sparse_cap + 0];
      d_lo[threadIdx.x] = S.ring_ids[so * S.sparse_cap + 1];
    }
    if (d_dense[threadIdx.x] != 1) d_all = 0;
  }
  __syncthreads();
  const bool all_dense = d_all != 0;
  if (all_dense) {
    int max_n = 0;
    for (int rr = 0; rr < n_rows; ++rr) max_n = max(max_n, d_n[rr]);
    for (int j = threadIdx.x; j < max_n; j += blockDim.x) {
      double a = 0.0;
      bool t = false;
      for (int c0 = 0; c0 < n_rows; c0 += K7_DCH) {
        float sv[K7_DCH];
#pragma unroll
        for (int u = 0; u < K7_DCH; ++u) {
          const int rr = c0 + u;
          sv[u] = (rr < n_rows && j < d_n[rr]) ? __ldg(S.ring_s + d_so[rr] * S.row_cap + j) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < K7_DCH; ++u) {
          const int rr = c0 + u;
          if (rr < n_rows && j < d_n[rr]) {
            a += static_cast<double>(row_weight(sv[u], d_m[rr], d_l[rr], d_inv[rr]));
            t = true;
          }
        }
      }
      acc[j] = a;  // == 0.0 + w_0 + w_1 + ... in row order, as the row-by-row adds
      if (t) atomicOr(touched + (j >> 5), 1u << (j & 31));
    }
    __syncthreads();
  }
  for (int r0 = 0; r0 < (all_dense ? 0 : n_rows); r0 += K7_RB) {
    const int nr = min(K7_RB, n_rows - r0);
    // row metadata of the round (one round trip: slots are always valid indices)
    int64_t so_r[K7_RB];
    int n_r[K7_RB], dense_r[K7_RB], na_r[K7_RB], lo_r[K7_RB];
    float m_r[K7_RB], l_r[K7_RB];
    int nmax = 0;
#pragma unroll
    for (int rr = 0; rr < K7_RB; ++rr) {
      const int R = r0 + rr;
      if (R < K7_DMAX) {  // staged in shared memory above
        so_r[rr] = d_so[R];
        n_r[rr] = d_n[R];
        dense_r[rr] = d_dense[R];
        na_r[rr] = d_na[R];
        lo_r[rr] = d_lo[R];
        m_r[rr] = d_m[R];
        l_r[rr] = d_l[R];
      } else {
        so_r[rr] = hr * S.window + (appended - n_rows + R) % S.window;
        n_r[rr] = __ldg(S.ring_n + so_r[rr]);
        dense_r[rr] = __ldg(S.ring_dense + so_r[rr]);
        na_r[rr] = __ldg(S.ring_ids + so_r[rr] * S.sparse_cap + 0);
        lo_r[rr] = __ldg(S.ring_ids + so_r[rr] * S.sparse_cap + 1);
        m_r[rr] = __ldg(S.ring_ml + so_r[rr] * 2);
        l_r[rr] = __ldg(S.ring_ml + so_r[rr] * 2 + 1);
      }
    }
#pragma unroll
    for (int rr = 0; rr < K7_RB; ++rr) {
      if (rr >= nr) n_r[rr] = 0;
      nmax = max(nmax, n_r[rr]);
    }
    if (rec && r0 == 0) rec[8] = gtime32();
    if (nmax <= K7_PF * static_cast<int>(blockDim.x)) {
      // the round's columns (second round trip), then the adds in row order
      float sv_r[K7_RB][K7_PF];
      int iv[K7_RB][K7_PF];
#pragma unroll
      for (int rr = 0; rr < K7_RB; ++rr)
#pragma unroll
        for (int e = 0; e < K7_PF; ++e) {
          const int j = threadIdx.x + e * blockDim.x;
          const bool ok = j < n_r[rr];
          iv[rr][e] = !ok                                   ? -1
                      : dense_r[rr] == 1                    ? j
                      : dense_r[rr] == LS_RING_WORKING_SET  ? working_id(S, hr, na_r[rr], lo_r[rr], j)
                                                            : __ldg(S.ring_ids + so_r[rr] * S.sparse_cap + j);
          sv_r[rr][e] = ok ? __ldg(S.ring_s + so_r[rr] * S.row_cap + j) : 0.f;
        }
      if (rec && r0 == 0) rec[9] = gtime32() + 0 * __float_as_int(sv_r[0][0]) + 0 * iv[0][0];
#pragma unroll
      for (int rr = 0; rr < K7_RB; ++rr) {
        if (rr < nr) {
          const float inv = l_r[rr] > 0.f ? 1.f / l_r[rr] : 0.f;
#pragma unroll
          for (int e = 0; e < K7_PF; ++e) {
            const int id = iv[rr][e];
            if (id >= 0) {
              acc[id] += static_cast<double>(row_weight(sv_r[rr][e], m_r[rr], l_r[rr], inv));
              atomicOr(touched + (id >> 5), 1u << (id & 31));
            }
          }
          __syncthreads();
        }
      }
    } else {
      for (int rr = 0; rr < nr; ++rr) {
        const int64_t so = hr * S.window + (appended - n_rows + r0 + rr) % S.window;
        const int n = S.ring_n[so];
        const int dense = S.ring_dense[so];
        const float M = S.ring_ml[so * 2], Lr = S.ring_ml[so * 2 + 1];
        const float inv = Lr > 0.f ? 1.f / Lr : 0.f;
        const float *sr = S.ring_s + so * S.row_cap;
        const int32_t *ids = S.ring_ids + so * S.sparse_cap;
        const int na = ids[0], lo = ids[1];
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
          const int id = dense == 1 ? j : dense == LS_RING_WORKING_SET ? working_id(S, hr, na, lo, j) : ids[j];
          acc[id] += static_cast<double>(row_weight(sr[j], M, Lr, inv));
          atomicOr(touched + (id >> 5), 1u << (id & 31));
        }
        __syncthreads();
      }
    }
  }
  if (rec) rec[2] = gtime32();
  int cnt = 0;
  for (int i = threadIdx.x; i < words; i += blockDim.x) cnt += __popc(touched[i]);
  const int n_cand = block_sum_int(cnt, shi);
  // after the first event only ~B + W ids are touched: list them (id order)
  // and run the radix passes and the ranking over the list, not all positions
  int32_t *cand = reinterpret_cast<int32_t *>(smem7 + static_cast<size_t>(K7_SMEM_CAP) * 8 + K7_SMEM_CAP / 8 + 64);
  const bool use_list = use_smem && n_cand <= K7_CAND_CAP;
  if (use_list) {
    int base_c = 0;
    for (int w0 = 0; w0 < words; w0 += blockDim.x) {
      const int w = w0 + threadIdx.x;
      uint32_t x = w < words ? touched[w] : 0u;
      int tot;
      int pos = base_c + block_excl_scan(__popc(x), shi, &tot);
      while (x) {
        const int b = __ffs(x) - 1;
        x &= x - 1;
        cand[pos++] = w * 32 + b;
      }
      base_c += tot;
    }
    __syncthreads();
  }
  if (rec) {
    rec[3] = gtime32();
    rec[7] = n_cand;
  }
  const int n_iter = use_list ? n_cand : length;  // loop domain: list entries or positions
  unsigned long long prefix = 0ull, pmask = 0ull;
  int need = budget;
  const bool take_all = budget >= n_cand;
  // few candidates (every event after the first: ~B + W ids): one bitonic
  // sort of (score desc, id asc) over the list instead of 8 radix passes
  const bool bitonic = use_list && !take_all && n_cand <= K7_BITONIC;
  double sc_reg[K7_BITONIC / K7_THREADS];
  int *flag = nullptr;
  if (bitonic) {
#pragma unroll
    for (int e = 0; e < K7_BITONIC / K7_THREADS; ++e) {
      const int k = threadIdx.x + e * K7_THREADS;
      sc_reg[e] = k < n_cand ? acc[cand[k]] : 0.0;
    }
    __syncthreads();  // the accumulator area is reused below
    unsigned long long *sk = reinterpret_cast<unsigned long long *>(smem7);
    int *sv = reinterpret_cast<int *>(smem7 + K7_BITONIC * 8);
    flag = sv + K7_BITONIC;
#pragma unroll
    for (int e = 0; e < K7_BITONIC / K7_THREADS; ++e) {
      const int k = threadIdx.x + e * K7_THREADS;
      sk[k] = k < n_cand ? ~dkey(sc_reg[e]) : ~0ull;  // ascending key = descending score
      sv[k] = k;                                      // list order = id order: ties by id
      flag[k] = 0;
    }
    __syncthreads();
    for (int size = 2; size <= K7_BITONIC; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int t = threadIdx.x; t < K7_BITONIC / 2; t += K7_THREADS) {
          const int i = 2 * t - (t & (stride - 1)), j = i + stride;
          const bool up = (i & size) == 0;
          const unsigned long long ki = sk[i], kj = sk[j];
          const int vi = sv[i], vj = sv[j];
          const bool gt = ki > kj || (ki == kj && vi > vj);
          if (gt == up) {
            sk[i] = kj;
            sk[j] = ki;
            sv[i] = vj;
            sv[j] = vi;
          }
        }
        __syncthreads();
      }
    }
    for (int t = threadIdx.x; t < budget; t += K7_THREADS) flag[sv[t]] = 1;
    __syncthreads();
  }
  if (!take_all && !bitonic) {
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      for (int k = threadIdx.x; k < n_iter; k += blockDim.x) {
        const int i = use_list ? cand[k] : k;
        if (!use_list && !((touched[i >> 5] >> (i & 31)) & 1u)) continue;
        const unsigned long long key = dkey(acc[i]);
        if ((key & pmask) != prefix) continue;
        atomicAdd(&hist[(key >> shift) & 0xff], 1);
      }
      __syncthreads();
      if (threadIdx.x < 32) {  // warp scan from the top digit down
        const int lane = threadIdx.x;
        int c[8], loc = 0;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          c[t] = hist[255 - (lane * 8 + t)];
          loc += c[t];
        }
        int incl = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const int excl = incl - loc;  // count above this lane's 8 digits
        const bool hit = excl < need && incl >= need;
        const unsigned hb = __ballot_sync(0xffffffffu, hit);
        if (lane == __ffs(hb) - 1) {
          int above = excl;
          for (int t = 0; t < 8; ++t) {
            if (above + c[t] >= need) {
              s_digit = 255 - (lane * 8 + t);
              s_above = above;
              break;
            }
            above += c[t];
          }
        }
      }
      __syncthreads();
      prefix |= static_cast<unsigned long long>(s_digit) << shift;
      pmask |= 0xffull << shift;
      need -= s_above;
      __syncthreads();
    }
  }
  if (rec) rec[4] = gtime32();
  const unsigned long long thr = prefix;
  int32_t *sel = S.sel_ids + hr * S.budget_cap;
  int base = 0, eq_seen = 0;
  double tot_mass = 0.0, kept_mass = 0.0;
  int in_window_picked = 0;
  const int lo = max(0, length - S.window);
  for (int i0 = 0; i0 < n_iter; i0 += blockDim.x) {
    const int k = i0 + threadIdx.x;
    const int i = use_list ? (k < n_iter ? cand[k] : length) : k;
    int is_t = 0, is_eq = 0, is_gt = 0;
    double scv = 0.0;
    if (bitonic) {
      if (k < n_cand) {
        is_t = 1;
        scv = sc_reg[i0 / K7_THREADS];
      }
    } else if (i < length && (use_list || ((touched[i >> 5] >> (i & 31)) & 1u))) {
      is_t = 1;
      scv = acc[i];
      if (!take_all) {
        const unsigned long long key = dkey(scv);
        is_gt = key > thr;
        is_eq = key == thr;
      }
    }
    int eq_tot;
    const int eq_rank = block_rank(is_eq, shi, &eq_tot);
    const int pick = take_all ? is_t : bitonic ? (is_t && flag[k]) : (is_gt || (is_eq && eq_seen + eq_rank < need));
    int pick_tot;
    const int rank = block_rank(pick, shi, &pick_tot);
    if (pick) sel[base + rank] = i;
    if (is_t) {
      tot_mass += scv;
      if (pick || i >= lo) kept_mass += scv;  // kvcompress.py:215 (working = picked U recent)
    }
    if (pick && i >= lo) in_window_picked += 1;
    base += pick_tot;
    eq_seen += eq_tot;
  }
  if (rec) rec[5] = gtime32();
  const double T = block_sum_double(tot_mass, shd);
  const double Kp = block_sum_double(kept_mass, shd);
  const int iw = block_sum_int(in_window_picked, shi);
  {
    // working-set split point for this step: picked ids below the window start
    int below = 0;
    for (int j = threadIdx.x; j < base; j += blockDim.x) below += sel[j] < lo ? 1 : 0;
    below = block_sum_int(below, shi);
    if (threadIdx.x == 0) S.n_a[hr] = below;
  }
  if (threadIdx.x == 0) {
    S.n_sel[hr] = base;
    if (retained_n) retained_n[hr] = base + (length - lo) - iw;
    if (score_cov) score_cov[hr] = T > 0 ? Kp / T : 1.0;
  }
  if (rec) rec[6] = gtime32();
}

constexpr int K7W_THREADS = 256;  // small CTAs: four per SM keep the sort's barriers overlapped
__global__ void __launch_bounds__(K7W_THREADS) select_ws_kernel(ls_decode_stack S, int budget, int cap,
                                                               int32_t *retained_n, double *score_cov) {
  extern __shared__ __align__(16) unsigned char smws[];
  __shared__ int shi[32];
  __shared__ double shd[32];
  __shared__ int hist[256];
  __shared__ int s_digit, s_above;
  __shared__ int64_t r_so[K7_DMAX];
  __shared__ int r_na[K7_DMAX], r_lo[K7_DMAX], r_end[K7_DMAX];
  __shared__ float r_m[K7_DMAX], r_inv[K7_DMAX];
  const int h = blockIdx.x, layer = blockIdx.y;
  const int64_t hr = head_row(S, layer, h);
  const WsEvent e = ws_event(S, hr, cap);
  if (!e.ok) return;
  const int n_rows = e.n_rows, n0 = e.n0, lo0 = e.lo0, n_cand = e.n_cand;
  const int length = S.step[0], appended = S.step[1];
  double *acc = reinterpret_cast<double *>(smws);          // [cap] scores
  int32_t *cid = reinterpret_cast<int32_t *>(acc + cap);   // [cap] candidate ids
  int32_t *srank = cid + cap;                              // [window + 1] pick index of a position
  const int32_t *sel_in = S.sel_ids + hr * S.budget_cap;
  if (threadIdx.x < n_rows) {
    const int r = threadIdx.x;
    const int64_t so = hr * S.window + (appended - n_rows + r) % S.window;
    r_so[r] = so;
    r_na[r] = S.ring_ids[so * S.sparse_cap];
    r_lo[r] = S.ring_ids[so * S.sparse_cap + 1];
    r_end[r] = r_lo[r] + (S.ring_n[so] - r_na[r]) - 1;
    r_m[r] = S.ring_ml[so * 2];
    const float l = S.ring_ml[so * 2 + 1];
    r_inv[r] = l > 0.f ? 1.f / l : 0.f;  // (select_kernel's row weight)
  }
  __syncthreads();
  // positions below a later row's window start appear in it only if picked:
  // srank[p - lo0] = the pick's column there (its index in sel_ids), or -1
  const int span = r_lo[n_rows - 1] - lo0;
  for (int p = threadIdx.x; p < span; p += blockDim.x) srank[p] = -1;
  __syncthreads();
  for (int k = n0 + threadIdx.x; k < r_na[n_rows - 1]; k += blockDim.x) srank[sel_in[k] - lo0] = k;
  __syncthreads();
  // scores: one thread per candidate, rows oldest -> newest in fp64
  for (int c = threadIdx.x; c < n_cand; c += blockDim.x) {
    const int p = c < n0 ? -1 : lo0 + (c - n0);
    cid[c] = c < n0 ? sel_in[c] : p;
    double a = 0.0;
    for (int r0 = 0; r0 < n_rows; r0 += K7_RB) {
      float v[K7_RB];
      bool in[K7_RB];
#pragma unroll
      for (int u = 0; u < K7_RB; ++u) {  // the round's loads first
        const int r = r0 + u;
        int j = -1;
        if (r < n_rows) {
          if (c < n0) j = c;
          else if (p >= r_lo[r]) j = p <= r_end[r] ? r_na[r] + (p - r_lo[r]) : -1;
          else j = srank[p - lo0];
        }
        in[u] = j >= 0;
        v[u] = in[u] ? __ldg(S.ring_s + r_so[r] * S.row_cap + j) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < K7_RB; ++u)
        if (in[u]) a += static_cast<double>(fast_exp2(v[u] - r_m[r0 + u]) * r_inv[r0 + u]);
    }
    acc[c] = a;
  }
  __syncthreads();
  const bool take_all = budget >= n_cand;
  // the B-th key of (score desc, id asc) by an MSD radix select over the
  // candidates (8-bit digits of the monotone fp64 key): picks are keys above
  // it plus the lowest-id `need` of the keys equal to it (candidate order is id order)
  unsigned long long prefix = 0ull, pmask = 0ull;
  int need = budget;
  if (!take_all) {
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      for (int k = threadIdx.x; k < n_cand; k += blockDim.x) {
        const unsigned long long key = dkey(acc[k]);
        if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 0xff], 1);
      }
      __syncthreads();
      if (threadIdx.x < 32) {  // warp scan from the top digit down
        const int lane = threadIdx.x;
        int cnt[8], loc = 0;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          cnt[t] = hist[255 - (lane * 8 + t)];
          loc += cnt[t];
        }
        int incl = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const int excl = incl - loc;
        const unsigned hb = __ballot_sync(0xffffffffu, excl < need && incl >= need);
        if (lane == __ffs(hb) - 1) {
          int above = excl;
          for (int t = 0; t < 8; ++t) {
            if (above + cnt[t] >= need) {
              s_digit = 255 - (lane * 8 + t);
              s_above = above;
              break;
            }
            above += cnt[t];
          }
        }
      }
      __syncthreads();
      prefix |= static_cast<unsigned long long>(s_digit) << shift;
      pmask |= 0xffull << shift;
      need -= s_above;
      __syncthreads();
    }
  }
  // picks in id order + the event-log fields, as select_kernel (the coverage
  // masses are fp64 sums over a different thread partition: equal up to rounding)
  int32_t *sel = S.sel_ids + hr * S.budget_cap;
  int base = 0, eq_seen = 0;
  double tot_mass = 0.0, kept_mass = 0.0;
  int in_window_picked = 0;
  const int lo = max(0, length - S.window);
  for (int i0 = 0; i0 < n_cand; i0 += blockDim.x) {
    const int k = i0 + threadIdx.x;
    const int is_t = k < n_cand;
    const int id = is_t ? cid[k] : length;
    const double scv = is_t ? acc[k] : 0.0;
    const unsigned long long key = dkey(scv);
    const int is_gt = is_t && !take_all && key > prefix, is_eq = is_t && !take_all && key == prefix;
    int eq_tot;
    const int eq_rank = block_rank(is_eq, shi, &eq_tot);
    const int pick = take_all ? is_t : (is_gt || (is_eq && eq_seen + eq_rank < need));
    eq_seen += eq_tot;
    int pick_tot;
    const int rank = block_rank(pick, shi, &pick_tot);
    if (pick) sel[base + rank] = id;
    if (is_t) {
      tot_mass += scv;
      if (pick || id >= lo) kept_mass += scv;  // kvcompress.py:215 (working = picked U recent)
    }
    if (pick && id >= lo) in_window_picked += 1;
    base += pick_tot;
  }
  const double T = block_sum_double(tot_mass, shd);
  const double Kp = block_sum_double(kept_mass, shd);
  const int iw = block_sum_int(in_window_picked, shi);
  {
    int below = 0;
    for (int j = threadIdx.x; j < base; j += blockDim.x) below += sel[j] < lo ? 1 : 0;
    below = block_sum_int(below, shi);
    if (threadIdx.x == 0) S.n_a[hr] = below;
  }
  if (threadIdx.x == 0) {
    S.n_sel[hr] = base;
    if (retained_n) retained_n[hr] = base + (length - lo) - iw;
    if (score_cov) score_cov[hr] = T > 0 ? Kp / T : 1.0;
  }
}

// ------------------------------------------------------------------ K8
__global__ void compact_kernel(ls_decode_stack S, const uint16_t *k, const uint16_t *v) {
  const int h = blockIdx.y, layer = blockIdx.z;
  const int d = S.head_dim;
  const int vec = d / 8;
  const int64_t hr = head_row(S, layer, h);
  const int n = S.n_sel[hr];
  const int kv = h / (S.n_heads / S.n_kv_heads);
  const int32_t *sel = S.sel_ids + hr * S.budget_cap;
  const int64_t base = static_cast<int64_t>(layer) * S.kv_layer_stride + static_cast<int64_t>(kv) * S.kv_head_stride;
  const uint4 *kb = reinterpret_cast<const uint4 *>(k + base);
  const uint4 *vb = reinterpret_cast<const uint4 *>(v + base);
  uint4 *ck = reinterpret_cast<uint4 *>(S.ck + hr * S.budget_cap * d);
  uint4 *cv = reinterpret_cast<uint4 *>(S.cv + hr * S.budget_cap * d);
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

static int check_stack(const ls_decode_stack *S) {
  LS_REQUIRE(S->head_dim == 64 || S->head_dim == 128, LS_ERR_UNSUPPORTED, "head_dim must be 64 or 128");
  LS_REQUIRE(S->n_heads > 0 && S->n_kv_heads > 0 && S->n_heads % S->n_kv_heads == 0, LS_ERR_DIMENSION_MISMATCH,
             "n_heads must be a multiple of n_kv_heads");
  LS_REQUIRE(S->window >= 1, LS_ERR_INVALID_CONFIG, "obs_window must be >= 1");
  LS_REQUIRE(S->sparse_cap >= S->budget_cap + S->window + 1, LS_ERR_INVALID_CONFIG,
             "sparse_cap must be >= budget_cap + window + 1");
  return LS_OK;
}

// split count = cluster size: the splits of a unit combine through DSMEM.
// 16 (non-portable) when the device accepts it, else 8; never more than the
// tiles of the longest row.
template <int D, int G>
static int launch_decode(int units, int max_cols, cudaStream_t st, const ls_decode_stack *S, int layer,
                         const uint16_t *q, int64_t q_head_stride, int q_from_archive, const uint16_t *k,
                         const uint16_t *v, int compressed, float sl, void *out, int out_bf16, int pdl) {
  const int smem = dec::k6_smem_bytes<D>(G);
  static_assert(2 * dec::K6_STAGES * dec::K6_TILE * D * 2 >= (4 * G * D + dec::k6_max_cluster(G) * G * (D + 2)) * 4,
                "gather + reduction buffers must fit in the tile buffers");
  static int max_cluster = 0;
  if (!max_cluster) {
    max_cluster = 8;
    if (dec::k6_max_cluster(G) > 8 &&
        cudaFuncSetAttribute(dec::decode_kernel<D, G>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess)
      max_cluster = dec::k6_max_cluster(G);
    cudaGetLastError();
  }
  LS_CUDA(cudaFuncSetAttribute(dec::decode_kernel<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  // compressed steps: 8-CTA clusters (enough splits for ~1K columns, best
  // co-scheduling); dense steps stream the whole archive: up to 16
  const int cl = compressed ? std::min(8, max_cluster) : max_cluster;
  const int n_split = std::max(1, std::min(cl, ceil_div(max_cols, dec::K6_TILE)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_split, units, 1);
  cfg.blockDim = dim3(dec::K6_THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = n_split;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  LS_CUDA(cudaLaunchKernelEx(&cfg, dec::decode_kernel<D, G>, *S, layer, q, q_head_stride, q_from_archive, k, v,
                             compressed, sl, out, out_bf16, pdl));
  return LS_OK;
}

namespace ls {
int make_tmap_bf16_3d_box(CUtensorMap *m, const void *base, int d, int64_t rows, int heads, int64_t row_stride_el,
                          int64_t head_stride_el, int box_rows);
}

template <int D, int G>
static int launch_decode_mma(int units, int max_cols, cudaStream_t st, const ls_decode_stack *S, int layer,
                             const uint16_t *q, int64_t q_head_stride, int q_from_archive, const uint16_t *k,
                             const uint16_t *v, int compressed, float sl, void *out, int out_bf16, int pdl) {
  LS_REQUIRE(S->partials != nullptr && S->counters != nullptr, LS_ERR_WORKSPACE,
             "decode stack without partials / counters (see ls_decode_partials_size)");
  // dense steps stream the archive: two groups of 4 consumer warps on
  // alternate 64-row tiles, 4 stages, one CTA per SM; compressed steps (~17 x
  // 64 rows per head): 4 warps, 3 stages, two CTAs per SM (the next layer's
  // CTAs start their prefetch beside this layer's). Measured: tools/sweep_dec.sh
#ifndef LS_K6_NST_C
#define LS_K6_NST_C 3
#endif
#ifndef LS_K6_NST_D
#define LS_K6_NST_D 4
#endif
#ifndef LS_K6_NG_D
#define LS_K6_NG_D 2
#endif
#ifndef LS_K6_NG_C
#define LS_K6_NG_C 1
#endif
#ifndef LS_K6_RPW_C
#define LS_K6_RPW_C 16
#endif
  constexpr int RPW_C = LS_K6_RPW_C, RPW_D = 16;
  constexpr int NST_D = LS_K6_NST_D, NW_D = 4, NG_D = LS_K6_NG_D, NST_C = LS_K6_NST_C, NW_C = 64 / RPW_C,
                NG_C = LS_K6_NG_C;
  const int tile = compressed ? RPW_C * NW_C : RPW_D * NW_D;
  dec::KmMaps maps;
  const int HR = S->n_layers * S->n_heads;
  const int64_t rows = S->kv_head_stride / D;
  int r = make_tmap_bf16_3d_box(&maps.ck, S->ck, D, S->budget_cap, HR, D, static_cast<int64_t>(S->budget_cap) * D,
                                tile);
  if (!r) r = make_tmap_bf16_3d_box(&maps.cv, S->cv, D, S->budget_cap, HR, D,
                                    static_cast<int64_t>(S->budget_cap) * D, tile);
  if (!r) r = make_tmap_bf16_3d_box(&maps.k, k, D, rows, S->n_kv_heads, D, S->kv_head_stride, tile);
  if (!r) r = make_tmap_bf16_3d_box(&maps.v, v, D, rows, S->n_kv_heads, D, S->kv_head_stride, tile);
  if (r) return r;
  // compressed steps split into a few tiles per CTA run a 2-stage ring (smaller
  // CTAs: one more fits an SM beside the next layer's); one CTA per unit streams
  // its whole working set through NST_C stages (measured: C2 196 -> 190 us/step)
  constexpr int NST_S = 2;
  constexpr int smem_d = dec::KmSmem<D, NST_D, NW_D, NG_D, RPW_D>::TOTAL, smem_c = dec::KmSmem<D, NST_C, NW_C, NG_C, RPW_C>::TOTAL,
                smem_s = dec::KmSmem<D, NST_S, NW_C, NG_C, RPW_C>::TOTAL;
  static bool attr_set = false;
  if (!attr_set) {
    LS_CUDA(cudaFuncSetAttribute(dec::decode_mma_kernel<D, G, NST_D, NW_D, NG_D, RPW_D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem_d));
    LS_CUDA(cudaFuncSetAttribute(dec::decode_mma_kernel<D, G, NST_C, NW_C, NG_C, RPW_C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem_c));
    LS_CUDA(cudaFuncSetAttribute(dec::decode_mma_kernel<D, G, NST_S, NW_C, NG_C, RPW_C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem_s));
    attr_set = true;
  }
  static int n_sm = 0;
  if (!n_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (n_sm <= 0) n_sm = 148;
  }
  // splits: fill the resident CTA slots (2 per SM at this shared-memory size);
  // compressed steps: ~3 tiles per split while the units leave slots free, one
  // split per unit once they fill the GPU (C4: 8 sessions x 28 q-heads = 224
  // units -> one CTA streams a head's whole working set, no combine; measured
  // 3.25 -> 4.57 TB/s)
  static const int env_split_dense = getenv("LS_K6_SPLIT_DENSE") ? atoi(getenv("LS_K6_SPLIT_DENSE")) : 0;
  static const int env_split_comp = getenv("LS_K6_SPLIT_COMP") ? atoi(getenv("LS_K6_SPLIT_COMP")) : 0;
  static const int env_cta_mult = getenv("LS_K6_CTAS_PER_SM") ? atoi(getenv("LS_K6_CTAS_PER_SM")) : 1;
  static const bool env_no_cluster = getenv("LS_K6_NO_CLUSTER") != nullptr;
  const int env_split = compressed ? env_split_comp : env_split_dense;
  const int tiles = ceil_div(max_cols, tile) + 1;  // + the segment boundary
  // dense: one CTA per SM; compressed: ~3 tiles per split (one cluster per unit)
  int n_split = env_split > 0 ? env_split
                : compressed ? std::max(1, std::min({8, ceil_div(tiles, 3), 2 * n_sm / units}))
                             : std::max(1, env_cta_mult * n_sm / units);
  n_split = std::max(1, std::min({n_split, tiles, dec::KM_MAX_SPLIT}));
  // splits combine in rank 0's shared memory when they fit one portable cluster
  static const bool env_dense_cluster = getenv("LS_K6_DENSE_CLUSTER") != nullptr;
  static int max_cl = 0;
  if (!max_cl) {  // 16-CTA clusters need the non-portable opt-in
    max_cl = 8;
    if (cudaFuncSetAttribute(dec::decode_mma_kernel<D, G, NST_D, NW_D, NG_D, RPW_D>,
                             cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess)
      max_cl = 16;
    cudaGetLastError();
  }
  if (!compressed && env_dense_cluster && env_split <= 0) n_split = std::min(n_split, max_cl);
  const int cl_cap = compressed ? 8 : max_cl;
  const int gather_b = compressed ? dec::km_gather_b(NG_C) : dec::km_gather_b(NG_D);
  int ccombine = !env_no_cluster && n_split > 1 && n_split <= cl_cap && n_split * G * (D + 2) * 4 <= gather_b;
  if (!ccombine && n_split > 1) {
    // all splits wait for each other only if every CTA of the grid is resident
    static int resident_d = -1, resident_c = -1;
    int &res = compressed ? resident_c : resident_d;
    if (res < 0) {
      int per_sm = 0;
      if (compressed)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dec::decode_mma_kernel<D, G, NST_C, NW_C, NG_C, RPW_C>,
                                                      32 * (NW_C * NG_C + 1), smem_c);
      else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dec::decode_mma_kernel<D, G, NST_D, NW_D, NG_D, RPW_D>,
                                                      32 * (NW_D * NG_D + 1), smem_d);
      cudaGetLastError();
      res = per_sm * n_sm;
    }
    // (measured at C2: no faster than the last-CTA combine; LS_K6_ALL_CTA=1 selects it)
    static const bool env_all_cta = getenv("LS_K6_ALL_CTA") != nullptr;
    if (env_all_cta && n_split * units <= res) ccombine = 2;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_split, units, 1);
  cfg.blockDim = dim3(32 * ((compressed ? NW_C * NG_C : NW_D * NG_D) + 1), 1, 1);
  const bool short_ring = compressed && n_split > 1 && NG_C == 1;
  cfg.dynamicSmemBytes = short_ring ? smem_s : compressed ? smem_c : smem_d;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (ccombine == 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = n_split;  // (ccombine == 1 only)
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  if (short_ring)
    LS_CUDA(cudaLaunchKernelEx(&cfg, dec::decode_mma_kernel<D, G, NST_S, NW_C, NG_C, RPW_C>, maps, *S, layer, q, q_head_stride,
                               q_from_archive, compressed, sl, out, out_bf16, pdl, ccombine, g_debug_buffer));
  else if (compressed)
    LS_CUDA(cudaLaunchKernelEx(&cfg, dec::decode_mma_kernel<D, G, NST_C, NW_C, NG_C, RPW_C>, maps, *S, layer, q, q_head_stride,
                               q_from_archive, compressed, sl, out, out_bf16, pdl, ccombine, g_debug_buffer));
  else
    LS_CUDA(cudaLaunchKernelEx(&cfg, dec::decode_mma_kernel<D, G, NST_D, NW_D, NG_D, RPW_D>, maps, *S, layer, q, q_head_stride,
                               q_from_archive, compressed, sl, out, out_bf16, pdl, ccombine, g_debug_buffer));
  return LS_OK;
}

// tensor-core K6 when the stack carries split-K partials; LS_K6_SIMT=1 selects
// the CUDA-core form (cluster combine), kept as the cross-check
template <int D, int G>
static int launch_k6(int units, int max_cols, cudaStream_t st, const ls_decode_stack *S, int layer, const uint16_t *q,
                     int64_t q_head_stride, int q_from_archive, const uint16_t *k, const uint16_t *v, int compressed,
                     float sl, void *out, int out_bf16, int pdl) {
  static const bool simt = getenv("LS_K6_SIMT") != nullptr;
  if (!simt && S->partials != nullptr && S->counters != nullptr)
    return launch_decode_mma<D, G>(units, max_cols, st, S, layer, q, q_head_stride, q_from_archive, k, v, compressed,
                                   sl, out, out_bf16, pdl);
  return launch_decode<D, G>(units, max_cols, st, S, layer, q, q_head_stride, q_from_archive, k, v, compressed, sl,
                             out, out_bf16, pdl);
}

extern "C" size_t ls_decode_partials_size(const ls_decode_stack *S, int32_t max_len) {
  (void)max_len;  // [unit][split][G][D + 2] floats: units x G = n_heads for every step kind
  return S ? static_cast<size_t>(S->n_heads) * dec::KM_MAX_SPLIT * (S->head_dim + 2) * sizeof(float) : 0;
}

static int decode_step_impl(const ls_decode_stack *S, int32_t layer, const uint16_t *q, int64_t q_head_stride,
                            int q_from_archive, const uint16_t *k_layer, const uint16_t *v_layer, int32_t compressed,
                            int32_t max_cols, void *out, int32_t out_bf16, int pdl, ls_stream_t stream) {
  int c = check_stack(S);
  if (c) return c;
  LS_REQUIRE(layer >= 0 && layer < S->n_layers, LS_ERR_DIMENSION_MISMATCH, "layer out of range");
  LS_REQUIRE(max_cols >= 1 && max_cols <= S->row_cap, LS_ERR_SEQUENCE_TOO_LONG,
             "max_cols %d exceeds the ring row capacity %d", max_cols, S->row_cap);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const float sl = kLog2e / sqrtf(static_cast<float>(S->head_dim));
  const int group = S->n_heads / S->n_kv_heads;
  int r = LS_OK;
#define LS_ARGS q, q_head_stride, q_from_archive, k_layer, v_layer
  // dense steps: one unit per kv-head with its whole q-group (each K/V row read
  // once); LS_DECODE_DENSE_PER_HEAD=1 splits them per q-head (measured slower)
  static const bool env_dense_per_head = getenv("LS_DECODE_DENSE_PER_HEAD") != nullptr;  // read once
  const bool per_head = compressed || env_dense_per_head;
  if (per_head) {
    r = S->head_dim == 128
            ? launch_k6<128, 1>(S->n_heads, max_cols, st, S, layer, LS_ARGS, compressed, sl, out, out_bf16, pdl)
            : launch_k6<64, 1>(S->n_heads, max_cols, st, S, layer, LS_ARGS, compressed, sl, out, out_bf16, pdl);
  } else {
#define LS_DENSE(DD, GG) \
  r = launch_k6<DD, GG>(S->n_kv_heads, max_cols, st, S, layer, LS_ARGS, 0, sl, out, out_bf16, pdl)
    if (S->head_dim == 128) {
      if (group == 1) LS_DENSE(128, 1);
      else if (group == 2) LS_DENSE(128, 2);
      else if (group == 4) LS_DENSE(128, 4);
      else if (group == 7) LS_DENSE(128, 7);
      else if (group == 8) LS_DENSE(128, 8);
      else LS_REQUIRE(false, LS_ERR_UNSUPPORTED, "GQA group size %d", group);
    } else {
      if (group == 1) LS_DENSE(64, 1);
      else if (group == 2) LS_DENSE(64, 2);
      else if (group == 4) LS_DENSE(64, 4);
      else LS_REQUIRE(false, LS_ERR_UNSUPPORTED, "GQA group size %d", group);
    }
#undef LS_DENSE
  }
#undef LS_ARGS
  if (r) return r;
  LS_LAUNCH_CHECK("decode_kernel");
  return LS_OK;
}

extern "C" int ls_decode_step(const ls_decode_stack *S, int32_t layer, const uint16_t *q, const uint16_t *k_layer,
                              const uint16_t *v_layer, int32_t compressed, int32_t max_cols, void *out,
                              int32_t out_bf16, ls_stream_t stream) {
  return decode_step_impl(S, layer, q, S->head_dim, 0, k_layer, v_layer, compressed, max_cols, out, out_bf16, 0,
                          stream);
}

extern "C" int ls_decode_step_archive(const ls_decode_stack *S, int32_t layer, const uint16_t *q_layer,
                                      int64_t q_head_stride, const uint16_t *k_layer, const uint16_t *v_layer,
                                      int32_t compressed, int32_t max_cols, void *out, int32_t out_bf16,
                                      int32_t flags, ls_stream_t stream) {
  // LS_DECODE_DERIVED_IDS: compressed rows record (n_a, lo) instead of their ids
  const int32_t kind = compressed && (flags & LS_DECODE_DERIVED_IDS) ? 2 : compressed ? 1 : 0;
  return decode_step_impl(S, layer, q_layer, q_head_stride, 1, k_layer, v_layer, kind, max_cols, out, out_bf16,
                          (flags & LS_DECODE_PDL) ? 1 : 0, stream);
}

extern "C" int ls_decode_advance(const ls_decode_stack *S, ls_stream_t stream) {
  dec::advance_kernel<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(*S, 1);
  LS_LAUNCH_CHECK("advance_kernel");
  return LS_OK;
}

extern "C" size_t ls_decode_select_workspace(const ls_decode_stack *S) {
  return static_cast<size_t>(S->n_layers) * S->n_heads *
             (static_cast<size_t>(S->row_cap) * 8 + (S->row_cap + 31) / 32 * 4) + 1024;
}

extern "C" int ls_decode_event(const ls_decode_stack *S, int32_t budget, int32_t max_len, const uint16_t *k_all,
                               const uint16_t *v_all, int32_t *retained_n, double *score_coverage, void *ws,
                               size_t ws_bytes, ls_stream_t stream) {
  int c = check_stack(S);
  if (c) return c;
  LS_REQUIRE(budget >= 1 && budget <= S->budget_cap, LS_ERR_INVALID_CONFIG, "budget outside [1, budget_cap]");
  LS_REQUIRE(max_len <= S->row_cap, LS_ERR_SEQUENCE_TOO_LONG, "length exceeds row_cap");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool smem = max_len <= dec::K7_SMEM_CAP;
  double *acc = nullptr;
  uint32_t *touched = nullptr;
  if (!smem) {
    LS_REQUIRE(ws_bytes >= ls_decode_select_workspace(S), LS_ERR_WORKSPACE, "decode_event workspace too small");
    Carver cv(ws, ws_bytes);
    acc = cv.take<double>(static_cast<size_t>(S->n_layers) * S->n_heads * S->row_cap);
    touched = cv.take<uint32_t>(static_cast<size_t>(S->n_layers) * S->n_heads * ((S->row_cap + 31) / 32));
  }
  const size_t dyn =
      smem ? static_cast<size_t>(dec::K7_SMEM_CAP) * 8 + dec::K7_SMEM_CAP / 8 + 64 + dec::K7_CAND_CAP * 4 : 0;
  if (dyn > 48 * 1024)
    LS_CUDA(cudaFuncSetAttribute(dec::select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)));
  // working-set events (all buffered rows LS_RING_WORKING_SET, <= ws_cap candidates:
  // budget + 2 window) first; select_kernel takes the other heads
  int ws_cap = 1;
  while (ws_cap < budget + 2 * S->window + 2) ws_cap <<= 1;
  static const bool env_no_ws = getenv("LS_K7_NO_WS") != nullptr;  // (A/B: select_kernel for every head)
  if (ws_cap > 4096 || S->window >= dec::K7_DMAX || env_no_ws) ws_cap = 0;
  if (ws_cap > 0) {
    const size_t dyn_ws = static_cast<size_t>(ws_cap) * 12 + static_cast<size_t>(S->window + 2) * 4;
    if (dyn_ws > 48 * 1024)
      LS_CUDA(cudaFuncSetAttribute(dec::select_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(dyn_ws)));
    dec::select_ws_kernel<<<dim3(S->n_heads, S->n_layers), dec::K7W_THREADS, dyn_ws, st>>>(*S, budget, ws_cap,
                                                                                          retained_n, score_coverage);
    LS_LAUNCH_CHECK("select_ws_kernel");
  }
  dec::select_kernel<<<dim3(S->n_heads, S->n_layers), dec::K7_THREADS, dyn, st>>>(*S, budget, acc, touched, smem ? 1 : 0,
                                                                                   retained_n, score_coverage, g_debug_buffer,
                                                                                   ws_cap);
  LS_LAUNCH_CHECK("select_kernel");
  dec::compact_kernel<<<dim3(16, S->n_heads, S->n_layers), 256, 0, st>>>(*S, k_all, v_all);
  LS_LAUNCH_CHECK("compact_kernel");
  return LS_OK;
}
