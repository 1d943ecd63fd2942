// K0 -- per-head row sampling, bit-exact with numpy.
//
// Replaces Session.head_seed (reference session.py:84-86) and sample_rows
// (reference prefill.py:125-135). The reference draws
//     SeedSequence(entropy=session_seed, spawn_key=(turn, layer, head))
//         .generate_state(1, uint64)[0]                      -> head seed
//     Generator(PCG64(head_seed)).choice(n_new-1, n_s-1, replace=False)
// and appends the last row. We restate numpy's published algorithms
// (numpy 2.3: bit_generator.pyx SeedSequence hashmix/mix, pcg64.h
// XSL-RR 128/64 with the 32-bit half buffering of next_uint32,
// distributions.c buffered Lemire bounded draws, _generator.pyx choice:
// Floyd's algorithm, or a tail Fisher-Yates shuffle when
// pop > 10000 and size > pop // 50). Only the sampled SET matters (the
// reference sorts), so Floyd's hash set is a bitmap here.
//
// One thread per head: the chain is sequential per head, heads run in
// parallel. The sorted output is produced by scanning the bitmap.

#include "ls_common.cuh"

namespace ls {
namespace sampler {

struct U128 {
  uint64_t hi, lo;
};

__host__ __device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return static_cast<uint64_t>((static_cast<unsigned __int128>(a) * b) >> 64);
#endif
}

__host__ __device__ __forceinline__ U128 mul128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = mulhi64(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}

__host__ __device__ __forceinline__ U128 add128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1u : 0u);
  return r;
}

// SeedSequence constants (numpy bit_generator.pyx)
constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u;
constexpr uint32_t INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
constexpr uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;

__host__ __device__ __forceinline__ uint32_t hashmix(uint32_t v, uint32_t &hc) {
  v ^= hc;
  hc *= MULT_A;
  v *= hc;
  v ^= v >> 16;
  return v;
}

__host__ __device__ __forceinline__ uint32_t mixw(uint32_t x, uint32_t y) {
  uint32_t r = MIX_L * x - MIX_R * y;
  r ^= r >> 16;
  return r;
}

// int -> uint32 words (numpy _int_to_uint32_array)
__host__ __device__ __forceinline__ int coerce_u64(uint64_t n, uint32_t *out) {
  if (n == 0) {
    out[0] = 0;
    return 1;
  }
  int k = 0;
  while (n > 0) {
    out[k++] = static_cast<uint32_t>(n & 0xffffffffu);
    n >>= 32;
  }
  return k;
}

// SeedSequence(entropy, spawn_key).generate_state(n_words32, uint32)
__host__ __device__ inline void seedseq_generate(const uint32_t *run, int n_run, const uint32_t *spawn,
                                                 int n_spawn, uint32_t *out, int n_out) {
  uint32_t ent[16];
  int n = 0;
  for (int i = 0; i < n_run; ++i) ent[n++] = run[i];
  if (n_spawn > 0)
    while (n < 4) ent[n++] = 0;  // gh-16539 padding when a spawn key is present
  for (int i = 0; i < n_spawn; ++i) ent[n++] = spawn[i];
  uint32_t hc = INIT_A;
  uint32_t mixer[4];
  for (int i = 0; i < 4; ++i) mixer[i] = hashmix(i < n ? ent[i] : 0u, hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) mixer[d] = mixw(mixer[d], hashmix(mixer[s], hc));
  for (int s = 4; s < n; ++s)
    for (int d = 0; d < 4; ++d) mixer[d] = mixw(mixer[d], hashmix(ent[s], hc));
  uint32_t hb = INIT_B;
  for (int i = 0; i < n_out; ++i) {
    uint32_t v = mixer[i & 3];
    v ^= hb;
    hb *= MULT_B;
    v *= hb;
    v ^= v >> 16;
    out[i] = v;
  }
}

__host__ __device__ inline uint64_t head_seed(uint64_t session_seed, int turn, int layer, int head) {
  uint32_t run[2], spawn[6], w[2];
  int nr = coerce_u64(session_seed, run);
  int ns = 0;
  ns += coerce_u64(static_cast<uint64_t>(turn), spawn + ns);
  ns += coerce_u64(static_cast<uint64_t>(layer), spawn + ns);
  ns += coerce_u64(static_cast<uint64_t>(head), spawn + ns);
  seedseq_generate(run, nr, spawn, ns, w, 2);
  return static_cast<uint64_t>(w[0]) | (static_cast<uint64_t>(w[1]) << 32);
}

// numpy PCG64 (XSL-RR 128/64) with the next_uint32 half buffer
struct Pcg64 {
  U128 state, inc;
  bool has32;
  uint32_t buf32;

  __host__ __device__ void step() {
    const U128 mult{2549297995355413924ull, 4865540595714422341ull};
    state = add128(mul128(state, mult), inc);
  }
  __host__ __device__ void seed(uint64_t s64) {
    uint32_t run[2], w[8];
    int nr = coerce_u64(s64, run);
    seedseq_generate(run, nr, nullptr, 0, w, 8);
    uint64_t v[4];
    for (int i = 0; i < 4; ++i) v[i] = static_cast<uint64_t>(w[2 * i]) | (static_cast<uint64_t>(w[2 * i + 1]) << 32);
    U128 initstate{v[0], v[1]}, initseq{v[2], v[3]};
    state = U128{0, 0};
    inc.hi = (initseq.hi << 1) | (initseq.lo >> 63);
    inc.lo = (initseq.lo << 1) | 1u;
    step();
    state = add128(state, initstate);
    step();
    has32 = false;
    buf32 = 0;
  }
  __host__ __device__ uint64_t next64() {
    step();
    uint64_t x = state.hi ^ state.lo;
    unsigned rot = static_cast<unsigned>(state.hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  __host__ __device__ uint32_t next32() {
    if (has32) {
      has32 = false;
      return buf32;
    }
    uint64_t n = next64();
    has32 = true;
    buf32 = static_cast<uint32_t>(n >> 32);
    return static_cast<uint32_t>(n & 0xffffffffu);
  }
  // random_bounded_uint64(off=0, rng, mask=0, use_masked=false) for rng < 2^32-1
  __host__ __device__ uint32_t bounded(uint32_t rng) {
    if (rng == 0) return 0;
    const uint32_t excl = rng + 1u;
    uint64_t m = static_cast<uint64_t>(next32()) * excl;
    uint32_t left = static_cast<uint32_t>(m);
    if (left < excl) {
      const uint32_t threshold = (0xffffffffu - rng) % excl;
      while (left < threshold) {
        m = static_cast<uint64_t>(next32()) * excl;
        left = static_cast<uint32_t>(m);
      }
    }
    return static_cast<uint32_t>(m >> 32);
  }
};

__host__ __device__ inline int sample_size(int n_new, double rate, int floor_) {
  double c = rate * static_cast<double>(n_new);
  long long ce = static_cast<long long>(c);
  if (static_cast<double>(ce) < c) ce += 1;  // math.ceil for positive values
  long long m = ce > floor_ ? ce : floor_;
  return static_cast<int>(m < n_new ? m : n_new);
}

// Selects size-1 of pop = n_new-1 into `bits` (pop bits, zeroed), using
// `scratch` (pop int32) for the tail-shuffle branch.
__host__ __device__ inline void choose_into_bitmap(Pcg64 &g, int pop, int size, uint32_t *bits,
                                                   int32_t *scratch) {
  if (size <= 0) return;
  if (pop > 10000 && size > pop / 50) {
    for (int i = 0; i < pop; ++i) scratch[i] = i;
    int first = pop - size > 1 ? pop - size : 1;
    for (int i = pop - 1; i >= first; --i) {
      uint32_t j = g.bounded(static_cast<uint32_t>(i));
      int32_t t = scratch[j];
      scratch[j] = scratch[i];
      scratch[i] = t;
    }
    for (int i = pop - size; i < pop; ++i) {
      int v = scratch[i];
      bits[v >> 5] |= 1u << (v & 31);
    }
  } else {
    for (int j = pop - size; j < pop; ++j) {
      uint32_t val = g.bounded(static_cast<uint32_t>(j));
      bool present = (bits[val >> 5] >> (val & 31)) & 1u;
      uint32_t ins = present ? static_cast<uint32_t>(j) : val;
      bits[ins >> 5] |= 1u << (ins & 31);
    }
  }
}

constexpr int SMEM_WORDS = 512;  // Floyd bitmap in shared memory up to n_new = 16385

// one thread per (layer, head); the Floyd bitmap lives in shared memory
__global__ void __launch_bounds__(32) sample_rows_kernel(uint64_t session_seed, int turn, int layer_begin,
                                                         int n_layers, int head_begin, int n_heads, int n_new,
                                                         int n_s, uint32_t *bits_ws, int32_t *scratch_ws,
                                                         int32_t *out) {
  extern __shared__ uint32_t sbits[];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int pop = n_new - 1;
  const int words = (pop + 31) / 32 > 0 ? (pop + 31) / 32 : 1;
  const bool in_smem = words <= SMEM_WORDS;
  if (t >= n_layers * n_heads) return;
  const int li = t / n_heads, h = t % n_heads;
  uint32_t *bits = in_smem ? sbits + threadIdx.x * words : bits_ws + static_cast<size_t>(t) * words;
  int32_t *scratch = scratch_ws + static_cast<size_t>(t) * (pop > 0 ? pop : 1);
  for (int i = 0; i < words; ++i) bits[i] = 0;
  if (n_s > 1) {
    Pcg64 g;
    g.seed(turn < 0 ? session_seed : head_seed(session_seed, turn, layer_begin + li, head_begin + h));
    choose_into_bitmap(g, pop, n_s - 1, bits, scratch);
  }
  int32_t *o = out + static_cast<size_t>(t) * n_s;
  int k = 0;
  for (int w = 0; w < words; ++w) {
    uint32_t x = bits[w];
    while (x) {
      int b = __ffs(x) - 1;
      x &= x - 1;
      o[k++] = w * 32 + b;
    }
  }
  o[k] = n_new - 1;
}

}  // namespace sampler
}  // namespace ls

using namespace ls;

extern "C" int ls_sample_size(int32_t n_new, double rate, int32_t floor_, int32_t *n_s) {
  LS_REQUIRE(n_new > 0, LS_ERR_EMPTY_BLOCK, "cannot sample rows of an empty block");
  LS_REQUIRE(rate > 0.0 && rate <= 1.0 && floor_ >= 1, LS_ERR_INVALID_CONFIG,
             "need 0 < rate <= 1 and floor >= 1");
  *n_s = sampler::sample_size(n_new, rate, floor_);
  return LS_OK;
}

extern "C" size_t ls_sample_rows_workspace(int32_t n_units, int32_t n_new) {
  size_t pop = n_new > 1 ? static_cast<size_t>(n_new - 1) : 1;
  size_t words = (pop + 31) / 32;
  bool big = words > sampler::SMEM_WORDS || (pop > 10000);
  return 1024 + (big ? static_cast<size_t>(n_units) * (words * 4 + pop * 4) : 0);
}

extern "C" int ls_sample_rows(uint64_t session_seed, int32_t turn, int32_t layer_begin, int32_t n_layers,
                              int32_t head_begin, int32_t n_heads, int32_t n_new, double rate, int32_t floor_,
                              int32_t *out_rows, void *ws, size_t ws_bytes, ls_stream_t stream) {
  int32_t n_s = 0;
  int st = ls_sample_size(n_new, rate, floor_, &n_s);
  if (st) return st;
  const int units = n_layers * n_heads;
  LS_REQUIRE(units > 0, LS_ERR_DIMENSION_MISMATCH, "need at least one (layer, head)");
  LS_REQUIRE(ws_bytes >= ls_sample_rows_workspace(units, n_new), LS_ERR_WORKSPACE,
             "sample_rows workspace too small");
  size_t pop = n_new > 1 ? static_cast<size_t>(n_new - 1) : 1;
  size_t words = (pop + 31) / 32;
  bool big = words > sampler::SMEM_WORDS || (pop > 10000);
  Carver c(ws, ws_bytes);
  uint32_t *bits = big ? c.take<uint32_t>(static_cast<size_t>(units) * words) : nullptr;
  int32_t *scratch = big ? c.take<int32_t>(static_cast<size_t>(units) * pop) : nullptr;
  const int threads = 32;
  const size_t smem = words <= static_cast<size_t>(sampler::SMEM_WORDS) ? threads * words * 4 : 0;
  if (smem > 48 * 1024)
    LS_CUDA(cudaFuncSetAttribute(sampler::sample_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  sampler::sample_rows_kernel<<<ceil_div(units, threads), threads, smem, static_cast<cudaStream_t>(stream)>>>(
      session_seed, turn, layer_begin, n_layers, head_begin, n_heads, n_new, n_s, bits, scratch, out_rows);
  LS_LAUNCH_CHECK("sample_rows_kernel");
  return LS_OK;
}

extern "C" uint64_t ls_head_seed_host(uint64_t session_seed, int32_t turn, int32_t layer, int32_t head) {
  return sampler::head_seed(session_seed, turn, layer, head);
}

extern "C" int ls_sample_rows_host(uint64_t session_seed, int32_t turn, int32_t layer, int32_t head,
                                   int32_t n_new, double rate, int32_t floor_, int32_t *out_rows) {
  int32_t n_s = 0;
  int st = ls_sample_size(n_new, rate, floor_, &n_s);
  if (st) return st;
  int pop = n_new - 1;
  size_t words = pop > 0 ? (pop + 31) / 32 : 1;
  std::string bits_buf(words * 4, '\0');
  std::string scratch_buf(static_cast<size_t>(pop > 0 ? pop : 1) * 4, '\0');
  uint32_t *bits = reinterpret_cast<uint32_t *>(&bits_buf[0]);
  int32_t *scratch = reinterpret_cast<int32_t *>(&scratch_buf[0]);
  if (n_s > 1) {
    sampler::Pcg64 g;
    g.seed(turn < 0 ? session_seed : sampler::head_seed(session_seed, turn, layer, head));
    sampler::choose_into_bitmap(g, pop, n_s - 1, bits, scratch);
  }
  int k = 0;
  for (size_t w = 0; w < words; ++w)
    for (int b = 0; b < 32; ++b)
      if ((bits[w] >> b) & 1u) out_rows[k++] = static_cast<int32_t>(w * 32 + b);
  out_rows[k] = n_new - 1;
  return LS_OK;
}
