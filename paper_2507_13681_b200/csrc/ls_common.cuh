// Shared device helpers for the LoopServe B200 kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/loopserve_b200.h"

namespace ls {

void set_error(const char *fmt, ...);
int32_t *device_status_ptr();  // capi.cu: device validation status word (ls_device_status)

// record a reference error found on the device (first one wins)
__device__ __forceinline__ void report_status(int32_t *status, int32_t code) {
  if (status) atomicCAS(status, 0, code);
}
int cuda_status(cudaError_t e, const char *where);

#define LS_CUDA(call)                                          \
  do {                                                         \
    cudaError_t _e = (call);                                   \
    if (_e != cudaSuccess) return ::ls::cuda_status(_e, #call); \
  } while (0)

#define LS_LAUNCH_CHECK(name)                                     \
  do {                                                            \
    cudaError_t _e = cudaGetLastError();                          \
    if (_e != cudaSuccess) return ::ls::cuda_status(_e, name);    \
  } while (0)

#define LS_REQUIRE(cond, code, ...)  \
  do {                               \
    if (!(cond)) {                   \
      ::ls::set_error(__VA_ARGS__);  \
      return (code);                 \
    }                                \
  } while (0)

constexpr float kLog2e = 1.4426950408889634f;
constexpr int kWarp = 32;

__device__ __forceinline__ float bf2f(uint16_t b) {
  return __uint_as_float(static_cast<uint32_t>(b) << 16);
}

__device__ __forceinline__ uint16_t f2bf(float f) {
  __nv_bfloat16 h = __float2bfloat16_rn(f);
  return *reinterpret_cast<uint16_t *>(&h);
}

// unpack 8 bf16 from a 16-byte vector
__device__ __forceinline__ void bf16x8_to_f32(const uint4 &u, float *f) {
  f[0] = __uint_as_float(u.x << 16);
  f[1] = __uint_as_float(u.x & 0xffff0000u);
  f[2] = __uint_as_float(u.y << 16);
  f[3] = __uint_as_float(u.y & 0xffff0000u);
  f[4] = __uint_as_float(u.z << 16);
  f[5] = __uint_as_float(u.z & 0xffff0000u);
  f[6] = __uint_as_float(u.w << 16);
  f[7] = __uint_as_float(u.w & 0xffff0000u);
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// packed fp32 pairs on the FMA pipe (FFMA2 / FADD2, sm_100): one issue slot per two lanes' worth
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long *>(&a)), "l"(*reinterpret_cast<unsigned long long *>(&b)),
        "l"(*reinterpret_cast<unsigned long long *>(&c)));
  return *reinterpret_cast<float2 *>(&r);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long *>(&a)), "l"(*reinterpret_cast<unsigned long long *>(&b)));
  return *reinterpret_cast<float2 *>(&r);
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA / integer pipes (no MUFU): x = n + f, n = round(x) by the
// 1.5 * 2^23 magic add, f in [-0.5, 0.5], 2^f by a degree-3 minimax polynomial
// (max relative error 7.6e-5, far below the bf16 rounding of the P operand it
// feeds); 2^n added to the exponent bits. x < -126 (incl. -inf) gives 0.
// Used for part of the softmax exponentials so the MUFU pipe is not the only
// exp2 unit (the FA4 split).
__device__ __forceinline__ float poly_exp2(float x) {
  const float xc = fmaxf(x, -126.f);
  const float j = __fadd_rn(xc, 12582912.f);
  const float n = __fsub_rn(j, 12582912.f);
  const float f = xc - n;
  float p = fmaf(f, 0.05517053f, 0.24260831f);
  p = fmaf(p, f, 0.69326092f);
  p = fmaf(p, f, 0.99992825f);
  const int bits = __float_as_int(p) + (__float_as_int(j) << 23);
  return x < -126.f ? 0.f : __int_as_float(bits);
}

// 2^x on the FMA / integer pipes at fp32 accuracy: the same range reduction as
// poly_exp2, 2^f on [-0.5, 0.5] by a degree-6 near-minimax polynomial (max
// relative error 1.0e-7 with fp32 Horner, within ex2.approx's 2^-22 bound).
// Lets a share of the exponentials bypass the MUFU / MIO path.
__device__ __forceinline__ float poly6_exp2(float x) {
  const float xc = fmaxf(x, -126.f);
  const float j = __fadd_rn(xc, 12582912.f);
  const float n = __fsub_rn(j, 12582912.f);
  const float f = xc - n;
  float p = fmaf(f, 1.5345795e-4f, 1.3399932e-3f);
  p = fmaf(p, f, 9.6184891e-3f);
  p = fmaf(p, f, 5.5503286e-2f);
  p = fmaf(p, f, 2.4022646e-1f);
  p = fmaf(p, f, 6.9314718e-1f);
  p = fmaf(p, f, 1.0f);
  const int bits = __float_as_int(p) + (__float_as_int(j) << 23);
  return x < -126.f ? 0.f : __int_as_float(bits);
}

// first index i in [0, n) with a[i] >= x (a sorted ascending)
template <typename T>
__device__ __forceinline__ int lower_bound_dev(const T *a, int n, T x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// workspace carving (256-byte aligned bumps)
struct Carver {
  char *base;
  size_t off = 0;
  size_t cap;
  Carver(void *b, size_t c) : base(static_cast<char *>(b)), cap(c) {}
  template <typename T>
  T *take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T *p = reinterpret_cast<T *>(base ? base + off : nullptr);
    off += n * sizeof(T);
    return p;
  }
  bool ok() const { return off <= cap; }
};

inline int ceil_div(int a, int b) { return (a + b - 1) / b; }
inline long long ceil_div_ll(long long a, long long b) { return (a + b - 1) / b; }

}  // namespace ls
