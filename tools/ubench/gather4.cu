// TMA tile::gather4 on sm_100a: 4 arbitrary rows of a [rows][128] bf16 matrix,
// two 64-column boxes, 128-B swizzle, into a 1024-B aligned tile laid out as
// [2][8 rows][128 B] (rows 4..7 from a second gather4); checks that the bytes
// land where a regular 64-row box load would put rows with the same slot index
// (chunk c of slot r at (c ^ (r & 7)) * 16). Diagnostics only.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
__global__ void k(const __grid_constant__ CUtensorMap m, const int *rows, uint16_t *out) {
  __shared__ __align__(1024) unsigned char s[2 * 8 * 128];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(s));
  const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(2 * 8 * 128) : "memory");
    for (int h = 0; h < 2; ++h)
      for (int g = 0; g < 2; ++g)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
                d + h * 1024 + g * 512),
            "l"(&m), "r"(h * 64), "r"(rows[4 * g]), "r"(rows[4 * g + 1]), "r"(rows[4 * g + 2]), "r"(rows[4 * g + 3]),
            "r"(b)
            : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"(b) : "memory");
  }
  __syncthreads();
  // un-swizzle: slot r, 16-B chunk c of half h at h * 1024 + r * 128 + ((c ^ (r & 7)) << 4)
  for (int e = threadIdx.x; e < 8 * 16; e += blockDim.x) {
    const int r = e / 16, c = e % 16, h = c / 8, cc = c % 8;
    const uint4 v = *reinterpret_cast<const uint4 *>(s + h * 1024 + r * 128 + ((cc ^ (r & 7)) << 4));
    *reinterpret_cast<uint4 *>(out + r * 128 + c * 8) = v;
  }
}
int main() {
  const int N = 5000, D = 128;
  std::vector<uint16_t> h(static_cast<size_t>(N) * D);
  for (size_t i = 0; i < h.size(); ++i) h[i] = static_cast<uint16_t>(i * 2654435761u >> 16);
  uint16_t *dm, *dout;
  int *drows;
  cudaMalloc(&dm, h.size() * 2);
  cudaMalloc(&dout, 8 * D * 2);
  cudaMalloc(&drows, 8 * 4);
  cudaMemcpy(dm, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  const int rows[8] = {7, 4999, 123, 0, 2048, 31, 4000, 1};
  cudaMemcpy(drows, rows, sizeof(rows), cudaMemcpyHostToDevice);
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(N)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(D) * 2};
  cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dm, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", static_cast<int>(r));
  k<<<1, 128>>>(m, drows, dout);
  printf("launch %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<uint16_t> o(8 * D);
  cudaMemcpy(o.data(), dout, o.size() * 2, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int s = 0; s < 8; ++s)
    for (int c = 0; c < D; ++c) bad += o[s * D + c] != h[static_cast<size_t>(rows[s]) * D + c];
  printf("gather4 mismatches: %d of %d\n", bad, 8 * D);
  return 0;
}
