// C-ABI plumbing: thread-local error string, status mapping, device info.
#include <cstdarg>
#include <cstring>

#include "ls_common.cuh"

namespace ls {

static thread_local char g_err[1024] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char *where) {
  set_error("CUDA error %s (%d) at %s", cudaGetErrorString(e), static_cast<int>(e), where);
  return LS_ERR_CUDA;
}

}  // namespace ls

namespace ls {
// device-side validation status (first error wins): kernels that find a
// reference error condition on the device (NonFiniteInput / AllMaskedRow in
// the sampled-row softmax, EmptyPlan in the sparse attention) record its
// ls_status code here; ls_device_status() reads and clears it.
static int32_t *g_status = nullptr;
int32_t *device_status_ptr() {
  if (!g_status) {
    if (cudaMalloc(&g_status, sizeof(int32_t)) != cudaSuccess) return nullptr;
    cudaMemset(g_status, 0, sizeof(int32_t));
  }
  return g_status;
}
}  // namespace ls

extern "C" int ls_device_status(int32_t *host_status, ls_stream_t stream) {
  int32_t *d = ls::device_status_ptr();
  LS_REQUIRE(d != nullptr, LS_ERR_CUDA, "device status word unavailable");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  LS_CUDA(cudaMemcpyAsync(host_status, d, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  LS_CUDA(cudaStreamSynchronize(st));
  LS_CUDA(cudaMemsetAsync(d, 0, sizeof(int32_t), st));
  return LS_OK;
}

extern "C" const char *ls_last_error(void) { return ls::g_err; }

extern "C" int ls_version(void) { return 1; }

extern "C" int ls_device_info(int *sm_count, char *name, int name_len) {
  int dev = 0;
  LS_CUDA(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  LS_CUDA(cudaGetDeviceProperties(&prop, dev));
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (name && name_len > 0) {
    strncpy(name, prop.name, name_len - 1);
    name[name_len - 1] = '\0';
  }
  return LS_OK;
}
