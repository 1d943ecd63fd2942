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
