// Error plumbing + version of the C ABI (include/texelfuse_b200.h).
#include <stdarg.h>
#include <string.h>

#include "common.cuh"

namespace tfb {

static thread_local char g_err[1024] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: CUDA error %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
    return TFB_ERR_CUDA;
  }
  return TFB_OK;
}

}  // namespace tfb

extern "C" const char *tfb_last_error(void) { return tfb::g_err; }

extern "C" int tfb_version(void) { return 1; }
