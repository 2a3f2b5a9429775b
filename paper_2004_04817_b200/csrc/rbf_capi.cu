// C-ABI plumbing: error reporting, version and device queries.
#include <cstring>

#include "rbf_internal.h"

namespace rbf {

static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int sm_count(int device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
  return n;
}

}  // namespace rbf

extern "C" int rbf_abi_version(void) { return RBF_ABI_VERSION; }

extern "C" const char* rbf_last_error(void) { return rbf::g_err; }
