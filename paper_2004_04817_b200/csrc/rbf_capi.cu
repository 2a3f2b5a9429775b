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

// ------------------------------------------------------------- diagnostics
// FP64 pipe probe: 8 independent DFMA chains per thread, a grid of 4 CTAs of
// 256 threads per SM. Used by bench.py to measure the FP64 peak that the
// roofline fractions are quoted against (the driver's MEASURED_PEAKS.json
// has no FP64 entry).
namespace rbf {
__global__ void __launch_bounds__(256) fp64_probe_kernel(double* out, int iters) {
  const double a = 0.999999999999, b = 1e-12;
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
  if (s == 12345.678) out[blockIdx.x * blockDim.x + threadIdx.x] = s;  // keep the chains live
}
}  // namespace rbf

extern "C" size_t rbf_fp64_probe_scratch_bytes(int device) {
  return (size_t)rbf::sm_count(device) * 4 * 256 * sizeof(double);
}

extern "C" int rbf_fp64_probe(int iters, double* scratch, double* flops_host, void* stream) {
  int dev = 0;
  RBF_CUDA_TRY(cudaGetDevice(&dev));
  const int sms = rbf::sm_count(dev);
  if (sms <= 0 || iters <= 0 || !scratch) return rbf::set_error(RBF_EARG, "bad probe arguments");
  const int blocks = sms * 4;
  rbf::fp64_probe_kernel<<<blocks, 256, 0, rbf::as_stream(stream)>>>(scratch, iters);
  RBF_LAUNCH_CHECK("fp64_probe_kernel");
  if (flops_host) *flops_host = 2.0 * 8.0 * 4.0 * (double)iters * (double)blocks * 256.0;
  return RBF_OK;
}
