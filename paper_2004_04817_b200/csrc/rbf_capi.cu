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

// --------------------------------------------------------- group partition
// numpy's Generator(PCG64).permutation(nb) dealt round-robin into m groups
// (reference selection.py:183-184: perm = default_rng(seed).permutation(nb),
// groups[j] = perm[j::m]), restated bit for bit on the host: PCG64 is the
// 128-bit LCG with XSL-RR output, numpy draws 32-bit values from the low
// then the high half of each 64-bit output, shuffle() is Fisher-Yates from
// the top with random_interval()'s masked rejection sampling. The caller
// passes the seeded 128-bit state and increment (bit_generator.state).
namespace {
struct Pcg64 {
  unsigned __int128 state, inc;
  bool has32 = false;
  uint32_t hi32 = 0;
  uint64_t next64() {
    const unsigned __int128 mult =
        ((unsigned __int128)0x2360ED051FC65DA4ull << 64) | (unsigned __int128)0x4385DF649FCCF645ull;
    state = state * mult + inc;
    const uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
    const unsigned rot = (unsigned)(state >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  uint32_t next32() {
    if (has32) {
      has32 = false;
      return hi32;
    }
    const uint64_t v = next64();
    has32 = true;
    hi32 = (uint32_t)(v >> 32);
    return (uint32_t)(v & 0xffffffffu);
  }
  uint64_t interval(uint64_t max) {
    if (max == 0) return 0;
    uint64_t mask = max;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    mask |= mask >> 32;
    uint64_t v;
    if (max <= 0xffffffffull) {
      while ((v = (next32() & mask)) > max) {
      }
    } else {
      while ((v = (next64() & mask)) > max) {
      }
    }
    return v;
  }
};
}  // namespace

extern "C" int rbf_partition(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                             int64_t nb, int64_t m, int32_t* group_pos_host, int32_t* group_off_host) {
  if (nb < 1 || m < 1 || m > nb || nb > INT32_MAX || !group_pos_host || !group_off_host)
    return rbf::set_error(RBF_EARG, "bad partition arguments");
  Pcg64 g;
  g.state = ((unsigned __int128)state_hi << 64) | state_lo;
  g.inc = ((unsigned __int128)inc_hi << 64) | inc_lo;
  int32_t* perm = new int32_t[nb];
  for (int64_t i = 0; i < nb; ++i) perm[i] = (int32_t)i;
  // Fisher-Yates from the top. The masked rejection loop of
  // random_interval() is walked draw by draw without a data-dependent branch:
  // a rejected draw swaps perm[i] with itself and leaves i where it is (the
  // accept/reject branch mispredicts on ~1 draw in 4 otherwise).
  // (nb <= INT32_MAX: every bound takes the 32-bit draws.)
  for (int64_t i = nb - 1; i >= 1;) {
    const uint64_t mask = ~0ull >> __builtin_clzll((uint64_t)i);
    const uint64_t v = g.next32() & mask;
    const bool take = v <= (uint64_t)i;
    const int64_t j = take ? (int64_t)v : i;
    const int32_t t = perm[j];
    perm[j] = perm[i];
    perm[i] = t;
    i -= take;
  }
  // group j = perm[j::m]: sizes are known, so one sequential pass over perm
  // deals it into the m groups (a strided read per group misses the cache
  // on every element once nb * 4 B outgrows L1)
  int64_t o = 0;
  for (int64_t j = 0; j < m; ++j) {
    group_off_host[j] = (int32_t)o;
    o += nb / m + (j < nb % m ? 1 : 0);
  }
  group_off_host[m] = (int32_t)o;
  for (int64_t base = 0, q = 0; base < nb; base += m, ++q) {
    const int64_t cnt = nb - base < m ? nb - base : m;
    for (int64_t j = 0; j < cnt; ++j) group_pos_host[group_off_host[j] + q] = perm[base + j];
  }
  delete[] perm;
  return RBF_OK;
}
