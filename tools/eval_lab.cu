// Volume-kernel lab: launch geometry x pair form x persistence, timed with
// CUDA events on synthetic configs[1]-like data (targets spread over a box,
// supports inside it), compared against the library's difference-form pair.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo \
//        -I paper_2004_04817_b200/csrc -o tools/eval_lab tools/eval_lab.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <random>
#include <cuda_runtime.h>

#include "rbf_common.cuh"

using namespace rbf;

// ---------------------------------------------------------------- kernels
// FORM 0: difference form (19 FP64/pair); FORM 1: expanded (17 FP64/pair)
// PERSIST: grid-stride over target chunks; supports staged once when they fit
template <int FORM, int NT, int TPT, int MINB, bool PERSIST>
__global__ void __launch_bounds__(NT, MINB)
lab_kernel(const double* __restrict__ tpts, int64_t nt, const double* __restrict__ spts,
           const double* __restrict__ sw, int nsup, int cap, double inv_r, double* __restrict__ out) {
  extern __shared__ double4 smem[];
  double4* s_a = smem;        // FORM 0: x,y,z,wx   FORM 1: -2x,-2y,-2z,S
  double4* s_b = smem + cap;  // FORM 0: wy,wz,-,-  FORM 1: wx,wy,wz,-
  const double ox = FORM ? spts[0] : 0.0, oy = FORM ? spts[1] : 0.0, oz = FORM ? spts[2] : 0.0;
  auto stage = [&](int t0, int cnt) {
    for (int j = threadIdx.x; j < cnt; j += NT) {
      const int g = t0 + j;
      const double x = (spts[3 * g] - ox) * inv_r, y = (spts[3 * g + 1] - oy) * inv_r,
                   z = (spts[3 * g + 2] - oz) * inv_r;
      if (FORM == 0) {
        s_a[j] = make_double4(x, y, z, sw[3 * g]);
        s_b[j] = make_double4(sw[3 * g + 1], sw[3 * g + 2], 0.0, 0.0);
      } else {
        s_a[j] = make_double4(-2.0 * x, -2.0 * y, -2.0 * z, fma(z, z, fma(y, y, x * x)));
        s_b[j] = make_double4(sw[3 * g], sw[3 * g + 1], sw[3 * g + 2], 0.0);
      }
    }
  };
  const bool resident = nsup <= cap;
  if (PERSIST && resident) {
    stage(0, nsup);
    __syncthreads();
  }
  const int64_t per_block = (int64_t)NT * TPT;
  const int64_t nchunks = (nt + per_block - 1) / per_block;
  for (int64_t c = blockIdx.x; c < nchunks; c += (PERSIST ? gridDim.x : nchunks)) {
    const int64_t base = c * per_block + threadIdx.x;
    double px[TPT], py[TPT], pz[TPT], pp[TPT], ax[TPT], ay[TPT], az[TPT];
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
      const int64_t r = base + (int64_t)k * NT;
      double x = 0.0, y = 0.0, z = 0.0;
      if (r < nt) {
        x = (tpts[3 * r] - ox) * inv_r;
        y = (tpts[3 * r + 1] - oy) * inv_r;
        z = (tpts[3 * r + 2] - oz) * inv_r;
      }
      px[k] = x; py[k] = y; pz[k] = z;
      pp[k] = fma(z, z, fma(y, y, x * x));
      ax[k] = ay[k] = az[k] = 0.0;
    }
    for (int t0 = 0; t0 < nsup; t0 += cap) {
      const int cnt = min(cap, nsup - t0);
      if (!(PERSIST && resident)) {
        __syncthreads();
        stage(t0, cnt);
        __syncthreads();
      }
#pragma unroll 2
      for (int j = 0; j < cnt; ++j) {
        const double4 a = s_a[j];
        const double4 b = s_b[j];
#pragma unroll
        for (int k = 0; k < TPT; ++k) {
          if (FORM == 0)
            pair_accum(px[k], py[k], pz[k], a.x, a.y, a.z, a.w, b.x, b.y, ax[k], ay[k], az[k]);
          else
            pair_accum_expanded(px[k], py[k], pz[k], pp[k], a.x, a.y, a.z, a.w, b.x, b.y, b.z, ax[k],
                                ay[k], az[k]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
      const int64_t r = base + (int64_t)k * NT;
      if (r >= nt) continue;
      out[3 * r] = tpts[3 * r] + ax[k];
      out[3 * r + 1] = tpts[3 * r + 1] + ay[k];
      out[3 * r + 2] = tpts[3 * r + 2] + az[k];
    }
  }
}

struct Data {
  int64_t nt;
  int ns;
  double* t;
  double* s;
  double* w;
  double* out;
  double* ref;
};

static int g_sms;

template <int FORM, int NT, int TPT, int MINB, bool PERSIST>
static void run(const char* name, Data& d, int cap_req, bool check) {
  auto k = lab_kernel<FORM, NT, TPT, MINB, PERSIST>;
  const int cap = PERSIST ? cap_req : 128;
  const size_t smem = 2 * sizeof(double4) * cap;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NT, smem);
  const int64_t per_block = (int64_t)NT * TPT;
  const int64_t nchunks = (d.nt + per_block - 1) / per_block;
  const int64_t grid = PERSIST ? std::min<int64_t>(nchunks, (int64_t)g_sms * occ) : nchunks;
  const double inv_r = 0.5;
  for (int i = 0; i < 2; ++i) k<<<(unsigned)grid, NT, smem>>>(d.t, d.nt, d.s, d.w, d.ns, cap, inv_r, d.out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 7; ++r) {
    cudaEventRecord(e0);
    k<<<(unsigned)grid, NT, smem>>>(d.t, d.nt, d.s, d.w, d.ns, cap, inv_r, d.out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  cudaError_t err = cudaGetLastError();
  double maxrel = 0;
  if (check) {
    std::vector<double> a(3 * d.nt), b(3 * d.nt), t(3 * d.nt);
    cudaMemcpy(a.data(), d.out, 24 * d.nt, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), d.ref, 24 * d.nt, cudaMemcpyDeviceToHost);
    cudaMemcpy(t.data(), d.t, 24 * d.nt, cudaMemcpyDeviceToHost);
    for (int64_t i = 0; i < 3 * d.nt; i += 7) {
      const double ua = a[i] - t[i], ub = b[i] - t[i];
      const double den = std::max(std::fabs(ub), 1e-3);
      maxrel = std::max(maxrel, std::fabs(ua - ub) / den);
    }
  }
  const double tf = 22.0 * d.nt * d.ns / (best * 1e-3) / 1e12;
  printf("%-28s nt %8lld ns %5d grid %6lld occ %d  %8.4f ms  %6.2f TF  maxrel %.2e %s\n", name,
         (long long)d.nt, d.ns, (long long)grid, occ, best, tf, maxrel, err ? cudaGetErrorString(err) : "");
}

static Data make(int64_t nt, int ns) {
  std::mt19937_64 g(42);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  std::vector<double> t(3 * nt), s(3 * ns), w(3 * ns);
  for (auto& x : t) x = 2.0 * u(g);
  for (auto& x : s) x = u(g);
  for (auto& x : w) x = 0.01 * u(g);
  Data d{nt, ns};
  cudaMalloc(&d.t, 24 * nt);
  cudaMalloc(&d.out, 24 * nt);
  cudaMalloc(&d.ref, 24 * nt);
  cudaMalloc(&d.s, 24 * ns);
  cudaMalloc(&d.w, 24 * ns);
  cudaMemcpy(d.t, t.data(), 24 * nt, cudaMemcpyHostToDevice);
  cudaMemcpy(d.s, s.data(), 24 * ns, cudaMemcpyHostToDevice);
  cudaMemcpy(d.w, w.data(), 24 * ns, cudaMemcpyHostToDevice);
  return d;
}

int main(int argc, char** argv) {
  cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0);
  for (int ns : {287, 854, 2000}) {
    Data d = make(2000000, ns);
    run<0, 128, 6, 3, false>("diff 128x6 b3 (lib v4)", d, 128, false);
    cudaMemcpy(d.ref, d.out, 24 * d.nt, cudaMemcpyDeviceToDevice);
    run<0, 128, 6, 3, true>("diff 128x6 b3 persist", d, 1024, true);
    run<0, 128, 4, 4, true>("diff 128x4 b4 persist", d, 768, true);
    run<0, 128, 8, 2, true>("diff 128x8 b2 persist", d, 1024, true);
    run<1, 128, 6, 3, false>("exp 128x6 b3", d, 128, true);
    run<1, 128, 6, 3, true>("exp 128x6 b3 persist", d, 1024, true);
    run<1, 128, 4, 4, true>("exp 128x4 b4 persist", d, 768, true);
    run<1, 128, 8, 2, true>("exp 128x8 b2 persist", d, 1024, true);
    run<1, 64, 8, 4, true>("exp 64x8 b4 persist", d, 768, true);
    run<1, 256, 4, 2, true>("exp 256x4 b2 persist", d, 1024, true);
    run<1, 128, 5, 3, true>("exp 128x5 b3 persist", d, 1024, true);
    run<1, 96, 6, 4, true>("exp 96x6 b4 persist", d, 768, true);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
