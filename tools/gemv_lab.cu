// Packed-triangle GEMV lab: y = A x over a row-packed lower triangle of
// order n (the selection loop's c0 / r / c1 passes), one pass per launch on
// 148 CTAs x 512 threads, timed with CUDA events. Variants:
//   rowwarp : one warp per row, rows strided over all warps (8 loads in flight per lane)
//   seg     : 256-entry segments, whole rows per CTA balanced by segment count,
//             two segments per warp iteration (the current L2-path kernel code)
//   flat    : every CTA takes an equal slice of the packed array; lanes map
//             flat indices to rows; per-row partials combined via atomics-free
//             two-level scheme (per-CTA smem, rows straddling CTAs via a second tiny pass)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2004_04817_b200/csrc \
//        -o tools/gemv_lab tools/gemv_lab.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "rbf_common.cuh"

using namespace rbf;
constexpr int kThreads = 512, kWarps = 16;
constexpr int kSegLen = 256, kSegMax = 2048;

__host__ __device__ inline int64_t tri(int64_t i) { return i * (i + 1) / 2; }
__device__ __forceinline__ int64_t seg_cs(int64_t m) {
  const int64_t q = m / kSegLen, r = m % kSegLen;
  return kSegLen * q * (q + 1) / 2 + r * (q + 1);
}
__device__ __forceinline__ int64_t seg_inv(int64_t S) {
  int64_t q = (int64_t)((sqrt(1.0 + (double)S / 32.0) - 1.0) * 0.5);
  while (128 * (q + 1) * (q + 2) <= S) ++q;
  while (q > 0 && 128 * q * (q + 1) > S) --q;
  return kSegLen * q + (S - 128 * q * (q + 1)) / (q + 1);
}

template <int kBatch>
__global__ void __launch_bounds__(kThreads, 1) rowwarp(const double* A, const double* x, double* y, int n) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kWarps + (threadIdx.x >> 5), nw = gridDim.x * kWarps;
  for (int i = gw; i < n; i += nw) {
    const double* a = A + tri(i);
    double acc = 0.0;
    for (int j0 = 0; j0 <= i; j0 += kBatch * 32) {
      double av[kBatch], xv[kBatch];
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int j = j0 + u * 32 + lane;
        av[u] = j <= i ? __ldcg(a + j) : 0.0;
        xv[u] = j <= i ? __ldcg(x + j) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kBatch; ++u) acc = fma(av[u], xv[u], acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) y[i] = acc;
  }
}

// rows balanced over the grid by entries, one warp per row inside the CTA
__global__ void __launch_bounds__(kThreads, 1) rowbal(const double* A, const double* x, double* y, int n) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t tot = tri(n);
  auto first_at = [&](int64_t t) {  // min i with tri(i) >= t
    int64_t i = (int64_t)ceil((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while (i > 0 && tri(i - 1) >= t) --i;
    while (tri(i) < t) ++i;
    return (int)(i < n ? i : (int64_t)n);
  };
  const int r0 = first_at(tot * blockIdx.x / gridDim.x), r1 = first_at(tot * (blockIdx.x + 1) / gridDim.x);
  for (int i = r0 + warp; i < r1; i += kWarps) {
    const double* a = A + tri(i);
    double acc = 0.0;
    for (int j0 = 0; j0 <= i; j0 += 8 * 32) {
      double av[8], xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + u * 32 + lane;
        av[u] = j <= i ? __ldcg(a + j) : 0.0;
        xv[u] = j <= i ? __ldcg(x + j) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = fma(av[u], xv[u], acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) y[i] = acc;
  }
}

__global__ void __launch_bounds__(kThreads, 1) seg(const double* A, const double* x, double* y, int n) {
  __shared__ double psum[kSegMax];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, b = blockIdx.x;
  const int64_t csn = seg_cs(n);
  auto cum = [&](int64_t v) { return seg_cs(v); };
  auto first_at = [&](int64_t t) -> int {
    if (t <= 0) return 0;
    if (t >= csn) return n;
    return (int)(seg_inv(t - 1) + 1);
  };
  const int v0 = first_at(csn * b / G), v1 = first_at(csn * (b + 1) / G);
  for (int pv0 = v0; pv0 < v1;) {
    const int64_t base = cum(pv0);
    const int pv1 = min(v1, max(pv0 + 1, first_at(base + kSegMax + 1) - 1));
    const int nseg = (int)(cum(pv1) - base);
    for (int s0 = warp; s0 < nseg; s0 += 2 * kWarps) {
      double av[16], xv[16];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int sg = s0 + h * kWarps;
        int v = -1, e0 = 0, len = 0;
        if (sg < nseg) {
          v = (int)seg_inv(base + sg);
          e0 = (int)(base + sg - cum(v)) * kSegLen;
          len = v + 1;
        }
        const double* ab = v >= 0 ? A + tri(v) : A;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * 32 + lane;
          const bool ok = v >= 0 && e < len;
          av[8 * h + u] = ok ? __ldcg(ab + e) : 0.0;
          xv[8 * h + u] = ok ? __ldcg(x + e) : 0.0;
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double acc = 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = fma(av[8 * h + u], xv[8 * h + u], acc);
        acc = warp_sum(acc);
        const int sg = s0 + h * kWarps;
        if (lane == 0 && sg < nseg) psum[sg] = acc;
      }
    }
    __syncthreads();
    for (int v = pv0 + tid; v < pv1; v += kThreads) {
      const int sb = (int)(cum(v) - base), se = (int)(cum(v + 1) - base);
      double acc = 0.0;
      for (int q = sb; q < se; ++q) acc += psum[q];
      y[v] = acc;
    }
    __syncthreads();
    pv0 = pv1;
  }
}

// x staged in shared memory (as the selection kernel does for long rows),
// kB loads of A per lane in flight, optional 16-byte loads
template <int kB, bool kVec>
__global__ void __launch_bounds__(kThreads, 1) rowwarp_sx(const double* A, const double* x, double* y, int n) {
  extern __shared__ double xs[];
  for (int j = threadIdx.x; j < n; j += kThreads) xs[j] = __ldcg(x + j);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kWarps + (threadIdx.x >> 5), nw = gridDim.x * kWarps;
  for (int i = gw; i < n; i += nw) {
    const double* a = A + tri(i);
    const int len = i + 1;
    double acc = 0.0;
    if (!kVec) {
      for (int j0 = 0; j0 < len; j0 += kB * 32) {
        double av[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int j = j0 + u * 32 + lane;
          av[u] = j < len ? __ldcg(a + j) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int j = j0 + u * 32 + lane;
          acc = fma(av[u], j < len ? xs[j] : 0.0, acc);
        }
      }
    } else {
      // peel to a 16-byte boundary, then double2 per lane
      const int head = (int)((reinterpret_cast<uintptr_t>(a) >> 3) & 1);  // 1 if a is 8 mod 16
      if (head && lane == 0) acc = fma(__ldcg(a), xs[0], acc);
      const double2* a2 = reinterpret_cast<const double2*>(a + head);
      const int len2 = (len - head) >> 1;
      for (int j0 = 0; j0 < len2; j0 += kB * 32) {
        double2 av[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int j = j0 + u * 32 + lane;
          av[u] = j < len2 ? __ldcg(a2 + j) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int j = j0 + u * 32 + lane;
          if (j < len2) {
            acc = fma(av[u].x, xs[head + 2 * j], acc);
            acc = fma(av[u].y, xs[head + 2 * j + 1], acc);
          }
        }
      }
      const int tail = head + 2 * len2;
      if (tail < len && lane == 0) acc = fma(__ldcg(a + tail), xs[tail], acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) y[i] = acc;
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int n : {854, 2200, 4379, 6400}) {
    const int64_t T = tri(n);
    std::vector<double> hA(T), hx(n);
    for (int64_t f = 0; f < T; ++f) hA[f] = 1.0 / (1 + (f % 97));
    for (int j = 0; j < n; ++j) hx[j] = 0.5 + (j % 13) * 0.01;
    double *A, *x, *y;
    cudaMalloc(&A, 8 * T);
    cudaMalloc(&x, 8 * n);
    cudaMalloc(&y, 8 * n);
    cudaMemcpy(A, hA.data(), 8 * T, cudaMemcpyHostToDevice);
    cudaMemcpy(x, hx.data(), 8 * n, cudaMemcpyHostToDevice);
    // a buffer to evict A from L2 between passes (cold) or not (warm)
    char* flush;
    cudaMalloc(&flush, 256 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto time = [&](const char* name, auto launch, bool cold) {
      float tot = 0;
      for (int r = 0; r < 12; ++r) {
        if (cold) cudaMemsetAsync(flush, r, 256 << 20);
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r >= 2) tot += ms;
      }
      tot /= 10;
      printf("n %5d %-12s %s %8.2f us  %7.1f GB/s\n", n, name, cold ? "cold" : "warm", tot * 1e3,
             8.0 * T / (tot * 1e-3) * 1e-9);
    };
    for (bool cold : {false, true}) {
      time("rowwarp8", [&] { rowwarp<8><<<sms, kThreads>>>(A, x, y, n); }, cold);
      time("rowwarp16", [&] { rowwarp<16><<<sms, kThreads>>>(A, x, y, n); }, cold);
      time("rowbal", [&] { rowbal<<<sms, kThreads>>>(A, x, y, n); }, cold);
      time("seg", [&] { seg<<<sms, kThreads>>>(A, x, y, n); }, cold);
      const size_t sm = 8 * (size_t)n;
      cudaFuncSetAttribute(rowwarp_sx<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
      cudaFuncSetAttribute(rowwarp_sx<32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
      cudaFuncSetAttribute(rowwarp_sx<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
      cudaFuncSetAttribute(rowwarp_sx<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
      time("sx16", [&] { rowwarp_sx<16, false><<<sms, kThreads, sm>>>(A, x, y, n); }, cold);
      time("sx32", [&] { rowwarp_sx<32, false><<<sms, kThreads, sm>>>(A, x, y, n); }, cold);
      time("sx_v8", [&] { rowwarp_sx<8, true><<<sms, kThreads, sm>>>(A, x, y, n); }, cold);
      time("sx_v16", [&] { rowwarp_sx<16, true><<<sms, kThreads, sm>>>(A, x, y, n); }, cold);
    }
    cudaFree(A); cudaFree(x); cudaFree(y); cudaFree(flush);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
