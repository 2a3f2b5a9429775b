// Does the FP64 tensor-core path (mma.sync m8n8k4 f64, "DMMA") run beside the
// FP64 vector pipe (DFMA) on sm_100a, or share it?  Four kernels, same grid:
//   dfma  : 8 independent DFMA chains per thread
//   dmma  : 4 independent m8n8k4 accumulators per warp
//   mixed : both streams in every warp (same instruction counts as above)
//   split : even warps DFMA, odd warps DMMA
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_bench tools/dmma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <bool kF, bool kM, bool kSplit>
__global__ void bench(double* out, double s) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = s * (threadIdx.x + i);
  double c[4][2] = {};
  double a = s * threadIdx.x, b = s + threadIdx.x;
  const bool odd = (threadIdx.x >> 5) & 1;
  const bool doF = kF && (!kSplit || !odd);
  const bool doM = kM && (!kSplit || odd);
  for (int it = 0; it < ITERS; ++it) {
    if (doF) {
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], 0.999999, 1e-7);
    }
    if (doM) {
#pragma unroll
      for (int i = 0; i < 4; ++i) dmma(c[i], a, b);
    }
  }
  double acc = 0;
  for (int i = 0; i < 8; ++i) acc += x[i];
  for (int i = 0; i < 4; ++i) acc += c[i][0] + c[i][1];
  if (acc == 12345.678) out[0] = acc;
}

template <bool kF, bool kM, bool kSplit>
static void run(const char* name, int blocks, int threads) {
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  bench<kF, kM, kSplit><<<blocks, threads>>>(out, 1e-3);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) bench<kF, kM, kSplit><<<blocks, threads>>>(out, 1e-3);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 5;
  double warps = (double)blocks * threads / 32;
  double wf = kSplit ? warps / 2 : warps;
  double fl_f = kF ? wf * 32 * ITERS * 16 * 2 : 0;        // DFMA flops
  double fl_m = kM ? wf * ITERS * 4 * 256 * 2 : 0;        // DMMA flops (8x8x4 fma)
  printf("%-6s blocks %4d thr %4d  %8.3f ms  dfma %7.2f TF  dmma %7.2f TF  total %7.2f TF\n", name, blocks,
         threads, ms, fl_f / ms * 1e-9, fl_m / ms * 1e-9, (fl_f + fl_m) / ms * 1e-9);
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int t : {256, 512}) {
    run<true, false, false>("dfma", sms * 4, t);
    run<false, true, false>("dmma", sms * 4, t);
    run<true, true, false>("mixed", sms * 4, t);
    run<true, true, true>("split", sms * 4, t);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
