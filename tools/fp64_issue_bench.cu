// FP64 pipe issue limits on sm_100a: DFMA with immediate vs register operands,
// and with one MUFU.RSQ64H per 17 FP64 instructions.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_issue_bench tools/fp64_issue_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 16384

template <int KIND>
__global__ void k(double* out, double s) {
  double x[8], y[8], z[8];
  for (int i = 0; i < 8; ++i) { x[i] = s * (threadIdx.x + i); y[i] = 0.999 + 1e-6 * i * s; z[i] = 1e-7 * (i + 1) * s; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) x[i] = fma(x[i], 0.999999, 1e-7);          // 1 register source
      if (KIND == 1) x[i] = fma(x[i], y[i], z[i]);               // 3 register sources
      if (KIND == 2) x[i] = fma(x[i], y[(i + 1) & 7], z[(i + 3) & 7]);
      if (KIND == 3) x[i] = x[i] * y[i];                         // DMUL reg-reg
      if (KIND == 5) asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(x[i]));
      if (KIND == 6) {                                           // 16 DFMA : 1 RSQ64H, independent
        x[i] = fma(x[i], y[i], z[i]);
        x[i] = fma(x[i], y[i], z[i]);
        if (i == 0) asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(z[7]));
      }
      if (KIND == 7) {                                           // 16 DFMA : 2 RSQ64H
        x[i] = fma(x[i], y[i], z[i]);
        x[i] = fma(x[i], y[i], z[i]);
        if (i == 0) asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(z[7]));
        if (i == 4) asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(z[6]));
      }
      if (KIND == 4) {                                           // 2 DFMA + 1/8.5 MUFU.RSQ64H
        double r;
        x[i] = fma(x[i], y[i], z[i]);
        if ((i & 3) == 0) { asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x[i])); z[i] = r * 1e-30; }
      }
    }
  }
  double acc = 0;
  for (int i = 0; i < 8; ++i) acc += x[i] + z[i];
  if (acc == 12345.678) out[0] = acc;
}

template <int KIND>
void run(const char* name, int sms) {
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = sms * 4, threads = 256;
  k<KIND><<<blocks, threads>>>(out, 1e-3);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<KIND><<<blocks, threads>>>(out, 1e-3);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
  double insts = (double)blocks * threads * ITERS * 8;   // FP64 lane-ops
  double peak_insts_per_s = 16.0 * 4 * sms * 1.965e9;    // 16 lanes/clk/SMSP at max clock
  printf("%-22s %8.3f ms  %7.3f T lane-ops/s  %5.1f %% of 16/clk/SMSP@1965MHz\n", name, ms,
         insts / ms * 1e-9, 100.0 * insts / (ms * 1e-3) / peak_insts_per_s);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("dfma imm", sms); run<1>("dfma 3reg", sms); run<2>("dfma 3reg mixed", sms);
  run<3>("dmul 2reg", sms); run<4>("dfma 3reg + rsq64h/4", sms);
  run<5>("rsq64h only (lane-ops)", sms); run<6>("16 dfma : 1 rsq (x2 ops)", sms); run<7>("16 dfma : 2 rsq (x2)", sms);
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
