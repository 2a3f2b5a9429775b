// Dependent-chain latency of FP64 DADD / DFMA / DMUL, a shuffle round trip and
// the double-double two-sum on one warp (clock64 over 4096 dependent ops).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_latency tools/fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double seed, double* out, long long* cyc) {
  double a = seed, b = seed * 0.5, c = 1.0000001;
  long long t0, t1;
  const int N = 4096;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) a = __dadd_rn(a, b);
  t1 = clock64();
  cyc[0] = t1 - t0;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) a = __fma_rn(a, c, b);
  t1 = clock64();
  cyc[1] = t1 - t0;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) a = __dmul_rn(a, c);
  t1 = clock64();
  cyc[2] = t1 - t0;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) a = __shfl_xor_sync(0xffffffffu, a, 1) + b;
  t1 = clock64();
  cyc[3] = t1 - t0;
  double s = a, e = 0.0;
  t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) {  // two-sum accumulate (dd)
    const double t = __dadd_rn(s, b);
    const double v = __dsub_rn(t, s);
    e = __dadd_rn(e, __dadd_rn(__dsub_rn(s, __dsub_rn(t, v)), __dsub_rn(b, v)));
    s = t;
  }
  t1 = clock64();
  cyc[4] = t1 - t0;
  float f = (float)seed;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) f = __fadd_rn(f, 0.5f);
  t1 = clock64();
  cyc[5] = t1 - t0;
  out[threadIdx.x] = a + s + e + f;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * sizeof(double));
  cudaMallocManaged(&cyc, 8 * sizeof(long long));
  lat<<<1, 32>>>(1.0, out, cyc);
  lat<<<1, 32>>>(1.0, out, cyc);
  cudaDeviceSynchronize();
  const char* names[] = {"DADD", "DFMA", "DMUL", "SHFL+DADD", "two-sum step", "FADD"};
  for (int i = 0; i < 6; ++i) printf("%-14s %.2f cycles/op\n", names[i], cyc[i] / 4096.0);
  return 0;
}
