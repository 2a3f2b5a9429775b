// Accuracy of MUFU.RSQ64H (rsqrt.approx.ftz.f64) and of cheap eta = sqrt(r2)
// refinements, over r2 in [1e-8, 8] (log-uniform). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rsqrt_precision rsqrt_precision.cu
#include <cstdio>
#include <cmath>
__device__ double rsq(double x) { double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y; }
__global__ void k(int n, double* err) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = exp(log(1e-8) + (log(8.0) - log(1e-8)) * (i + 0.5) / n);
  double s = sqrt(x);
  double y0 = rsq(x);
  double e0 = fabs(y0 * s - 1.0);                     // rsqrt approx rel. error
  double eta0 = x * y0;                                // one Newton step on eta
  double h = fma(-eta0, eta0, x);
  double eta1 = fma(h, 0.5 * y0, eta0);
  double e1 = fabs(eta1 - s) / s;
  double e = fma(-x, y0 * y0, 1.0);                    // current: cubic on y then t
  double p = fma(e, 0.375, 0.5);
  double y = fma(p, y0 * e, y0);
  double e2 = fabs(x * y - s) / s;
  err[3 * i] = e0; err[3 * i + 1] = e1; err[3 * i + 2] = e2;
}
int main() {
  const int n = 1 << 22;
  double* d; cudaMalloc(&d, 3 * n * sizeof(double));
  k<<<(n + 255) / 256, 256>>>(n, d);
  double* h = new double[3 * n];
  cudaMemcpy(h, d, 3 * n * sizeof(double), cudaMemcpyDeviceToHost);
  double m[3] = {0, 0, 0};
  for (int i = 0; i < n; ++i) for (int c = 0; c < 3; ++c) m[c] = fmax(m[c], h[3 * i + c]);
  printf("max rel err: rsqrt.approx %.3e (2^%.1f)  eta one-Newton %.3e (2^%.1f)  current %.3e (2^%.1f)\n",
         m[0], log2(m[0]), m[1], log2(m[1]), m[2], log2(m[2]));
  return 0;
}
