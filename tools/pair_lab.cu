// Pair-body lab: FP64-pipe instruction count vs accuracy of the Wendland-C2
// pair (volume evaluation / error scans). Forms:
//   0  library difference form: third-order rsqrt correction      (19 FP64 / pair)
//   2  difference form, one Newton step on eta = sqrt(r2) with
//      y0/2 formed by an integer exponent decrement               (17 FP64 / pair)
//   3  expanded r2 = (P + S) + p.(-2s) with the Newton step on eta  (15 FP64 / pair)
// Prints (1) the MUFU.RSQ64H relative error and the eta error of each form
// over r2 in [1e-10, 1.2]; (2) max |phi_form - phi_exact| where phi_exact is
// the reference's separately-rounded chain on a correctly rounded cdist;
// (3) throughput on 2M random targets for several launch geometries, with the
// max relative deviation of the displacement from the exact-chain kernel.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo \
//        -I paper_2004_04817_b200/csrc -o tools/pair_lab tools/pair_lab.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

#include "rbf_common.cuh"

using namespace rbf;

__device__ __forceinline__ double half_exp(double y) {  // y / 2 on the integer pipe
  return __hiloint2double(__double2hiint(y) - 0x00100000, __double2loint(y));
}

__device__ __forceinline__ double lift_tiny(double r2) {
  const int kTinyHi = 0x16687e92;  // high word of 1e-200
  return __hiloint2double(max(__double2hiint(r2), kTinyHi), __double2loint(r2));
}

// t = 1 - eta from r2 (eta^2) by one Newton step on eta
__device__ __forceinline__ double t_newton(double r2) {
  const double y0 = rsqrt_approx(r2);
  const double e0 = r2 * y0;                 // eta_0
  const double h = fma(-e0, e0, r2);         // r2 - eta_0^2
  const double c = 1.0 - e0;
  return fma(-h, half_exp(y0), c);           // 1 - (eta_0 + h y0 / 2)
}

// t = 1 - eta, third order in e = 1 - r2 y0^2 with 5 FP64 instructions:
//   eta = eta0 (1 + e (1/2 + 3e/8)),  eta0 = r2 y0
__device__ __forceinline__ double t_cubic5(double r2) {
  const double y0 = rsqrt_approx(r2);
  const double e0 = r2 * y0;
  const double e = fma(-e0, y0, 1.0);
  const double p = fma(e, 0.375, 0.5);
  const double w = fma(e, p, 1.0);
  return fma(-e0, w, 1.0);
}

__device__ __forceinline__ double fma_asm(double a, double b, double c) {
  double d;
  asm("fma.rn.f64 %0, %1, %2, %3;" : "=d"(d) : "d"(a), "d"(b), "d"(c));
  return d;
}

template <int FORM>
__device__ __forceinline__ void pair(double px, double py, double pz, double P, double4 a, double4 b,
                                     double& ax, double& ay, double& az) {
  if (FORM == 0) {
    pair_accum(px, py, pz, a.x, a.y, a.z, a.w, b.x, b.y, ax, ay, az);
    return;
  }
  if (FORM == 6) {  // form 4 with the DMULs issued as DFMA(a, b, -0)
    const double dx = px - a.x, dy = py - a.y, dz = pz - a.z;
    double r2 = fma(dz, dz, fma(dy, dy, fma_asm(dx, dx, -0.0)));
    r2 = lift_tiny(r2);
    const double y0 = rsqrt_approx(r2);
    const double e0 = fma_asm(r2, y0, -0.0);
    const double e = fma(-e0, y0, 1.0);
    const double p = fma(e, 0.375, 0.5);
    const double w = fma(e, p, 1.0);
    double t = clamp_nonneg(fma(-e0, w, 1.0));
    const double q = fma(-4.0, t, 5.0);
    t = fma_asm(t, t, -0.0);
    const double f = fma_asm(fma_asm(t, t, -0.0), q, -0.0);
    ax = fma(a.w, f, ax);
    ay = fma(b.x, f, ay);
    az = fma(b.y, f, az);
    return;
  }
  double r2;
  double wx, wy, wz;
  if (FORM == 2 || FORM == 4) {
    const double dx = px - a.x, dy = py - a.y, dz = pz - a.z;
    r2 = fma(dz, dz, fma(dy, dy, dx * dx));
    wx = a.w; wy = b.x; wz = b.y;
  } else {
    r2 = fma(pz, a.z, fma(py, a.y, fma(px, a.x, P + a.w)));
    wx = b.x; wy = b.y; wz = b.z;
  }
  r2 = lift_tiny(r2);
  double t = clamp_nonneg(FORM >= 4 ? t_cubic5(r2) : t_newton(r2));
  const double q = fma(-4.0, t, 5.0);
  t = t * t;
  const double f = (t * t) * q;
  ax = fma(wx, f, ax);
  ay = fma(wy, f, ay);
  az = fma(wz, f, az);
}

// ------------------------------------------------------------ precision
__global__ void precision_kernel(int n, double* err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double lo = log(1e-10), hi = log(1.2);
  // half the samples log-uniform, half uniform in [0, 1.2]
  const double x = (i & 1) ? exp(lo + (hi - lo) * (i + 0.5) / n) : 1.2 * (i + 0.5) / n;
  const double s = __dsqrt_rn(x);
  const double y0 = rsqrt_approx(x);
  err[4 * i] = fabs(y0 * s - 1.0);
  // current form's eta
  const double e = fma(-x, y0 * y0, 1.0);
  const double y = fma(fma(e, 0.375, 0.5), y0 * e, y0);
  err[4 * i + 1] = fabs(fma(-x, y, 1.0) - (1.0 - s));  // abs error of t (vs t from exact eta)
  err[4 * i + 2] = fabs(t_cubic5(x) - (1.0 - s));
  // phi error (Newton form) vs reference chain
  double t = fmax(__dsub_rn(1.0, s), 0.0);
  t = __dmul_rn(t, t);
  const double phi_ref = __dmul_rn(__dmul_rn(t, t), __dadd_rn(__dmul_rn(4.0, s), 1.0));
  double tn = clamp_nonneg(t_newton(x));
  const double q = fma(-4.0, tn, 5.0);
  tn = tn * tn;
  err[4 * i + 3] = fabs((tn * tn) * q - phi_ref);
}

// --------------------------------------------------------------- kernels
// exact: reference chain per pair (cdist_exact / phi_exact), the yardstick
__global__ void exact_kernel(const double* __restrict__ t, int64_t nt, const double* __restrict__ s,
                             const double* __restrict__ w, int ns, double radius, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nt) return;
  double ax = 0, ay = 0, az = 0;
  for (int j = 0; j < ns; ++j) {
    const double f = phi_exact(cdist_exact(t[3 * i], t[3 * i + 1], t[3 * i + 2], s[3 * j], s[3 * j + 1],
                                           s[3 * j + 2]), radius);
    ax = fma(w[3 * j], f, ax);
    ay = fma(w[3 * j + 1], f, ay);
    az = fma(w[3 * j + 2], f, az);
  }
  out[3 * i] = ax; out[3 * i + 1] = ay; out[3 * i + 2] = az;
}

template <int FORM, int NT, int TPT, int MINB>
__global__ void __launch_bounds__(NT, MINB)
lab_kernel(const double* __restrict__ tpts, int64_t nt, const double* __restrict__ spts,
           const double* __restrict__ sw, int nsup, double inv_r, double* __restrict__ out) {
  constexpr int TILE = 128;
  constexpr bool EXPANDED = FORM == 3 || FORM == 5;
  __shared__ double4 s_a[TILE];
  __shared__ double4 s_b[TILE];
  const double ox = EXPANDED ? spts[0] : 0.0, oy = EXPANDED ? spts[1] : 0.0,
               oz = EXPANDED ? spts[2] : 0.0;
  const int64_t base = (int64_t)blockIdx.x * NT * TPT + threadIdx.x;
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
  for (int t0 = 0; t0 < nsup; t0 += TILE) {
    const int cnt = min(TILE, nsup - t0);
    __syncthreads();
    for (int j = threadIdx.x; j < cnt; j += NT) {
      const int g = t0 + j;
      const double x = (spts[3 * g] - ox) * inv_r, y = (spts[3 * g + 1] - oy) * inv_r,
                   z = (spts[3 * g + 2] - oz) * inv_r;
      if (!EXPANDED) {
        s_a[j] = make_double4(x, y, z, sw[3 * g]);
        s_b[j] = make_double4(sw[3 * g + 1], sw[3 * g + 2], 0.0, 0.0);
      } else {
        s_a[j] = make_double4(-2.0 * x, -2.0 * y, -2.0 * z, fma(z, z, fma(y, y, x * x)));
        s_b[j] = make_double4(sw[3 * g], sw[3 * g + 1], sw[3 * g + 2], 0.0);
      }
    }
    __syncthreads();
#pragma unroll 2
    for (int j = 0; j < cnt; ++j) {
      const double4 a = s_a[j];
      const double4 b = s_b[j];
#pragma unroll
      for (int k = 0; k < TPT; ++k) pair<FORM>(px[k], py[k], pz[k], pp[k], a, b, ax[k], ay[k], az[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const int64_t r = base + (int64_t)k * NT;
    if (r >= nt) continue;
    out[3 * r] = ax[k];
    out[3 * r + 1] = ay[k];
    out[3 * r + 2] = az[k];
  }
}

struct Data {
  int64_t nt;
  int ns;
  double *t, *s, *w, *out, *ref;
  double wsum;  // sum |w| (per component max), the conditioning yardstick
};

template <int FORM, int NT, int TPT, int MINB>
static void run(const char* name, Data& d) {
  auto k = lab_kernel<FORM, NT, TPT, MINB>;
  const int64_t grid = (d.nt + NT * TPT - 1) / (NT * TPT);
  const double inv_r = 0.5;
  for (int i = 0; i < 2; ++i) k<<<(unsigned)grid, NT>>>(d.t, d.nt, d.s, d.w, d.ns, inv_r, d.out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 7; ++r) {
    cudaEventRecord(e0);
    k<<<(unsigned)grid, NT>>>(d.t, d.nt, d.s, d.w, d.ns, inv_r, d.out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  cudaError_t err = cudaGetLastError();
  std::vector<double> a(3 * d.nt), b(3 * d.nt);
  cudaMemcpy(a.data(), d.out, 24 * d.nt, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), d.ref, 24 * d.nt, cudaMemcpyDeviceToHost);
  double maxabs = 0, umax = 0;
  for (int64_t i = 0; i < 3 * d.nt; ++i) {
    maxabs = std::max(maxabs, std::fabs(a[i] - b[i]));
    umax = std::max(umax, std::fabs(b[i]));
  }
  const double tf = 22.0 * d.nt * d.ns / (best * 1e-3) / 1e12;
  printf("%-26s ns %5d  %8.4f ms  %6.2f TF  max|du|/max|u| %.2e  max|du|/sum|w| %.2e %s\n", name, d.ns,
         best, tf, maxabs / umax, maxabs / d.wsum, err ? cudaGetErrorString(err) : "");
}

static Data make(int64_t nt, int ns, double wscale, bool alternating) {
  std::mt19937_64 g(42);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  std::vector<double> t(3 * nt), s(3 * ns), w(3 * ns);
  for (auto& x : t) x = 2.0 * u(g);
  for (auto& x : s) x = u(g);
  double ws = 0;
  for (int j = 0; j < ns; ++j)
    for (int c = 0; c < 3; ++c) {
      // alternating large weights mimic an ill-conditioned system's cancellation
      w[3 * j + c] = alternating ? wscale * ((j & 1) ? 1.0 : -1.0) * (1.0 + 0.1 * u(g)) : wscale * u(g);
      if (c == 0) ws += std::fabs(w[3 * j]);
    }
  Data d{nt, ns};
  d.wsum = ws;
  cudaMalloc(&d.t, 24 * nt);
  cudaMalloc(&d.out, 24 * nt);
  cudaMalloc(&d.ref, 24 * nt);
  cudaMalloc(&d.s, 24 * ns);
  cudaMalloc(&d.w, 24 * ns);
  cudaMemcpy(d.t, t.data(), 24 * nt, cudaMemcpyHostToDevice);
  cudaMemcpy(d.s, s.data(), 24 * ns, cudaMemcpyHostToDevice);
  cudaMemcpy(d.w, w.data(), 24 * ns, cudaMemcpyHostToDevice);
  exact_kernel<<<(unsigned)((nt + 255) / 256), 256>>>(d.t, nt, d.s, d.w, ns, 2.0, d.ref);
  return d;
}

static void release(Data& d) {
  cudaFree(d.t); cudaFree(d.out); cudaFree(d.ref); cudaFree(d.s); cudaFree(d.w);
}

int main() {
  {
    const int n = 1 << 22;
    double* d;
    cudaMalloc(&d, 4 * sizeof(double) * n);
    precision_kernel<<<n / 256, 256>>>(n, d);
    std::vector<double> h(4 * (size_t)n);
    cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
    double m[4] = {0, 0, 0, 0};
    for (int i = 0; i < n; ++i)
      for (int c = 0; c < 4; ++c) m[c] = std::max(m[c], h[4 * (size_t)i + c]);
    printf("RSQ64H max rel err %.3e (2^%.1f); |t err| current %.3e, cubic5 %.3e; |phi err| newton %.3e\n",
           m[0], std::log2(m[0]), m[1], m[2], m[3]);
    cudaFree(d);
  }
  for (int ns : {287, 854}) {
    for (int alt = 0; alt < 2; ++alt) {
      Data d = make(2000000, ns, alt ? 1e4 : 0.01, alt);
      printf("-- %s weights\n", alt ? "alternating 1e4" : "random 0.01");
      run<0, 128, 6, 3>("form0 (19) 128x6 b3", d);
      run<4, 128, 6, 3>("form4 (18) 128x6 b3", d);
      run<5, 128, 6, 3>("form5 (16) 128x6 b3", d);
      run<3, 128, 6, 3>("form3 (15) 128x6 b3", d);
      if (!alt) {
        run<6, 128, 6, 3>("form6 (18, fma) 128x6 b3", d);
        run<4, 128, 4, 4>("form4 (18) 128x4 b4", d);
        run<4, 128, 5, 4>("form4 (18) 128x5 b4", d);
        run<4, 128, 8, 2>("form4 (18) 128x8 b2", d);
        run<4, 96, 6, 4>("form4 (18) 96x6 b4", d);
        run<4, 64, 6, 6>("form4 (18) 64x6 b6", d);
        run<5, 128, 4, 4>("form5 (16) 128x4 b4", d);
        run<5, 128, 5, 4>("form5 (16) 128x5 b4", d);
      }
      release(d);
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
