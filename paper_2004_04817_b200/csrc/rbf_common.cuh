// Shared device helpers for the B200 RBF hot path (sm_100a, FP64 CUDA cores).
//
// Two evaluations of the Wendland C2 kernel live here:
//  * phi_exact(): the reference's per-element chain with every operation
//    rounded separately (no FMA contraction), used for Cholesky rows so the
//    factored matrix is bit-identical to the reference's
//    (reference: core.py:45-50 `_phi`, selection.py:289-295 / 342-347 the
//    row `[phi(cdist/R)..., 1.0]`; cdist is sqrt((dx*dx+dy*dy)+dz*dz)).
//  * pair_accum(): the throughput path for the error scan and volume
//    evaluation (reference: core.py:316-326 `_eval_displacements` inner
//    tile), coordinates pre-scaled by 1/R so eta = |p - s| directly.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rbf {

constexpr int kWarp = 32;

// ---------------------------------------------------------------- numerics
__device__ __forceinline__ double cdist_exact(double ax, double ay, double az,
                                              double bx, double by, double bz) {
  double dx = __dsub_rn(ax, bx), dy = __dsub_rn(ay, by), dz = __dsub_rn(az, bz);
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                              __dmul_rn(dz, dz)));
}

// reference core.py:45-50 with eta = d / R (numpy true division)
__device__ __forceinline__ double phi_exact(double d, double radius) {
  double eta = __ddiv_rn(d, radius);
  double t = fmax(__dsub_rn(1.0, eta), 0.0);
  t = __dmul_rn(t, t);
  t = __dmul_rn(t, t);
  return __dmul_rn(t, __dadd_rn(__dmul_rn(4.0, eta), 1.0));
}

__device__ __forceinline__ double rsqrt_approx(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// max(t, 0) for the Wendland factor in ONE integer instruction: a negative t
// has a negative high word, which max(hi, 0) replaces by 0 while the low word
// stays -- the result is a subnormal (< 2^-1042), whose square underflows to
// exactly +0, so phi = t^4 (5 - 4t) = 0 exactly as with a full clamp. (Every
// non-FP64 instruction costs an issue slot the FP64 pipe then idles for:
// measured 2 x FP64 + 1 x other issue cycles per pair.)
__device__ __forceinline__ double clamp_nonneg(double t) {
  return __hiloint2double(max(__double2hiint(t), 0), __double2loint(t));
}

// t = 1 - eta from r2 = eta^2 in 5 FP64 instructions. y0 = MUFU.RSQ64H(r2)
// has relative error up to 2^-20 (tools/pair_lab.cu, measured on B200), so
// with eta0 = r2 y0 and e = 1 - r2 y0^2 = 1 - eta0 y0,
//   eta = eta0 (1 - e)^(-1/2) = eta0 (1 + e (1/2 + 3e/8)) + O(e^3),
// a third-order correction (truncation ~2^-62) written as two nested FMAs:
// |t - (1 - sqrt(r2))| <= 2.8e-16 over r2 in [1e-10, 1.2] (pair_lab), the
// same ulp-level error as the 6-instruction rsqrt refinement it replaces.
__device__ __forceinline__ double t_from_seed(double r2, double y0) {
  const double eta0 = r2 * y0;
  const double e = fma(-eta0, y0, 1.0);
  const double p = fma(e, 0.375, 0.5);
  const double w = fma(e, p, 1.0);
  return fma(-eta0, w, 1.0);
}

__device__ __forceinline__ double t_from_r2(double r2) { return t_from_seed(r2, rsqrt_approx(r2)); }

// phi = max(t, 0)^4 (5 - 4t) from r2 and its rsqrt seed y0 = MUFU.RSQ64H(r2)
__device__ __forceinline__ double phi_from_seed(double r2, double y0) {
  double t = clamp_nonneg(t_from_seed(r2, y0));
  const double q = fma(-4.0, t, 5.0);
  t = t * t;
  return (t * t) * q;
}

// Throughput pair: target (px,py,pz) and support (sx,sy,sz) already scaled
// by 1/R; pair_phi() returns phi(|p - s|), pair_accum() accumulates
// w * phi(|p - s|) into (ax, ay, az).
//
// FP64-pipe budget per pair: 3 DADD (differences) + 3 (r^2) + 5 (t = 1 - eta)
// + 4 (q = 5 - 4t = 4 eta + 1, t^2, t^4, t^4 q) + 3 DFMA (accumulate) = 18.
// t_from_r2() never forms sqrt(r2) separately; see there. r2 carries a 1e-200
// addend (eta = 1e-100 gives phi = 1 exactly, like eta = 0) so the rsqrt never
// sees zero. The clamp t = max(t, 0) is one integer instruction.
__device__ __forceinline__ double pair_r2(double px, double py, double pz,
                                          double sx, double sy, double sz) {
  const double dx = px - sx, dy = py - sy, dz = pz - sz;
  // the 1e-200 rides in the first FMA: it vanishes in the rounding of any
  // r2 > 1e-184 and keeps the rsqrt away from zero for coincident points
  return fma(dz, dz, fma(dy, dy, fma(dx, dx, 1e-200)));
}

__device__ __forceinline__ double pair_phi(double px, double py, double pz,
                                           double sx, double sy, double sz) {
  const double r2 = pair_r2(px, py, pz, sx, sy, sz);
  return phi_from_seed(r2, rsqrt_approx(r2));
}

__device__ __forceinline__ void pair_accum(double px, double py, double pz,
                                           double sx, double sy, double sz,
                                           double wx, double wy, double wz,
                                           double& ax, double& ay, double& az) {
  const double f = pair_phi(px, py, pz, sx, sy, sz);
  ax = fma(wx, f, ax);
  ay = fma(wy, f, ay);
  az = fma(wz, f, az);
}

// residual norm exactly as selection.py:220-221: sqrt((r0*r0 + r1*r1) + r2*r2)
__device__ __forceinline__ double residual_norm(double dx, double dy, double dz,
                                                double ux, double uy, double uz) {
  double r0 = __dsub_rn(dx, ux), r1 = __dsub_rn(dy, uy), r2 = __dsub_rn(dz, uz);
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(r0, r0), __dmul_rn(r1, r1)),
                              __dmul_rn(r2, r2)));
}

// ------------------------------------------------------- (err, pos) argmax
// Larger error wins; exact ties go to the lowest position (= lowest id, since
// boundary indices are strictly increasing: selection.py:46-52, 231-234).
struct Best {
  double err;
  int pos;
};

__device__ __forceinline__ bool better(double e1, int p1, double e2, int p2) {
  return e1 > e2 || (e1 == e2 && p1 < p2);
}

__device__ __forceinline__ Best best_of(Best a, Best b) {
  return better(b.err, b.pos, a.err, a.pos) ? b : a;
}

// Warp arg-max in three warp-wide integer reductions (redux.sync) instead of
// a five-level shuffle butterfly of (double, int) pairs: the error's bit
// pattern is mapped to an unsigned key that orders like the double (sign bit
// flipped for err >= 0, all bits inverted for the negative sentinel), its high
// and low words are maximised in turn, and the lowest position among the
// lanes holding the maximum wins -- the same (err, lowest pos) result as
// folding the lanes with better(). Every lane returns the warp's best.
__device__ __forceinline__ Best warp_best(Best b) {
  const unsigned full = 0xffffffffu;
  const unsigned hi = (unsigned)__double2hiint(b.err), lo = (unsigned)__double2loint(b.err);
  const unsigned neg = (unsigned)((int)hi >> 31);
  const unsigned khi = hi ^ (neg | 0x80000000u), klo = lo ^ neg;
  const unsigned mhi = __reduce_max_sync(full, khi);
  const unsigned mlo = __reduce_max_sync(full, khi == mhi ? klo : 0u);
  const bool top = khi == mhi && klo == mlo;
  const unsigned mp = __reduce_min_sync(full, top ? (unsigned)b.pos : 0xffffffffu);
  const unsigned mneg = (mhi & 0x80000000u) ? 0u : 0xffffffffu;
  return Best{__hiloint2double((int)(mhi ^ (mneg | 0x80000000u)), (int)(mlo ^ mneg)), (int)mp};
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}

// ---------------------------------------------------------- memory helpers
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ int ldcg(const int* p) { return __ldcg(p); }

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ------------------------------------------------------------ grid barrier
// Sense-counting barrier for a cooperative (co-resident) grid. A spin that
// exceeds the watchdog sets *fault and traps instead of hanging the GPU.
struct GridBarrier {
  unsigned count;
  unsigned gen;
};

__device__ __forceinline__ void grid_sync(GridBarrier* bar, unsigned nblocks, int* fault) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g = ld_acquire(&bar->gen);
    __threadfence();
    unsigned prev = atomicAdd(&bar->count, 1u);
    if (prev == nblocks - 1) {
      bar->count = 0;
      __threadfence();
      st_release(&bar->gen, g + 1);
    } else {
      uint64_t t0 = globaltimer_ns();
      unsigned spins = 0;
      while (ld_acquire(&bar->gen) == g) {
        if ((++spins & 1023u) == 0 && globaltimer_ns() - t0 > 20ull * 1000000000ull) {
          atomicExch(fault, 1);
          __trap();
        }
      }
    }
    __threadfence();
  }
  __syncthreads();
}

}  // namespace rbf
