// Device-resident GCB / greedy selection loop (replaces reference
// selection.py:274-421 `_gcb_run` statement for statement, seeds
// selection.py:198-212 included; SURVEY.md Appendix A lists the semantics).
//
// One persistent kernel. Every CTA of the team runs the same control flow:
// decisions (arg-max, accept/reject, streaks, termination) are recomputed
// redundantly by every CTA from the same data in the same order, so they
// agree bit for bit and the only synchronisation is a team barrier between
// data-parallel phases:
//
//   scan   supports staged into shared memory (SoA), group errors, per-CTA
//          (err, lowest position) partials for all and for eligible nodes   | B1
//   append row phi(|p - s_j|/R) (reference arithmetic, every CTA), then
//          c0 = Li row                                                        | B2
//          r  = row - L c0                                                    | B3
//          c  = c0 + Li r, per-CTA partial sums c.c and c.y                   | B4
//          pivot^2 = 1 - c.c; l; y_n = (d - c.y)/l;
//          u = Li^T c, v = Li^T y  ->  Li[n] = -u/l, weights v + Li[n] y_n,
//          L[n] = [c, l]                                                      | B5
//
// Team = one 16-CTA thread-block cluster (hardware barrier.cluster, ~0.3 us)
// for small and medium problems, or a cooperative grid of one CTA per SM
// with a single-word software barrier (~1.2 us) when group scans are large.
// Every loop in a phase issues its global loads back to back (unrolled), so
// a phase costs about one L2 round trip (~160 ns on B200) plus its math.
#include <cooperative_groups.h>

#include <cmath>
#include <cstdint>

#include "rbf_common.cuh"
#include "rbf_internal.h"
#include "rbf_tri.cuh"

namespace cg = cooperative_groups;

namespace rbf {

constexpr int kLoopThreads = 512;
constexpr int kLoopWarps = kLoopThreads / 32;
constexpr int kClusterCTAs = 16;
constexpr int kSupTile = 2048;       // supports staged per scan tile (SoA, 96 KB)
constexpr int kRowSmemMax = 8192;    // row held in shared memory (64 KB)
constexpr int kAutoClusterMaxCard = 2048;

struct LoopScratch {
  unsigned* bar;   // grid barrier word
  int* fault;
  Best* part;      // [ctas][2]: unrestricted, eligible-only
  double* red;     // [ctas][4]: c.c, c.y(3)
  double* err;     // [nb]   errors of the group being scanned
  double* dmin;    // [nb]   seed farthest-point distances
  double* c0;      // [cap]
  double* r;       // [cap]
  double* c1;      // [cap]
};

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

static LoopScratch carve(void* base, int nb, int cap, int ctas, size_t* total) {
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* q = p ? p + off : nullptr;
    off += align256(bytes);
    return q;
  };
  LoopScratch s{};
  char* b = take(64);
  s.bar = reinterpret_cast<unsigned*>(b);
  s.fault = reinterpret_cast<int*>(b ? b + 32 : nullptr);
  s.part = reinterpret_cast<Best*>(take(sizeof(Best) * 2 * ctas));
  s.red = reinterpret_cast<double*>(take(sizeof(double) * 4 * ctas));
  s.err = reinterpret_cast<double*>(take(sizeof(double) * (size_t)nb));
  s.dmin = reinterpret_cast<double*>(take(sizeof(double) * (size_t)nb));
  s.c0 = reinterpret_cast<double*>(take(sizeof(double) * (size_t)cap));
  s.r = reinterpret_cast<double*>(take(sizeof(double) * (size_t)cap));
  s.c1 = reinterpret_cast<double*>(take(sizeof(double) * (size_t)cap));
  if (total) *total = off;
  return s;
}

// ------------------------------------------------------------------ teams
struct ClusterTeam {
  __device__ __forceinline__ void sync() const { cg::this_cluster().sync(); }
};

// Single-word grid barrier (the scheme of cooperative_groups' grid sync):
// CTA 0 adds 2^31 - (G - 1), the others add 1, so bit 31 flips exactly when
// all G have arrived and the low bits return to zero. A waiter spinning
// past the watchdog sets *fault and traps instead of hanging the GPU.
struct GridTeam {
  unsigned* word;
  int* fault;
  __device__ __forceinline__ void sync() const {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned add = blockIdx.x == 0 ? (0x80000000u - (gridDim.x - 1)) : 1u;
      __threadfence();
      const unsigned old = atomicAdd(word, add);
      uint64_t t0 = 0;
      unsigned spins = 0;
      while (((old ^ ld_acquire(word)) & 0x80000000u) == 0) {
        if ((++spins & 1023u) == 0) {
          const uint64_t now = globaltimer_ns();
          if (t0 == 0) t0 = now;
          else if (now - t0 > 20ull * 1000000000ull) {
            atomicExch(fault, 1);
            __trap();
          }
        }
      }
    }
    __syncthreads();
  }
};

struct Shared {
  double sx[kSupTile], sy[kSupTile], sz[kSupTile];
  double wx[kSupTile], wy[kSupTile], wz[kSupTile];
  double red[kLoopWarps * 32 * 4];
  Best wb[kLoopWarps][2];
  double wred[kLoopWarps][4];
  Best bcast[2];
  double dbl[8];
  double phase[12];
};

// CTA 0's SM clock at phase boundaries (diagnostics in rbf_gcb_state)
// (thread 0 of CTA 0 only; accumulators live in shared memory)
struct PhaseClock {
  double* acc;
  long long last;
  bool on;
  __device__ __forceinline__ void start(double* smem_acc) {
    acc = smem_acc;
    on = blockIdx.x == 0 && threadIdx.x == 0;
    if (on) {
      for (int i = 0; i < 12; ++i) acc[i] = 0.0;
      last = clock64();
    }
  }
  __device__ __forceinline__ void mark(int phase) {
    if (on) {
      const long long now = clock64();
      acc[phase] += (double)(now - last);
      last = now;
    }
  }
  __device__ __forceinline__ void count(int slot) {
    if (on) acc[slot] += 1.0;
  }
};

__device__ __forceinline__ uint64_t leader_timer() {
  return (blockIdx.x == 0 && threadIdx.x == 0) ? globaltimer_ns() : 0ull;
}

// Fold per-warp bests into one per CTA (thread 0 of warp 0 ends with it).
__device__ __forceinline__ void cta_best(Shared& sh, Best b, int slot, Best* out) {
  b = warp_best(b);
  if ((threadIdx.x & 31) == 0) sh.wb[threadIdx.x >> 5][slot] = b;
  __syncthreads();
  if (threadIdx.x < 32) {
    Best v = threadIdx.x < kLoopWarps ? sh.wb[threadIdx.x][slot] : Best{-1.0, 0x7fffffff};
    v = warp_best(v);
    if (threadIdx.x == 0) *out = v;
  }
}

// All CTAs fold the per-CTA partials (G <= 148) in the same fixed tree order.
__device__ __forceinline__ void fold_partials(const LoopScratch& s, Shared& sh, int nslots) {
  const int G = gridDim.x;
  if (threadIdx.x < 32 * nslots) {
    const int slot = threadIdx.x >> 5, lane = threadIdx.x & 31;
    Best b{-1.0, 0x7fffffff};
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const int c = lane + 32 * q;
      if (c < G) {
        const Best v{__ldcg(&s.part[2 * c + slot].err), __ldcg(&s.part[2 * c + slot].pos)};
        b = best_of(b, v);
      }
    }
    b = warp_best(b);
    if (lane == 0) sh.bcast[slot] = b;
  }
  __syncthreads();
}

// ------------------------------------------------------------------ scan
// Errors of `card` boundary rows (positions gpos[t], or t when gpos is null)
// against the n supports; writes err[t] and this CTA's two arg-max partials.
// The team's CTAs split the rows; inside a CTA, S lanes share one row and
// split its supports (S chosen so the rows fill the CTA), supports are
// staged through shared memory in SoA tiles.
__device__ void scan_phase(const rbf_gcb_args& a, const LoopScratch& s, Shared& sh,
                           const int* gpos, int card, int n, double inv_r) {
  const int tid = threadIdx.x, G = gridDim.x;
  const int lo = (int)((int64_t)card * blockIdx.x / G);
  const int hi = (int)((int64_t)card * (blockIdx.x + 1) / G);
  const int mine = hi - lo;
  int S = 32;
  while (S > 1 && mine * S > kLoopThreads) S >>= 1;
  while (S > 1 && (S >> 1) >= n) S >>= 1;
  const int groups = kLoopThreads / S;
  const int g = tid / S, sub = tid % S;
  const int rounds = (mine + groups - 1) / groups;
  const double* gx = a.sup;
  const int cap = a.cap;

  Best bu{-1.0, 0x7fffffff}, br{-1.0, 0x7fffffff};
  for (int rd = 0; rd < rounds; ++rd) {
    const int t = lo + rd * groups + g;
    const bool active = t < hi;
    int pos = 0;
    double px = 0.0, py = 0.0, pz = 0.0;
    if (active) {
      pos = gpos ? __ldg(gpos + t) : t;
      px = __ldg(a.points + 3 * (int64_t)pos) * inv_r;
      py = __ldg(a.points + 3 * (int64_t)pos + 1) * inv_r;
      pz = __ldg(a.points + 3 * (int64_t)pos + 2) * inv_r;
    }
    double ax = 0.0, ay = 0.0, az = 0.0;
    for (int t0 = 0; t0 < n; t0 += kSupTile) {
      const int cnt = min(kSupTile, n - t0);
      if (rd == 0 || n > kSupTile) {
        __syncthreads();
        for (int j = tid; j < cnt; j += kLoopThreads) {
          sh.sx[j] = __ldcg(gx + t0 + j) * inv_r;
          sh.sy[j] = __ldcg(gx + cap + t0 + j) * inv_r;
          sh.sz[j] = __ldcg(gx + 2 * cap + t0 + j) * inv_r;
          sh.wx[j] = __ldcg(gx + 3 * cap + t0 + j);
          sh.wy[j] = __ldcg(gx + 4 * cap + t0 + j);
          sh.wz[j] = __ldcg(gx + 5 * cap + t0 + j);
        }
        __syncthreads();
      }
      if (active) {
#pragma unroll 4
        for (int j = sub; j < cnt; j += S)
          pair_accum(px, py, pz, sh.sx[j], sh.sy[j], sh.sz[j], sh.wx[j], sh.wy[j], sh.wz[j], ax, ay,
                     az);
      }
    }
    for (int off = S >> 1; off > 0; off >>= 1) {
      ax += __shfl_xor_sync(0xffffffffu, ax, off);
      ay += __shfl_xor_sync(0xffffffffu, ay, off);
      az += __shfl_xor_sync(0xffffffffu, az, off);
    }
    if (active && sub == 0) {
      const double e = residual_norm(__ldg(a.disp + 3 * (int64_t)pos), __ldg(a.disp + 3 * (int64_t)pos + 1),
                                     __ldg(a.disp + 3 * (int64_t)pos + 2), ax, ay, az);
      s.err[t] = e;
      if (better(e, pos, bu.err, bu.pos)) bu = Best{e, pos};
      if (!__ldcg(reinterpret_cast<const unsigned char*>(a.inel) + pos) && better(e, pos, br.err, br.pos))
        br = Best{e, pos};
    }
  }
  cta_best(sh, bu, 0, &s.part[2 * blockIdx.x]);
  cta_best(sh, br, 1, &s.part[2 * blockIdx.x + 1]);
}

// Next candidate after a rejection: eligible arg-max over the stored group
// errors (rare path; every CTA scans the whole group redundantly).
__device__ Best rescan_candidate(const rbf_gcb_args& a, const LoopScratch& s, Shared& sh,
                                 const int* gpos, int card) {
  Best b{-1.0, 0x7fffffff};
  for (int t = threadIdx.x; t < card; t += kLoopThreads) {
    const int pos = gpos ? __ldg(gpos + t) : t;
    if (__ldcg(reinterpret_cast<const unsigned char*>(a.inel) + pos)) continue;
    const double e = __ldcg(s.err + t);
    if (better(e, pos, b.err, b.pos)) b = Best{e, pos};
  }
  __syncthreads();
  cta_best(sh, b, 1, &sh.bcast[1]);
  __syncthreads();
  return sh.bcast[1];
}

// ------------------------------------------------------------------ seeds
// selection.py:198-212: argmax |d| (first occurrence), then twice
// argmax dmin with dmin = min(dmin, |P - P_next|); norms are
// sqrt((x0*x0 + x1*x1) + x2*x2), numpy's bits for a (n, 3) row norm.
template <class Team>
__device__ void device_seeds(const rbf_gcb_args& a, const LoopScratch& s, Shared& sh,
                             const Team& team, int seeds[3]) {
  const int nb = a.nb, G = gridDim.x;
  const int lo = (int)((int64_t)nb * blockIdx.x / G), hi = (int)((int64_t)nb * (blockIdx.x + 1) / G);
  Best b{-1.0, 0x7fffffff};
  for (int i = lo + threadIdx.x; i < hi; i += kLoopThreads) {
    const double m = residual_norm(__ldg(a.disp + 3 * (int64_t)i), __ldg(a.disp + 3 * (int64_t)i + 1),
                                   __ldg(a.disp + 3 * (int64_t)i + 2), 0.0, 0.0, 0.0);
    if (better(m, i, b.err, b.pos)) b = Best{m, i};
  }
  cta_best(sh, b, 0, &s.part[2 * blockIdx.x]);
  team.sync();
  fold_partials(s, sh, 1);
  seeds[0] = sh.bcast[0].pos;
  for (int q = 1; q < 3; ++q) {
    const int p = seeds[q - 1];
    const double qx = __ldg(a.points + 3 * (int64_t)p), qy = __ldg(a.points + 3 * (int64_t)p + 1),
                 qz = __ldg(a.points + 3 * (int64_t)p + 2);
    Best bb{-1.0, 0x7fffffff};
    for (int i = lo + threadIdx.x; i < hi; i += kLoopThreads) {
      double d = residual_norm(__ldg(a.points + 3 * (int64_t)i), __ldg(a.points + 3 * (int64_t)i + 1),
                               __ldg(a.points + 3 * (int64_t)i + 2), qx, qy, qz);
      if (q == 2) d = fmin(s.dmin[i], d);
      s.dmin[i] = d;
      if (better(d, i, bb.err, bb.pos)) bb = Best{d, i};
    }
    __syncthreads();
    cta_best(sh, bb, 0, &s.part[2 * blockIdx.x]);
    team.sync();
    fold_partials(s, sh, 1);
    seeds[q] = sh.bcast[0].pos;
  }
}

// ------------------------------------------------------------------ append
enum AppendResult { kAccepted = 0, kRejectDup = 1, kRejectPivot = 2 };

// Warp-cooperative dot product of packed row i of A with x[0..i], every load
// of the lane issued before the first FMA (8 in flight per lane).
template <typename XL>
__device__ __forceinline__ double row_dot(const double* arow, int len, XL xload, int lane) {
  double acc = 0.0;
  for (int j0 = 0; j0 < len; j0 += 8 * kWarp) {
    double av[8], xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = j0 + u * kWarp + lane;
      av[u] = j < len ? __ldcg(arow + j) : 0.0;
      xv[u] = j < len ? xload(j) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = fma(av[u], xv[u], acc);
  }
  return warp_sum(acc);
}

// Bordered append of boundary position `pos` (reference core.py:153-185 via
// selection.py:288-297 / 341-356). All CTAs call it; the result is uniform.
template <class Team>
__device__ int append_node(const rbf_gcb_args& a, const LoopScratch& s, Shared& sh, double* row,
                           const Team& team, int pos, int& n, bool check_dup, double inv_r,
                           double* pivot2_out, PhaseClock& pc) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x;
  const double px = __ldg(a.points + 3 * (int64_t)pos), py = __ldg(a.points + 3 * (int64_t)pos + 1),
               pz = __ldg(a.points + 3 * (int64_t)pos + 2);
  // row[j] = phi(cdist(p, s_j) / R) with the reference's rounding; min distance
  double dmin = INFINITY;
  for (int j = tid; j < n; j += kLoopThreads) {
    const double d = cdist_exact(px, py, pz, __ldcg(a.sup + j), __ldcg(a.sup + a.cap + j),
                                 __ldcg(a.sup + 2 * (int64_t)a.cap + j));
    row[j] = phi_exact(d, a.radius);
    dmin = fmin(dmin, d);
  }
  dmin = warp_min(dmin);
  if (lane == 0) sh.wred[warp][0] = dmin;
  __syncthreads();
  if (tid < 32) {
    double m = tid < kLoopWarps ? sh.wred[tid][0] : INFINITY;
    m = warp_min(m);
    if (tid == 0) sh.dbl[0] = m;
  }
  __syncthreads();
  if (check_dup && n > 0 && sh.dbl[0] < a.dup_dist) return kRejectDup;

  pc.mark(1);
  const int gw = blockIdx.x * kLoopWarps + warp, nw = G * kLoopWarps;
  // c0 = Li row
  for (int i = gw; i < n; i += nw) {
    const double v = row_dot(a.Li + tri_off(i), i + 1, [&](int j) { return row[j]; }, lane);
    if (lane == 0) s.c0[i] = v;
  }
  team.sync();
  pc.mark(2);
  // r = row - L c0
  for (int i = gw; i < n; i += nw) {
    const double v = row_dot(a.L + tri_off(i), i + 1, [&](int j) { return __ldcg(s.c0 + j); }, lane);
    if (lane == 0) s.r[i] = row[i] - v;
  }
  team.sync();
  pc.mark(3);
  // c = c0 + Li r, with per-warp partial sums of c.c and c.y
  double pcc = 0.0, pcy0 = 0.0, pcy1 = 0.0, pcy2 = 0.0;
  for (int i = gw; i < n; i += nw) {
    const double v = row_dot(a.Li + tri_off(i), i + 1, [&](int j) { return __ldcg(s.r + j); }, lane);
    if (lane == 0) {
      const double c = __ldcg(s.c0 + i) + v;
      s.c1[i] = c;
      pcc = fma(c, c, pcc);
      pcy0 = fma(c, __ldcg(a.y + 3 * (int64_t)i), pcy0);
      pcy1 = fma(c, __ldcg(a.y + 3 * (int64_t)i + 1), pcy1);
      pcy2 = fma(c, __ldcg(a.y + 3 * (int64_t)i + 2), pcy2);
    }
  }
  if (lane == 0) {
    sh.wred[warp][0] = pcc;
    sh.wred[warp][1] = pcy0;
    sh.wred[warp][2] = pcy1;
    sh.wred[warp][3] = pcy2;
  }
  __syncthreads();
  if (tid < 4) {
    double t = 0.0;
    for (int w = 0; w < kLoopWarps; ++w) t += sh.wred[w][tid];
    s.red[4 * blockIdx.x + tid] = t;
  }
  team.sync();
  pc.mark(4);
  // every CTA folds the G partials with the same fixed tree
  if (tid < 128) {
    const int q = tid >> 5, ln = tid & 31;
    double t = 0.0;
#pragma unroll
    for (int u = 0; u < 5; ++u) {
      const int c = ln + 32 * u;
      if (c < G) t += __ldcg(s.red + 4 * c + q);
    }
    t = warp_sum(t);
    if (ln == 0) sh.dbl[1 + q] = t;
  }
  __syncthreads();
  const double pivot2 = 1.0 - sh.dbl[1];  // row[n] = phi(0) = 1 exactly
  *pivot2_out = pivot2;
  if (!(pivot2 > 0.0)) {
    __syncthreads();
    return kRejectPivot;
  }
  const double l = sqrt(pivot2);
  const double yn0 = (__ldg(a.disp + 3 * (int64_t)pos) - sh.dbl[2]) / l;
  const double yn1 = (__ldg(a.disp + 3 * (int64_t)pos + 1) - sh.dbl[3]) / l;
  const double yn2 = (__ldg(a.disp + 3 * (int64_t)pos + 2) - sh.dbl[4]) / l;
  // u = Li^T c, v = Li^T y -> new Li row, new L row, refreshed weights
  double* Lrow = a.L + tri_off(n);
  double* Lirow = a.Li + tri_off(n);
  double* wgt = a.sup + 3 * (int64_t)a.cap;
  const int cap = a.cap;
  tri_cols<4, kLoopWarps>(
      a.Li, n,
      [&](int i, int c) { return c == 0 ? __ldcg(s.c1 + i) : __ldcg(a.y + 3 * (int64_t)i + (c - 1)); },
      (int)blockIdx.x, G, sh.red, [&](int j, const double* sum) {
        const double lij = -sum[0] / l;
        Lirow[j] = lij;
        Lrow[j] = __ldcg(s.c1 + j);
        wgt[j] = fma(lij, yn0, sum[1]);
        wgt[cap + j] = fma(lij, yn1, sum[2]);
        wgt[2 * cap + j] = fma(lij, yn2, sum[3]);
      });
  if (blockIdx.x == 0 && tid == 0) {
    Lirow[n] = 1.0 / l;
    Lrow[n] = l;
    a.y[3 * (int64_t)n] = yn0;
    a.y[3 * (int64_t)n + 1] = yn1;
    a.y[3 * (int64_t)n + 2] = yn2;
    a.sup[n] = px;
    a.sup[cap + n] = py;
    a.sup[2 * cap + n] = pz;
    wgt[n] = yn0 / l;
    wgt[cap + n] = yn1 / l;
    wgt[2 * cap + n] = yn2 / l;
    a.sel[n] = pos;
  }
  if (tid == 0) a.inel[pos] = 1;
  n += 1;
  team.sync();
  pc.mark(5);
  return kAccepted;
}

// ------------------------------------------------------------------ kernel
template <class Team>
__device__ void gcb_body(const rbf_gcb_args& a, const LoopScratch& s, const Team& team) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Shared& sh = *reinterpret_cast<Shared*>(smem_raw);
  double* row = reinterpret_cast<double*>(smem_raw + sizeof(Shared));
  const int tid = threadIdx.x;
  const bool leader = blockIdx.x == 0 && tid == 0;
  const double inv_r = 1.0 / a.radius;
  rbf_gcb_state* st = a.state;

  int n = __ldcg(&st->n);
  int k = __ldcg(&st->k);
  int streak_ok = __ldcg(&st->streak_ok);
  int streak_noadd = __ldcg(&st->streak_noadd);
  int nrec = __ldcg(&st->n_records);
  int done_loop = __ldcg(&st->done_loop);
  double t2_carry = __ldcg(&st->t2_carry);
  const int m = a.m;

  PhaseClock pc;
  pc.start(sh.phase);
  auto save = [&](int status) {
    if (leader) {
      for (int i = 0; i < 12; ++i) st->phase_cycles[i] += sh.phase[i];
      st->n = n;
      st->k = k;
      st->streak_ok = streak_ok;
      st->streak_noadd = streak_noadd;
      st->n_records = nrec;
      st->done_loop = done_loop;
      st->t2_carry = t2_carry;
      st->status = status;
    }
  };

  if (n == 0) {
    if (a.cap < 3 || a.rec_cap < 1) {
      save(RBF_EGROW);
      return;
    }
    int seeds[3];
    device_seeds(a, s, sh, team, seeds);
    pc.mark(7);
    // seed appends (selection.py:288-297): no near-duplicate guard, NotPD propagates
    for (int q = 0; q < 3; ++q) {
      double p2 = 0.0;
      const int res = append_node(a, s, sh, row, team, seeds[q], n, false, inv_r, &p2, pc);
      if (res != kAccepted) {
        if (leader) {
          st->fail_row = n;
          st->fail_pivot2 = p2;
        }
        save(RBF_ENOTPD);
        return;
      }
    }
    k = 3;
    streak_ok = streak_noadd = 0;
    nrec = 0;
    t2_carry = 0.0;
  }

  while (!done_loop) {
    if (n >= a.max_supports) {
      done_loop = 1;
      break;
    }
    if (n >= a.cap || nrec >= a.rec_cap || n >= kRowSmemMax) {
      save(RBF_EGROW);
      return;
    }
    const uint64_t t_a = leader_timer();
    const int gi = k % m;
    const int off = __ldg(a.group_off + gi);
    const int card = __ldg(a.group_off + gi + 1) - off;
    const int* gpos = a.group_pos + off;
    pc.mark(6);
    scan_phase(a, s, sh, gpos, card, n, inv_r);
    team.sync();
    pc.mark(0);
    pc.count(10);
    fold_partials(s, sh, 2);
    const Best bu = sh.bcast[0];
    Best cand = sh.bcast[1];
    const uint64_t t_b = leader_timer();
    const int n_before = n;
    const double local_max = bu.err;
    bool added = false;
    int added_pos = -1;
    if (local_max > a.tol) {
      while (cand.pos != 0x7fffffff && cand.err > a.tol) {
        double p2;
        const int res = append_node(a, s, sh, row, team, cand.pos, n, true, inv_r, &p2, pc);
        pc.count(9);
        if (res == kAccepted) {
          added = true;
          added_pos = cand.pos;
          break;
        }
        if (tid == 0) {
          a.inel[cand.pos] = 1;
          __threadfence();
        }
        __syncthreads();
        cand = rescan_candidate(a, s, sh, gpos, card);
      }
    }
    const uint64_t t_c = leader_timer();
    if (leader) {
      rbf_gcb_record rec;
      rec.group = gi;
      rec.node_pos = added ? added_pos : bu.pos;
      rec.added = added ? 1 : 0;
      rec.n_before = n_before;
      rec.local_max = local_max;
      rec.t1_s = (double)(t_b - t_a) * 1e-9;
      rec.t2_s = t2_carry;
      a.records[nrec] = rec;
    }
    nrec += 1;
    t2_carry = (local_max > a.tol) ? (double)(t_c - t_b) * 1e-9 : 0.0;
    if (!added) {
      streak_noadd += 1;
      streak_ok = (local_max <= a.tol) ? streak_ok + 1 : 0;
      if (streak_ok >= m) {
        done_loop = 1;
        break;
      }
      if (streak_noadd >= m) {
        save(RBF_ESTALL);
        return;
      }
    } else {
      streak_noadd = 0;
      streak_ok = 0;
    }
    k += 1;
  }

  // final verification sweep (selection.py:388-412)
  if (nrec >= a.rec_cap) {
    save(RBF_EGROW);
    return;
  }
  const uint64_t t_a = leader_timer();
  pc.mark(6);
  scan_phase(a, s, sh, nullptr, a.nb, n, inv_r);
  team.sync();
  fold_partials(s, sh, 1);
  pc.mark(8);
  const Best bu = sh.bcast[0];
  const uint64_t t_b = leader_timer();
  if (leader) {
    rbf_gcb_record rec;
    rec.group = -1;
    rec.node_pos = bu.pos;
    rec.added = 0;
    rec.n_before = n;
    rec.local_max = bu.err;
    rec.t1_s = (double)(t_b - t_a) * 1e-9;
    rec.t2_s = t2_carry;
    a.records[nrec] = rec;
    st->final_max = bu.err;
    st->final_pos = bu.pos;
  }
  nrec += 1;
  save(1);
}

__global__ void __launch_bounds__(kLoopThreads, 1) gcb_cluster_kernel(rbf_gcb_args a, LoopScratch s) {
  gcb_body(a, s, ClusterTeam{});
}

__global__ void __launch_bounds__(kLoopThreads, 1) gcb_grid_kernel(rbf_gcb_args a, LoopScratch s) {
  gcb_body(a, s, GridTeam{s.bar, s.fault});
}

static size_t loop_smem_bytes() { return sizeof(Shared) + (size_t)kRowSmemMax * sizeof(double); }

static int resolve_mode(int mode, int nb, int m) {
  if (mode != RBF_GCB_AUTO) return mode;
  const int card = (nb + m - 1) / m;
  return card <= kAutoClusterMaxCard ? RBF_GCB_CLUSTER : RBF_GCB_GRID;
}

}  // namespace rbf

using namespace rbf;

extern "C" int rbf_device_info(int device, int* sm_count_host, int* loop_ctas_host) {
  const int sms = sm_count(device);
  if (sms <= 0) return set_error(RBF_ECUDA, "no CUDA device %d", device);
  if (sm_count_host) *sm_count_host = sms;
  if (loop_ctas_host) *loop_ctas_host = sms;
  return RBF_OK;
}

extern "C" int rbf_gcb_ctas(int32_t mode, int32_t nb, int32_t m, int32_t* ctas_host,
                            int32_t* resolved_mode_host) {
  if (nb < 1 || m < 1) return set_error(RBF_EARG, "bad nb/m");
  int dev = 0;
  RBF_CUDA_TRY(cudaGetDevice(&dev));
  const int r = resolve_mode(mode, nb, m);
  const int sms = sm_count(dev);
  if (sms <= 0) return set_error(RBF_ECUDA, "no CUDA device");
  if (ctas_host) *ctas_host = r == RBF_GCB_CLUSTER ? kClusterCTAs : sms;
  if (resolved_mode_host) *resolved_mode_host = r;
  return RBF_OK;
}

extern "C" size_t rbf_gcb_scratch_bytes(int32_t nb, int32_t cap, int32_t ctas) {
  size_t total = 0;
  carve(nullptr, nb, cap, ctas, &total);
  return total;
}

extern "C" int rbf_gcb_run(const rbf_gcb_args* args, void* stream) {
  if (!args) return set_error(RBF_EARG, "null args");
  const rbf_gcb_args& a = *args;
  if (a.nb < 3 || a.m < 1 || a.m > a.nb) return set_error(RBF_EARG, "bad nb/m");
  if (!(a.radius > 0.0) || !(a.tol > 0.0)) return set_error(RBF_EARG, "bad radius/tol");
  if (!a.points || !a.disp || !a.group_pos || !a.group_off || !a.L || !a.Li || !a.y || !a.sup ||
      !a.sel || !a.inel || !a.records || !a.state || !a.scratch)
    return set_error(RBF_EARG, "null pointer");
  int ctas = 0, mode = 0;
  int rc = rbf_gcb_ctas(a.mode, a.nb, a.m, &ctas, &mode);
  if (rc != RBF_OK) return rc;
  size_t need = 0;
  LoopScratch s = carve(a.scratch, a.nb, a.cap, ctas, &need);
  if (a.scratch_bytes < need)
    return set_error(RBF_EARG, "scratch too small (%zu < %zu)", a.scratch_bytes, need);
  cudaStream_t st = as_stream(stream);
  RBF_CUDA_TRY(cudaMemsetAsync(s.bar, 0, 64, st));
  const size_t smem = loop_smem_bytes();
  rbf_gcb_args acopy = a;
  if (mode == RBF_GCB_CLUSTER) {
    RBF_CUDA_TRY(cudaFuncSetAttribute(gcb_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    RBF_CUDA_TRY(cudaFuncSetAttribute(gcb_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kClusterCTAs);
    cfg.blockDim = dim3(kLoopThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kClusterCTAs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    RBF_CUDA_TRY(cudaLaunchKernelEx(&cfg, gcb_cluster_kernel, acopy, s));
  } else {
    RBF_CUDA_TRY(cudaFuncSetAttribute(gcb_grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    void* kargs[] = {&acopy, &s};
    RBF_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)gcb_grid_kernel, dim3(ctas), dim3(kLoopThreads),
                                             kargs, smem, st));
  }
  return RBF_OK;
}
