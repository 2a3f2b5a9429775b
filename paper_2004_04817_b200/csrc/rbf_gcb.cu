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
//   scan   group errors, per-CTA (err, lowest position) partials for all and
//          for eligible nodes                                                | B1
//   append row phi(|p - s_j|/R) (reference arithmetic, every CTA), then
//          c0 = Li row                                                        | B2
//          r  = row - L c0                                                    | B3
//          c  = c0 + Li r, per-CTA partial sums c.c and c.y                   | B4
//          pivot^2 = 1 - c.c; l; y_n = (d - c.y)/l;
//          u = Li^T c, v = Li^T y  ->  Li[n] = -u/l, weights v + Li[n] y_n,
//          L[n] = [c, l]                                                      | B5
//
// Two storage paths behind one driver (gcb_driver):
//  * SmemPath: one 16-CTA thread-block cluster (hardware barrier.cluster,
//    ~0.3 us). Supports, weights and the work vectors are replicated in every
//    CTA's shared memory; a value computed by one CTA is stored into all 16
//    copies through distributed shared memory, so a phase reads nothing but
//    its factor rows from L2. Group scans use 4 targets per lane.
//  * GlobalPath: all state in global memory (L2), team = the same cluster or
//    a cooperative grid of one CTA per SM (large scans, n >= 1024).
// Both keep the global copies (L, Li, y, supports, weights) current, so a
// run can pause (RBF_EGROW) and resume in either path.
#include <cooperative_groups.h>

#include <cmath>
#include <cstdint>
#include <mutex>
#include <set>
#include <utility>

#include "rbf_common.cuh"
#include "rbf_internal.h"
#include "rbf_tri.cuh"

namespace cg = cooperative_groups;

namespace rbf {

constexpr int kLoopThreads = 512;
constexpr int kLoopWarps = kLoopThreads / 32;
static_assert(kLoopThreads == 512, "scan prologues shift by log2(kLoopThreads) = 9");
constexpr int kClusterCTAs = 16;
static_assert(kClusterCTAs == 16, "one-cluster scans split rows with >> 4");
constexpr int kSupTile = 2048;       // GlobalPath: supports staged per scan tile
constexpr int kRowSmemMax = 8192;    // GlobalPath: row held in shared memory below this n
                                     // (beyond it, in global scratch: LoopScratch::rowg)
constexpr int kSmallMax = 1024;      // SmemPath: supports resident in shared memory
#ifndef RBF_AUTO_CLUSTER_MAX_CARD
#define RBF_AUTO_CLUSTER_MAX_CARD 2048
#endif
constexpr int kAutoClusterMaxCard = RBF_AUTO_CLUSTER_MAX_CARD;
// (measured, tools/sel_time.py on configs[2], card 1,667: 2.5e5 -> 17.6 ms,
// 4e5 -> 17.06, 6e5 -> 16.71, 8e5 and above -> 16.68: the one-cluster appends
// (~4 us) beat the grid's (~11 us at small n) for longer than its scans lose)
#ifndef RBF_CLUSTER_SCAN_PAIRS
#define RBF_CLUSTER_SCAN_PAIRS 800000
#endif
constexpr int64_t kClusterScanPairs = RBF_CLUSTER_SCAN_PAIRS;  // per group scan, see gcb_driver
// when the MSG path's resident capacity is reached, scans of more pairs than
// this go to the grid rather than to the shared-memory cluster path
// (configs[4] m = 187: 31.0 -> 23.6 ms; tools/greedy_ab.py)
constexpr int64_t kSmemScanPairs = 150000;
constexpr int kMsgDefaultClusters = 1;         // MSG path: clusters sharing the scans
constexpr int kNone = 0x7fffffff;
#ifndef RBF_PAIR_ROWS
#define RBF_PAIR_ROWS 1
#endif
constexpr bool kPairRows = RBF_PAIR_ROWS != 0;  // GlobalPath::tri_gemv: complementary vectors per warp
// internal rbf_gcb_args.flags bits (set by rbf_gcb_run on its own copy)
constexpr int kFlagTailSweep = 1 << 16;  // one-cluster launch: stop before the final sweep,
                                         // which a whole-GPU tail launch runs
constexpr int kFlagTailOnly = 1 << 17;   // that tail launch: final sweep of a finished loop only
// one-cluster paths: after this many consecutive groups within tolerance
// (and m >= 2x it) the rest of the run is resolved by the tail launch from
// one whole-boundary pass (the weights do not change until an append)
// (configs[1] selection with 5 / 6 / 7 / 8 / 10: 2.31 / 2.24 / 2.26 / 2.27 / 2.29 ms)
#ifndef RBF_STREAK_HANDOVER
#define RBF_STREAK_HANDOVER 6
#endif
constexpr int kStreakHandover = RBF_STREAK_HANDOVER;
// MSG path: the append's refinement step (r = row - L c0, c = c0 + Li r)
// runs once the smallest pivot^2 so far (min l_i^2) drops below this; above
// it the factor is well enough conditioned that c = Li row alone keeps the
// weights within ~3e-10 of the reference's, and the append
// saves two of its dependent DSMEM hops. 0 = always refine.
#ifndef RBF_REFINE_BELOW_P2
#define RBF_REFINE_BELOW_P2 1e-7
#endif
constexpr double kRefineBelowP2 = RBF_REFINE_BELOW_P2;
constexpr int kFlagResumeOnly = 1 << 18;  // a second one-cluster launch queued behind the tail:
                                          // runs only if the state asks to resume in its shape

struct LoopScratch {
  unsigned* bar;   // grid barrier word
  int* fault;
  Best* part;      // [2 parities][ctas][2]: unrestricted, eligible-only
  double* red;     // [ctas][4]: c.c, c.y(3)
  double* err;     // [nb]   errors of the group being scanned
  double* dmin;    // [nb]   seed farthest-point distances
  double* c0;      // [cap]
  double* r;       // [cap]
  double* c1;      // [cap]
  double* gpt;     // [nb][3] boundary points in group order
  double* gdisp;   // [nb][3] displacements in group order
  double* xc;      // [2 parities][16 clusters][4]: per-cluster (err, pos) x 2
  unsigned* xseq;  // [2][16] publication sequence numbers
  double* lic;     // [cap(cap+1)/2] column-packed copy of Li (L2 paths)
  double* rowg;    // [ctas][cap] candidate rows once n >= kRowSmemMax (L2 paths; one per
                   // CTA: every CTA computes the whole row, as in shared memory below it)
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
  s.part = reinterpret_cast<Best*>(take(sizeof(Best) * 4 * ctas));
  s.red = reinterpret_cast<double*>(take(sizeof(double) * 4 * ctas));
  s.err = reinterpret_cast<double*>(take(sizeof(double) * (size_t)nb));
  s.dmin = reinterpret_cast<double*>(take(sizeof(double) * (size_t)nb));
  s.c0 = reinterpret_cast<double*>(take(sizeof(double) * (size_t)cap));
  s.r = reinterpret_cast<double*>(take(sizeof(double) * (size_t)cap));
  s.c1 = reinterpret_cast<double*>(take(sizeof(double) * (size_t)cap));
  s.gpt = reinterpret_cast<double*>(take(sizeof(double) * 3 * (size_t)nb));
  s.gdisp = reinterpret_cast<double*>(take(sizeof(double) * 3 * (size_t)nb));
  s.xc = reinterpret_cast<double*>(take(sizeof(double) * 2 * 16 * 4));
  s.xseq = reinterpret_cast<unsigned*>(take(sizeof(unsigned) * 2 * 16));
  s.lic = reinterpret_cast<double*>(take(sizeof(double) * (size_t)cap * (cap + 1) / 2));
  s.rowg = reinterpret_cast<double*>(take(cap >= kRowSmemMax ? sizeof(double) * (size_t)ctas * cap : 8));
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
      // arrive with release semantics (cumulative over the CTA's writes via
      // the __syncthreads above), spin with acquire loads; the short sleep
      // keeps 148 pollers off the barrier line (tools/gridbar_bench.cu:
      // ~2260 cycles per barrier vs ~2720 for fence + relaxed atomic)
      const unsigned add = blockIdx.x == 0 ? (0x80000000u - (gridDim.x - 1)) : 1u;
      unsigned old;
      asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(word), "r"(add) : "memory");
      uint64_t t0 = 0;
      unsigned spins = 0;
      while (((old ^ ld_acquire(word)) & 0x80000000u) == 0) {
        __nanosleep(32);
        if ((++spins & 1023u) == 0) {
          const uint64_t now = globaltimer_ns();
          if (t0 == 0) {
            t0 = now;
          } else if (now - t0 > 20ull * 1000000000ull) {
            atomicExch(fault, 1);
            __trap();
          }
        }
      }
    }
    __syncthreads();
  }
};

// CTA 0's SM clock at phase boundaries (diagnostics in rbf_gcb_state),
// kept by thread 0 of CTA 0 in shared memory.
template <bool kOn>
struct PhaseClockT {  // kOn = false compiles every mark away (the clock reads are
  double* acc;        // volatile and cost ~4 % of the loop as scheduling fences)
  long long last;
  bool on;
  __device__ __forceinline__ void start(double* smem_acc) {
    acc = smem_acc;
    on = kOn && blockIdx.x == 0 && threadIdx.x == 0;
    if (kOn && on) {
      for (int i = 0; i < 16; ++i) acc[i] = 0.0;
      last = clock64();
    }
  }
  __device__ __forceinline__ void mark(int phase) {
    if (kOn && on) {
      const long long now = clock64();
      acc[phase] += (double)(now - last);
      last = now;
    }
  }
  __device__ __forceinline__ void count(int slot) {
    if (kOn && on) acc[slot] += 1.0;
  }
};

__device__ __forceinline__ uint64_t leader_timer() {
  return (blockIdx.x == 0 && threadIdx.x == 0) ? globaltimer_ns() : 0ull;
}

// Per-CTA small shared state common to both paths.
struct Common {
  double red[kLoopWarps * 32 * 4];
  Best wb[kLoopWarps][2];
  double wred[kLoopWarps][4];
  Best bcast[2];
  double dbl[8];
  double phase[16];
};

// Fold per-warp bests; every lane of warp 0 ends with the CTA's best.
__device__ __forceinline__ Best cta_best(Common& cm, Best b, int slot) {
  b = warp_best(b);
  if ((threadIdx.x & 31) == 0) cm.wb[threadIdx.x >> 5][slot] = b;
  __syncthreads();
  Best v{-1.0, kNone};
  if (threadIdx.x < 32) {
    v = threadIdx.x < kLoopWarps ? cm.wb[threadIdx.x][slot] : Best{-1.0, kNone};
    v = warp_best(v);
  }
  return v;
}

// Warp-cooperative dot product of packed row `arow` (len entries) with x,
// every load of the lane issued before the first FMA (8 in flight per lane).
// kB loads of the row per lane are in flight before the first FMA; every
// lane accumulates its entries in increasing j whatever kB is, so the result
// does not depend on kB.
template <int kB = 8, typename XL>
__device__ __forceinline__ double row_dot(const double* arow, int len, XL xload, int lane) {
  double acc = 0.0;
  for (int j0 = 0; j0 < len; j0 += kB * kWarp) {
    double av[kB], xv[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int j = j0 + u * kWarp + lane;
      av[u] = j < len ? __ldcg(arow + j) : 0.0;
      xv[u] = j < len ? xload(j) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kB; ++u) acc = fma(av[u], xv[u], acc);
  }
  return warp_sum(acc);
}

// row_dot with x in shared memory: only the row is held in registers and x
// is read from shared memory at the FMA (row_dot buffers both in registers).
// configs[3] selection 326.7 -> 301.1 ms (the r / c / u products 10-20 %
// faster; 16 and 32 row loads in flight per lane measure the same,
// tools/sel_time.py). Same per-lane order as row_dot, so the same bits.
#ifndef RBF_SX_BATCH
#define RBF_SX_BATCH 16
#endif
template <int kB, typename XL>
__device__ __forceinline__ double row_dot_sx(const double* arow, int len, XL xs, int lane) {
  double acc = 0.0;
  for (int j0 = 0; j0 < len; j0 += kB * kWarp) {
    double av[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int j = j0 + u * kWarp + lane;
      av[u] = j < len ? __ldcg(arow + j) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int j = j0 + u * kWarp + lane;
      acc = fma(av[u], j < len ? xs(j) : 0.0, acc);
    }
  }
  return warp_sum(acc);
}

enum AppendResult { kAccepted = 0, kRejectDup = 1, kRejectPivot = 2 };

// Row phi(cdist(p, s_j) / R) of candidate p against the n supports with the
// reference's rounding (every CTA computes the full row), plus the
// near-duplicate test min_j d_j < dup (selection.py:342-345) as a block-wide
// flag.
template <typename PL>
__device__ __forceinline__ bool exact_row(Common& cm, double* row, int n, double px, double py,
                                          double pz, double radius, double dup, PL sup_xyz) {
  if (threadIdx.x == 0) cm.dbl[0] = 0.0;
  __syncthreads();
  bool near = false;
  for (int j = threadIdx.x; j < n; j += kLoopThreads) {
    double sx, sy, sz;
    sup_xyz(j, sx, sy, sz);
    const double d = cdist_exact(px, py, pz, sx, sy, sz);
    row[j] = phi_exact(d, radius);
    near |= d < dup;
  }
  if (__any_sync(0xffffffffu, near) && (threadIdx.x & 31) == 0) cm.dbl[0] = 1.0;
  __syncthreads();
  return cm.dbl[0] != 0.0;
}

// Compensated incremental weights. Every append moves the
// weights by Li[n][j] y_n; summed naively over thousands of appends the
// rounding of those updates drifts the residuals by more than the gap between
// near-tied candidates at kappa ~ 1e10 (configs[3]: the sequence left the
// reference's at support 4,125). So each weight is carried as hi + lo: the
// product's rounding error (an FMA) and the sum's (two-sum) accumulate in lo,
// and the scans read the rounded hi + lo.
__device__ __forceinline__ double comp_add(double& hi, double& lo, double a, double b) {
  const double p = __dmul_rn(a, b);
  const double pe = fma(a, b, -p);
  const double t = __dadd_rn(hi, p);
  const double bb = __dsub_rn(t, hi);
  const double e = __dadd_rn(__dsub_rn(hi, __dsub_rn(t, bb)), __dsub_rn(p, bb));
  hi = t;
  lo = __dadd_rn(lo, __dadd_rn(e, pe));
  return __dadd_rn(hi, lo);
}

// ================================================================ GlobalPath
// column j of a column-packed lower triangle with capacity cap: entries
// i = j .. cap-1 contiguous from here
__device__ __forceinline__ int64_t col_off(int64_t j, int64_t cap) { return j * cap - j * (j - 1) / 2; }

struct GlobalShared {
  Common cm;
  double sx[kSupTile], sy[kSupTile], sz[kSupTile];
  double wx[kSupTile], wy[kSupTile], wz[kSupTile];
  double row[kRowSmemMax];
  double gred[kLoopWarps];  // row products: per-warp partials of a shared row
};

template <class Team, class Clock>
struct GlobalPath {
  const rbf_gcb_args& a;
  const LoopScratch& s;
  GlobalShared& sh;
  Team team;
  double inv_r;
  Clock& pc;

  static constexpr int kMaxN = 1 << 30;  // the factor grows with the capacity (host side)
  __device__ Common& cm() { return sh.cm; }
  __device__ void sync() { team.sync(); }
  // shared-memory (err, pos) cache for the tail launch's walk over group
  // bests: the scan staging area (sx..wz), idle once a scan has been gathered
  __device__ Best* best_cache() { return reinterpret_cast<Best*>(sh.sx); }
  __device__ static constexpr int best_cache_cap() { return (int)(6 * kSupTile * sizeof(double) / sizeof(Best)); }
  // rebuild the column-packed copy of Li (rows < n) for this launch's capacity
  __device__ void begin(int n) {
    const int64_t total = (int64_t)n * (n + 1) / 2;
    const int64_t cap = a.cap;
    for (int64_t f = (int64_t)blockIdx.x * kLoopThreads + threadIdx.x; f < total;
         f += (int64_t)gridDim.x * kLoopThreads) {
      int64_t i = (int64_t)((sqrt(8.0 * (double)f + 1.0) - 1.0) * 0.5);
      while (tri_off(i + 1) <= f) ++i;
      while (tri_off(i) > f) --i;
      const int64_t j = f - tri_off(i);
      s.lic[col_off(j, cap) + (i - j)] = __ldcg(a.Li + f);
    }
  }
  __device__ int group_off(int g) { return __ldg(a.group_off + g); }

  // this CTA's partial -> global, double-buffered by parity
  __device__ void publish(Best b, int slot, int par) {
    if (threadIdx.x == 0) s.part[(par * gridDim.x + blockIdx.x) * 2 + slot] = b;
  }
  __device__ void gather(int par, int nslots) {
    team.sync();
    fold(par, nslots);
  }
  __device__ void finish() {}
  __device__ void fold(int par, int nslots) {
    const int G = gridDim.x;
    if (threadIdx.x < 32 * nslots) {
      const int slot = threadIdx.x >> 5, lane = threadIdx.x & 31;
      Best b{-1.0, kNone};
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        const int c = lane + 32 * q;
        if (c < G) {
          const Best* p = &s.part[(par * G + c) * 2 + slot];
          b = best_of(b, Best{__ldcg(&p->err), __ldcg(&p->pos)});
        }
      }
      b = warp_best(b);
      if (lane == 0) sh.cm.bcast[slot] = b;
    }
    __syncthreads();
  }

  // errors of `card` rows. The team's CTAs split the rows; a CTA takes its
  // rows in rounds. Full rounds give each of the 512 lanes one row. The last
  // round (rem < 512 rows) spreads its rows over the warps: S lanes per row
  // (the largest power of two <= 32 with rem * S <= 512), each lane
  // accumulating supports j = sub (mod S), combined by a butterfly. Each
  // row's position, eligibility and displacement are prefetched into shared
  // memory before the pair loop, so the epilogues never wait on a global
  // load. (An arbitrary S with shared-memory partials filling all 512 lanes
  // measured slower: tools/greedy_ab.py, configs[3].)
  static constexpr bool kHasOv = false;
  __device__ bool ov_fits(int, int) { return false; }
  __device__ int append_ov(int pos, int& n, bool check_dup, double* p2, int, int) {
    return append(pos, n, check_dup, p2);
  }
  __device__ void scan_ov(const int*, const double*, int, int, int) {}

  __device__ __forceinline__ void scan(const int* gpos, const double* gpt, const double* gdisp, int card,
                                       int n, int par) {
    const int tid = threadIdx.x, G = gridDim.x;
    // 32-bit division when card * G fits (Nb <= 2^31 / 148): cheaper than 64-bit in every warp
    const bool narrow = (int64_t)card * G < (1ll << 31);
    const int lo = narrow ? (int)((unsigned)(card * blockIdx.x) / (unsigned)G) : (int)((int64_t)card * blockIdx.x / G);
    const int hi = narrow ? (int)((unsigned)(card * (blockIdx.x + 1)) / (unsigned)G)
                          : (int)((int64_t)card * (blockIdx.x + 1) / G);
    const double* gx = a.sup;
    const int cap = a.cap;
    // tail-round operands in the (idle) row buffer
    double* md = sh.row;                                            // [kLoopThreads][3] displacements
    int* mpos = reinterpret_cast<int*>(sh.row + 3 * kLoopThreads);  // [kLoopThreads] pos (~pos: ineligible)
    Best bu{-1.0, kNone}, br{-1.0, kNone};
    bool staged = false;
    auto stage = [&](int s0, int cnt) {
      __syncthreads();
      for (int j = tid; j < cnt; j += kLoopThreads) {
        sh.sx[j] = __ldcg(gx + s0 + j) * inv_r;
        sh.sy[j] = __ldcg(gx + cap + s0 + j) * inv_r;
        sh.sz[j] = __ldcg(gx + 2 * cap + s0 + j) * inv_r;
        sh.wx[j] = __ldcg(gx + 3 * cap + s0 + j);
        sh.wy[j] = __ldcg(gx + 4 * cap + s0 + j);
        sh.wz[j] = __ldcg(gx + 5 * cap + s0 + j);
      }
      __syncthreads();
    };
    auto finish_row = [&](int t, int pos, bool elig, double dx, double dy, double dz, double ux, double uy,
                          double uz) {
      const double e = residual_norm(dx, dy, dz, ux, uy, uz);
      s.err[t] = e;
      if (better(e, pos, bu.err, bu.pos)) bu = Best{e, pos};
      if (elig && better(e, pos, br.err, br.pos)) br = Best{e, pos};
    };
    for (int t0 = lo; t0 < hi;) {
      const int rem = hi - t0;
      if (rem >= kLoopThreads) {  // full round: one row per lane
        const int t = t0 + tid;
        const int pos = gpos ? __ldg(gpos + t) : t;
        const double px = __ldcg(gpt + 3 * (int64_t)t) * inv_r, py = __ldcg(gpt + 3 * (int64_t)t + 1) * inv_r,
                     pz = __ldcg(gpt + 3 * (int64_t)t + 2) * inv_r;
        double ax = 0.0, ay = 0.0, az = 0.0;
        for (int s0 = 0; s0 < n; s0 += kSupTile) {
          const int cnt = min(kSupTile, n - s0);
          if (!staged || n > kSupTile) {
            stage(s0, cnt);
            staged = true;
          }
#pragma unroll 4
          for (int j = 0; j < cnt; ++j)
            pair_accum(px, py, pz, sh.sx[j], sh.sy[j], sh.sz[j], sh.wx[j], sh.wy[j], sh.wz[j], ax, ay, az);
        }
        if (t0 == lo) pc.mark(11);
        finish_row(t, pos, !__ldcg(reinterpret_cast<const unsigned char*>(a.inel) + pos),
                   __ldcg(gdisp + 3 * (int64_t)t), __ldcg(gdisp + 3 * (int64_t)t + 1),
                   __ldcg(gdisp + 3 * (int64_t)t + 2), ax, ay, az);
        t0 += kLoopThreads;
        continue;
      }
      // tail round: rem rows over the warps, kT rows per lane group
      if (rem > kLoopWarps)
        tail_round<2>(gpos, gpt, gdisp, t0, rem, n, md, mpos, staged, lo, stage, finish_row);
      else
        tail_round<1>(gpos, gpt, gdisp, t0, rem, n, md, mpos, staged, lo, stage, finish_row);
      t0 += rem;
    }
    pc.mark(13);
    publish(cta_best(sh.cm, bu, 0), 0, par);
    publish(cta_best(sh.cm, br, 1), 1, par);
    pc.mark(14);
  }

  // The last round of a scan: rem (< 512) rows, kT rows per group of S lanes
  // (S the largest power of two <= 32 with groups * S <= 512, and S <= n);
  // each lane takes supports j = sub (mod S) for its kT rows (kT = 2 doubles
  // the independent pair chains per lane once rem > 16), a butterfly combines
  // the S partials, lane sub = 0 finishes the group's rows from the operands
  // prefetched into shared memory.
  template <int kT, class Stage, class FinishRow>
  __device__ __forceinline__ void tail_round(const int* gpos, const double* gpt, const double* gdisp, int t0,
                                             int rem, int n, double* md, int* mpos, bool& staged, int lo,
                                             Stage& stage, FinishRow& finish_row) {
    const int tid = threadIdx.x;
    const int groups = (rem + kT - 1) / kT;
    int lg = 5;  // S = 2^lg lanes per group: shifts and masks, no divisions
    while (lg > 0 && (groups << lg) > kLoopThreads) --lg;
    while (lg > 0 && (1 << (lg - 1)) >= n) --lg;
    const int S = 1 << lg;
    const int g = tid >> lg, sub = tid & (S - 1);
    const bool active = g < groups;
    // row tid's epilogue operands: position and displacement are requested
    // here, together with the rows' points and (below) the first support
    // tile, so the three arrive in one L2 round trip; the eligibility byte
    // (addressed by the position) follows and is not needed before the
    // epilogue
    int my_pos = 0;
    double d0 = 0.0, d1 = 0.0, d2 = 0.0;
    if (tid < rem) {
      const int tt = t0 + tid;
      my_pos = gpos ? __ldg(gpos + tt) : tt;
      d0 = __ldcg(gdisp + 3 * (int64_t)tt);
      d1 = __ldcg(gdisp + 3 * (int64_t)tt + 1);
      d2 = __ldcg(gdisp + 3 * (int64_t)tt + 2);
    }
    double px[kT], py[kT], pz[kT], ax[kT], ay[kT], az[kT];
#pragma unroll
    for (int q = 0; q < kT; ++q) {
      const int r = kT * g + q;
      const bool ok = active && r < rem;
      const int t = t0 + r;
      px[q] = ok ? __ldcg(gpt + 3 * (int64_t)t) * inv_r : 0.0;
      py[q] = ok ? __ldcg(gpt + 3 * (int64_t)t + 1) * inv_r : 0.0;
      pz[q] = ok ? __ldcg(gpt + 3 * (int64_t)t + 2) * inv_r : 0.0;
      ax[q] = ay[q] = az[q] = 0.0;
    }
    bool first_staged = false;
    if (n > 0 && (!staged || n > kSupTile)) {
      stage(0, min(kSupTile, n));
      staged = true;
      first_staged = true;
    }
    if (tid < rem) {
      const bool elig = !__ldcg(reinterpret_cast<const unsigned char*>(a.inel) + my_pos);
      mpos[tid] = elig ? my_pos : ~my_pos;
      md[3 * tid] = d0;
      md[3 * tid + 1] = d1;
      md[3 * tid + 2] = d2;
    }
    for (int s0 = 0; s0 < n; s0 += kSupTile) {
      const int cnt = min(kSupTile, n - s0);
      if (!(s0 == 0 && first_staged) && (!staged || n > kSupTile)) {
        stage(s0, cnt);
        staged = true;
      }
      if (active) {
#pragma unroll 4
        for (int j = sub; j < cnt; j += S) {
          const double sx = sh.sx[j], sy = sh.sy[j], sz = sh.sz[j];
          const double wx = sh.wx[j], wy = sh.wy[j], wz = sh.wz[j];
#pragma unroll
          for (int q = 0; q < kT; ++q) pair_accum(px[q], py[q], pz[q], sx, sy, sz, wx, wy, wz, ax[q], ay[q], az[q]);
        }
      }
    }
    if (t0 == lo) pc.mark(11);
#pragma unroll
    for (int q = 0; q < kT; ++q) {
      for (int off = S >> 1; off > 0; off >>= 1) {
        ax[q] += __shfl_xor_sync(0xffffffffu, ax[q], off);
        ay[q] += __shfl_xor_sync(0xffffffffu, ay[q], off);
        az[q] += __shfl_xor_sync(0xffffffffu, az[q], off);
      }
    }
    __syncthreads();  // prefetched operands visible
    if (active && sub == 0) {
#pragma unroll
      for (int q = 0; q < kT; ++q) {
        const int r = kT * g + q;
        if (r >= rem) continue;
        const int mp = mpos[r];
        const bool elig = mp >= 0;
        finish_row(t0 + r, elig ? mp : ~mp, elig, md[3 * r], md[3 * r + 1], md[3 * r + 2], ax[q], ay[q], az[q]);
      }
    }
    __syncthreads();
  }

  // Products with the n vectors of a packed triangle: rows of a row-packed
  // triangle (vector i, length i + 1) or, with kCols, columns of the
  // column-packed copy (vector j = rows j..n-1, x index j + e); one warp per
  // vector, vectors strided over every warp of the team, 16 loads per lane
  // in flight once the factor is long. finish(v, sum) runs on lane 0.
  // pre(v) -> POD: the finishing lane's operands of vector v, loaded
  // before the dot product so their L2 latency overlaps it
  template <bool kCols, class XL, class Pre, class Fin>
  __device__ __forceinline__ void tri_gemv(const double* A, int n, XL xload, Pre pre, Fin finish,
                                           bool x_smem = false) {
    const int lane = threadIdx.x & 31;
    const int G = gridDim.x;
    const int64_t cap = a.cap;
    // short factors: several warps of one CTA share a row (wpr warps per
    // row, the largest power of two that still gives every row a group in
    // one round), their partial sums added in warp order through shared
    // memory -- fewer dependent load batches per row when rows are few
    int wpr = 1;
    while (wpr < kLoopWarps && (int64_t)(kLoopWarps / (2 * wpr)) * G >= n) wpr *= 2;
    if (wpr > 1) {
      const int warp = threadIdx.x >> 5, grp = warp / wpr, sub = warp % wpr;
      const int v = grp * G + (int)blockIdx.x;  // rows interleaved over the CTAs
      double acc = 0.0;
      decltype(pre(0)) pf{};
      if (v < n && sub == 0 && lane == 0) pf = pre(v);
      if (v < n) {
        const double* av = A + (kCols ? col_off(v, cap) : tri_off(v));
        const int len = kCols ? n - v : v + 1;
        const int stride = wpr * kWarp;
        for (int j0 = sub * kWarp; j0 < len; j0 += 8 * stride) {
          double aa[8], xx[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int j = j0 + u * stride + lane;
            aa[u] = j < len ? __ldcg(av + j) : 0.0;
            xx[u] = j < len ? xload(v, j) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) acc = fma(aa[u], xx[u], acc);
        }
      }
      acc = warp_sum(acc);
      if (lane == 0) sh.gred[warp] = acc;
      __syncthreads();
      if (v < n && sub == 0 && lane == 0) {
        double t = sh.gred[grp * wpr];
        for (int h = 1; h < wpr; ++h) t += sh.gred[grp * wpr + h];
        finish(v, t, pf);
      }
      __syncthreads();
      return;
    }
    const int gw = blockIdx.x * kLoopWarps + (threadIdx.x >> 5), nw = G * kLoopWarps;
    auto one = [&](int v) {
      const double* av = A + (kCols ? col_off(v, cap) : tri_off(v));
      const int len = kCols ? n - v : v + 1;
      auto xl = [&](int e) { return xload(v, e); };
      decltype(pre(0)) pf{};
      if (lane == 0) pf = pre(v);
      const double acc = x_smem ? row_dot_sx<RBF_SX_BATCH>(av, len, xl, lane)
                                : len > 1024 ? row_dot<16>(av, len, xl, lane) : row_dot<8>(av, len, xl, lane);
      if (lane == 0) finish(v, acc, pf);
    };
    // More vectors than warps: a warp takes vectors p and n-1-p (n+1 entries
    // together), so every warp streams the same amount -- with v, v + nw
    // (the lengths of a triangle's vectors grow with v) the heaviest warps
    // read ~1.5x the mean and every product waits for them. One call site of
    // the dot product (a second one spills the loop kernel's registers).
    const bool pair = kPairRows && n > nw;
    const int lim = pair ? (n + 1) >> 1 : n;
    for (int p = gw, k = 0; p < lim;) {
      const int v = k ? n - 1 - p : p;
      if (!k || v != p) one(v);
      if (pair && !k) {
        k = 1;
      } else {
        k = 0;
        p += nw;
      }
    }
  }

  // x (n doubles) into shared memory (the scan's staging area is idle
  // during an append) once it is long enough for the copy to pay
  __device__ __forceinline__ const double* stage_x(const double* x, int n) {
    if (n <= 1024 || n > kRowSmemMax) return nullptr;
    double* xs = sh.sx;  // sx..wz: 6 * kSupTile contiguous doubles >= kRowSmemMax
    for (int j = threadIdx.x; j < n; j += kLoopThreads) xs[j] = __ldcg(x + j);
    __syncthreads();
    return xs;
  }

  __device__ int append(int pos, int& n, bool check_dup, double* pivot2_out) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x;
    const int cap = a.cap;
    const double px = __ldg(a.points + 3 * (int64_t)pos), py = __ldg(a.points + 3 * (int64_t)pos + 1),
                 pz = __ldg(a.points + 3 * (int64_t)pos + 2);
    double* row = n < kRowSmemMax ? sh.row : s.rowg + (int64_t)blockIdx.x * cap;
    const bool near = exact_row(sh.cm, row, n, px, py, pz, a.radius, a.dup_dist, [&](int j, double& x, double& y, double& z) {
      x = __ldcg(a.sup + j);
      y = __ldcg(a.sup + cap + j);
      z = __ldcg(a.sup + 2 * (int64_t)cap + j);
    });
    if (check_dup && n > 0 && near) return kRejectDup;
    pc.mark(1);
    // c0 = Li row
    auto no_pre = [](int) { return make_double4(0.0, 0.0, 0.0, 0.0); };
    tri_gemv<false>(a.Li, n, [&](int, int e) { return row[e]; }, no_pre,
                    [&](int v, double acc, const double4&) { s.c0[v] = acc; }, n < kRowSmemMax);
    team.sync();
    pc.mark(2);
    // r = row - L c0
    const double* xs = stage_x(s.c0, n);
    tri_gemv<false>(a.L, n, [&](int, int e) { return xs ? xs[e] : __ldcg(s.c0 + e); },
                    no_pre,
                    [&](int v, double acc, const double4&) { s.r[v] = row[v] - acc; }, xs != nullptr);
    team.sync();
    pc.mark(3);
    // c = c0 + Li r, with this CTA's partials of c.c and c.y
    double pcc = 0.0, pcy0 = 0.0, pcy1 = 0.0, pcy2 = 0.0;
    __syncthreads();
    xs = stage_x(s.r, n);
    tri_gemv<false>(
        a.Li, n, [&](int, int e) { return xs ? xs[e] : __ldcg(s.r + e); },
        [&](int v) {
          return make_double4(__ldcg(s.c0 + v), __ldcg(a.y + 3 * (int64_t)v), __ldcg(a.y + 3 * (int64_t)v + 1),
                              __ldcg(a.y + 3 * (int64_t)v + 2));
        },
        [&](int v, double acc, const double4& pf) {
          const double c = pf.x + acc;
          s.c1[v] = c;
          pcc = fma(c, c, pcc);
          pcy0 = fma(c, pf.y, pcy0);
          pcy1 = fma(c, pf.z, pcy1);
          pcy2 = fma(c, pf.w, pcy2);
        },
        xs != nullptr);
    Common& cm = sh.cm;
    if (lane == 0) {
      cm.wred[warp][0] = pcc;
      cm.wred[warp][1] = pcy0;
      cm.wred[warp][2] = pcy1;
      cm.wred[warp][3] = pcy2;
    }
    __syncthreads();
    if (tid < 4) {
      double t = 0.0;
      for (int w = 0; w < kLoopWarps; ++w) t += cm.wred[w][tid];
      s.red[4 * blockIdx.x + tid] = t;
    }
    team.sync();
    pc.mark(4);
    if (tid < 128) {  // every CTA folds the G partials with the same tree
      const int q = tid >> 5, ln = tid & 31;
      double t = 0.0;
#pragma unroll
      for (int u = 0; u < 5; ++u) {
        const int c = ln + 32 * u;
        if (c < G) t += __ldcg(s.red + 4 * c + q);
      }
      t = warp_sum(t);
      if (ln == 0) cm.dbl[1 + q] = t;
    }
    __syncthreads();
    const double pivot2 = 1.0 - cm.dbl[1];  // row[n] = phi(0) = 1 exactly
    *pivot2_out = pivot2;
    if (!(pivot2 > 0.0)) {
      __syncthreads();
      return kRejectPivot;
    }
    const double l = sqrt(pivot2);
    const double inv_l = 1.0 / l;  // one division; every later 1/l is a multiply
    const double yn0 = (__ldg(a.disp + 3 * (int64_t)pos) - cm.dbl[2]) * inv_l;
    const double yn1 = (__ldg(a.disp + 3 * (int64_t)pos + 1) - cm.dbl[3]) * inv_l;
    const double yn2 = (__ldg(a.disp + 3 * (int64_t)pos + 2) - cm.dbl[4]) * inv_l;
    double* Lrow = a.L + tri_off(n);
    double* Lirow = a.Li + tri_off(n);
    double* wgt = a.sup + 3 * (int64_t)cap;
    // u = Li^T c over the column copy; Li[n][j] = -u_j / l, and the weights
    // move by Li[n][j] y_n (w = Li^T y with the new row appended)
    const int nn = n;
    xs = stage_x(s.c1, n);
    double* whi = a.sup + 6 * (int64_t)cap;  // compensated weights: hi (3 rows), lo (3 rows)
    double* wlo = a.sup + 9 * (int64_t)cap;
    struct Pf7 {
      double c, h[3], l[3];
    };
    tri_gemv<true>(
        s.lic, n, [&](int v, int e) { return xs ? xs[v + e] : __ldcg(s.c1 + v + e); },
        [&](int j) {
          Pf7 q;
          q.c = __ldcg(s.c1 + j);
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            q.h[k] = __ldcg(whi + k * (int64_t)cap + j);
            q.l[k] = __ldcg(wlo + k * (int64_t)cap + j);
          }
          return q;
        },
        [&](int j, double u, const Pf7& pf) {
          const double lij = -u * inv_l;
          Lirow[j] = lij;
          s.lic[col_off(j, cap) + (nn - j)] = lij;
          Lrow[j] = pf.c;
          const double yn[3] = {yn0, yn1, yn2};
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            double h = pf.h[k], lo = pf.l[k];
            wgt[k * (int64_t)cap + j] = comp_add(h, lo, lij, yn[k]);
            whi[k * (int64_t)cap + j] = h;
            wlo[k * (int64_t)cap + j] = lo;
          }
        },
        xs != nullptr);
    if (blockIdx.x == 0 && tid == 0) {
      Lirow[n] = inv_l;
      s.lic[col_off(n, cap)] = inv_l;
      Lrow[n] = l;
      a.y[3 * (int64_t)n] = yn0;
      a.y[3 * (int64_t)n + 1] = yn1;
      a.y[3 * (int64_t)n + 2] = yn2;
      a.sup[n] = px;
      a.sup[cap + n] = py;
      a.sup[2 * cap + n] = pz;
      wgt[n] = whi[n] = yn0 * inv_l;
      wgt[cap + n] = whi[cap + n] = yn1 * inv_l;
      wgt[2 * cap + n] = whi[2 * cap + n] = yn2 * inv_l;
      wlo[n] = wlo[cap + n] = wlo[2 * cap + n] = 0.0;
      a.sel[n] = pos;
    }
    if (tid == 0) a.inel[pos] = 1;
    n += 1;
    team.sync();
    pc.mark(5);
    return kAccepted;
  }
};

// ================================================================= SmemPath
constexpr int kGoffSmem = 4096;  // group offsets cached in shared memory

struct SmemShared {
  Common cm;
  double ux[kSmallMax], uy[kSmallMax], uz[kSmallMax];  // support coordinates
  double sx[kSmallMax], sy[kSmallMax], sz[kSmallMax];  // ... scaled by 1/R
  double wx[kSmallMax], wy[kSmallMax], wz[kSmallMax];  // weights
  double y0[kSmallMax], y1[kSmallMax], y2[kSmallMax];  // forward-substituted d
  double row[kSmallMax], c0[kSmallMax], r[kSmallMax], c1[kSmallMax];
  double colp[kSmallMax][4];      // this CTA's column partials of Li^T [c, y]
  double acc[kLoopWarps][4][4];   // scan: per-warp reduced sums (4 targets x 3 comps)
  int goff[kGoffSmem + 1];
  Best part[2][kClusterCTAs][2];  // scan partials, written by every CTA (DSMEM)
  double rpart[kClusterCTAs][4];  // c.c, c.y partials (DSMEM)
};

// Reduce-scatter butterfly over a full warp: v[16] per lane -> each value
// summed over the 32 lanes with 16 shuffled doubles per lane (instead of 80
// for independent xor trees). Returns the sum of value index `idx` (set on
// return); lanes l and l^1 hold the same index.
__device__ __forceinline__ double warp_reduce_scatter16(double (&v)[16], int lane, int& idx) {
  int base = 0;
#pragma unroll
  for (int lev = 0; lev < 4; ++lev) {
    const int off = 16 >> lev, half = 8 >> lev;
    const bool hi = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double send = hi ? v[i] : v[i + half];
      const double keep = hi ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
    if (hi) base += half;
  }
  idx = base;
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// Both arg-max partials of a CTA in one pass; every lane of warp 0 ends with
// them. `lanes` = how many low lanes of each warp hold candidates (1..32).
__device__ __forceinline__ void cta_best2(Common& cm, Best& bu, Best& br, int lanes) {
  if (lanes > 4) {  // lanes past `lanes` hold the neutral record: fold the whole warp (3 redux each)
    bu = warp_best(bu);
    br = warp_best(br);
  } else {
    for (int off = 1; off < lanes; off <<= 1) {
      const double eu = __shfl_xor_sync(0xffffffffu, bu.err, off);
      const int pu = __shfl_xor_sync(0xffffffffu, bu.pos, off);
      const double er = __shfl_xor_sync(0xffffffffu, br.err, off);
      const int pr = __shfl_xor_sync(0xffffffffu, br.pos, off);
      if (better(eu, pu, bu.err, bu.pos)) bu = Best{eu, pu};
      if (better(er, pr, br.err, br.pos)) br = Best{er, pr};
    }
  }
  if ((threadIdx.x & 31) == 0) {
    cm.wb[threadIdx.x >> 5][0] = bu;
    cm.wb[threadIdx.x >> 5][1] = br;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int l = threadIdx.x;
    bu = warp_best(l < kLoopWarps ? cm.wb[l][0] : Best{-1.0, kNone});
    br = warp_best(l < kLoopWarps ? cm.wb[l][1] : Best{-1.0, kNone});
  }
}

// Dot products of two packed rows (a: len_a entries, b: len_b) with x, the
// two rows' elements dealt over the lanes as one list so that a short and a
// long row together cost about one batch of loads.
template <typename XL>
__device__ __forceinline__ void row_dot_pair(const double* ra, int len_a, const double* rb, int len_b,
                                             XL xload, int lane, double& sa, double& sb) {
  constexpr int U = 12;
  const int total = len_a + len_b;
  double acc_a = 0.0, acc_b = 0.0;
  for (int e0 = 0; e0 < total; e0 += U * kWarp) {
    double av[U], xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * kWarp + lane;
      const bool in_a = e < len_a;
      const int j = in_a ? e : e - len_a;
      const bool ok = e < total;
      av[u] = ok ? __ldcg((in_a ? ra : rb) + j) : 0.0;
      xv[u] = ok ? xload(j) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * kWarp + lane;
      if (e < len_a)
        acc_a = fma(av[u], xv[u], acc_a);
      else
        acc_b = fma(av[u], xv[u], acc_b);
    }
  }
  sa = warp_sum(acc_a);
  sb = warp_sum(acc_b);
}

template <class Clock>
struct SmemPath {
  const rbf_gcb_args& a;
  const LoopScratch& s;
  SmemShared& sh;
  double inv_r;
  Clock& pc;

  static constexpr int kMaxN = kSmallMax;
  __device__ Best* best_cache() { return nullptr; }  // (the tail launch is a GlobalPath)
  __device__ static constexpr int best_cache_cap() { return 0; }
  static constexpr int kTPT = 4;  // targets per lane in group scans
  __device__ Common& cm() { return sh.cm; }
  __device__ void sync() { cg::this_cluster().sync(); }

  // pointer to the same shared-memory object in CTA `rank` of the cluster
  template <typename T>
  __device__ __forceinline__ T* at(T* p, int rank) {
    return cg::this_cluster().map_shared_rank(p, rank);
  }

  // load the resident copies from the global state (every launch)
  __device__ void begin(int n) {
    const int cap = a.cap;
    for (int j = threadIdx.x; j < n; j += kLoopThreads) {
      const double x = __ldcg(a.sup + j), y = __ldcg(a.sup + cap + j), z = __ldcg(a.sup + 2 * cap + j);
      sh.ux[j] = x;
      sh.uy[j] = y;
      sh.uz[j] = z;
      sh.sx[j] = x * inv_r;
      sh.sy[j] = y * inv_r;
      sh.sz[j] = z * inv_r;
      sh.wx[j] = __ldcg(a.sup + 3 * cap + j);
      sh.wy[j] = __ldcg(a.sup + 4 * cap + j);
      sh.wz[j] = __ldcg(a.sup + 5 * cap + j);
      sh.y0[j] = __ldcg(a.y + 3 * j);
      sh.y1[j] = __ldcg(a.y + 3 * j + 1);
      sh.y2[j] = __ldcg(a.y + 3 * j + 2);
    }
    for (int g = threadIdx.x; g <= a.m && g <= kGoffSmem; g += kLoopThreads) sh.goff[g] = __ldg(a.group_off + g);
    __syncthreads();
  }
  __device__ int group_off(int g) { return a.m <= kGoffSmem ? sh.goff[g] : __ldg(a.group_off + g); }

  // lanes 0..15 of warp 0 (which all hold b) store it into every CTA's slot
  __device__ void publish(Best b, int slot, int par) {
    if (threadIdx.x < kClusterCTAs) *at(&sh.part[par][blockIdx.x][slot], (int)threadIdx.x) = b;
  }
  __device__ void gather(int par, int nslots) {
    sync();
    fold(par, nslots);
  }
  __device__ void finish() {}
  __device__ void fold(int par, int nslots) {
    if (threadIdx.x < 32 * nslots) {
      const int slot = threadIdx.x >> 5, lane = threadIdx.x & 31;
      Best b = lane < kClusterCTAs ? sh.part[par][lane][slot] : Best{-1.0, kNone};
      b = warp_best(b);
      if (lane == 0) sh.cm.bcast[slot] = b;
    }
    __syncthreads();
  }

  static constexpr bool kHasOv = false;
  __device__ bool ov_fits(int, int) { return false; }
  __device__ int append_ov(int pos, int& n, bool check_dup, double* p2, int, int) {
    return append(pos, n, check_dup, p2);
  }
  __device__ void scan_ov(const int*, const double*, int, int, int) {}

  __device__ __forceinline__ void scan(const int* gpos, const double* gpt, const double* gdisp, int card, int n,
                       int par) {
    const int tid = threadIdx.x, lane = tid & 31;
    const int lo = (int)(((unsigned)card * blockIdx.x) >> 4);  // kClusterCTAs = 16
    const int hi = (int)(((unsigned)card * (blockIdx.x + 1)) >> 4);
    const int tgroups = (hi - lo + kTPT - 1) / kTPT;
    int lg = 5;  // S = 2^lg lanes per target group: shifts and masks only
    while (lg > 0 && (tgroups << lg) > kLoopThreads) --lg;
    const int S = 1 << lg;
    const int per_round = kLoopThreads >> lg;
    const int rounds = (tgroups + per_round - 1) >> (9 - lg);  // kLoopThreads = 2^9
    const int sub = tid & (S - 1);
    Best bu{-1.0, kNone}, br{-1.0, kNone};
    for (int rd = 0; rd < rounds; ++rd) {
      const int tg = rd * per_round + (tid >> lg);
      double px[kTPT], py[kTPT], pz[kTPT];
      double v[16];
#pragma unroll
      for (int q = 0; q < kTPT; ++q) {
        const int t = lo + kTPT * tg + q;
        const bool ok = tg < tgroups && t < hi;
        px[q] = ok ? __ldcg(gpt + 3 * (int64_t)t) * inv_r : 0.0;
        py[q] = ok ? __ldcg(gpt + 3 * (int64_t)t + 1) * inv_r : 0.0;
        pz[q] = ok ? __ldcg(gpt + 3 * (int64_t)t + 2) * inv_r : 0.0;
        v[4 * q] = v[4 * q + 1] = v[4 * q + 2] = v[4 * q + 3] = 0.0;
      }
      // the lane that finishes target q (lane q of the group when S == 32,
      // else sub == 0) prefetches its position, eligibility and displacement
      const int myq = S == 32 ? lane : 0;
      const int my_t = lo + kTPT * tg + myq;
      const bool mine = (S == 32 ? lane < kTPT : sub == 0) && tg < tgroups && my_t < hi;
      int my_pos = -1;
      bool my_elig = false;
      double dx = 0.0, dy = 0.0, dz = 0.0;
      if (mine && S == 32) {
        my_pos = gpos ? __ldg(gpos + my_t) : my_t;
        my_elig = !__ldcg(reinterpret_cast<const unsigned char*>(a.inel) + my_pos);
        dx = __ldcg(gdisp + 3 * (int64_t)my_t);
        dy = __ldcg(gdisp + 3 * (int64_t)my_t + 1);
        dz = __ldcg(gdisp + 3 * (int64_t)my_t + 2);
      }
      if (tg < tgroups) {
#pragma unroll 1
        for (int j = sub; j < n; j += S) {
          const double sx = sh.sx[j], sy = sh.sy[j], sz = sh.sz[j];
          const double wx = sh.wx[j], wy = sh.wy[j], wz = sh.wz[j];
#pragma unroll
          for (int q = 0; q < kTPT; ++q)
            pair_accum(px[q], py[q], pz[q], sx, sy, sz, wx, wy, wz, v[4 * q], v[4 * q + 1], v[4 * q + 2]);
        }
      }
      if (rd == 0) pc.mark(11);
      if (S == 32) {
        // one target group per warp: reduce-scatter, then lane q finishes target q
        int idx;
        const double tot = warp_reduce_scatter16(v, lane, idx);
        const int w = tid >> 5;
        if ((lane & 1) == 0 && (idx & 3) != 3) sh.acc[w][idx >> 2][idx & 3] = tot;
        __syncwarp();
        if (rd == 0) pc.mark(12);
        if (mine) {
          const double e = residual_norm(dx, dy, dz, sh.acc[w][lane][0], sh.acc[w][lane][1],
                                         sh.acc[w][lane][2]);
          s.err[my_t] = e;
          bu = Best{e, my_pos};
          if (my_elig) br = Best{e, my_pos};
        }
        __syncwarp();
      } else {
#pragma unroll
        for (int q = 0; q < kTPT; ++q) {
          for (int off = S >> 1; off > 0; off >>= 1) {
            v[4 * q] += __shfl_xor_sync(0xffffffffu, v[4 * q], off);
            v[4 * q + 1] += __shfl_xor_sync(0xffffffffu, v[4 * q + 1], off);
            v[4 * q + 2] += __shfl_xor_sync(0xffffffffu, v[4 * q + 2], off);
          }
        }
        if (rd == 0) pc.mark(12);
        if (sub == 0 && tg < tgroups) {
#pragma unroll
          for (int q = 0; q < kTPT; ++q) {
            const int t = lo + kTPT * tg + q;
            if (t >= hi) continue;
            const int pos = gpos ? __ldg(gpos + t) : t;
            const double e = residual_norm(__ldcg(gdisp + 3 * (int64_t)t), __ldcg(gdisp + 3 * (int64_t)t + 1),
                                           __ldcg(gdisp + 3 * (int64_t)t + 2), v[4 * q], v[4 * q + 1],
                                           v[4 * q + 2]);
            s.err[t] = e;
            if (better(e, pos, bu.err, bu.pos)) bu = Best{e, pos};
            if (!__ldcg(reinterpret_cast<const unsigned char*>(a.inel) + pos) && better(e, pos, br.err, br.pos))
              br = Best{e, pos};
          }
        }
      }
      if (rd == 0) pc.mark(13);
    }
    cta_best2(sh.cm, bu, br, S == 32 ? kTPT : 32);
    if (tid < 32) {
      publish(bu, 0, par);
      publish(br, 1, par);
    }
    pc.mark(14);
  }

  __device__ int append(int pos, int& n, bool check_dup, double* pivot2_out) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rank = blockIdx.x;
    const int cap = a.cap;
    const double px = __ldg(a.points + 3 * (int64_t)pos), py = __ldg(a.points + 3 * (int64_t)pos + 1),
                 pz = __ldg(a.points + 3 * (int64_t)pos + 2);
    const bool near = exact_row(sh.cm, sh.row, n, px, py, pz, a.radius, a.dup_dist,
                                  [&](int j, double& x, double& y, double& z) {
                                    x = sh.ux[j];
                                    y = sh.uy[j];
                                    z = sh.uz[j];
                                  });
    if (check_dup && n > 0 && near) return kRejectDup;
    pc.mark(1);
    // rows are dealt in pairs (p, n-1-p) so every warp carries about n+1
    // elements; pair p lives on CTA p % 16, warp (p / 16) % 16
    const int npairs = (n + 1) / 2;
    auto for_my_pairs = [&](auto&& body) {
      for (int p = rank + kClusterCTAs * warp; p < npairs; p += kClusterCTAs * kLoopWarps) {
        const int ia = p, ib = n - 1 - p;
        body(ia, ib == ia ? -1 : ib);
      }
    };
    // c0 = Li row
    for_my_pairs([&](int ia, int ib) {
      double va, vb;
      row_dot_pair(a.Li + tri_off(ia), ia + 1, a.Li + tri_off(ib < 0 ? 0 : ib), ib < 0 ? 0 : ib + 1,
                   [&](int j) { return sh.row[j]; }, lane, va, vb);
      if (lane < kClusterCTAs) {
        *at(&sh.c0[ia], lane) = va;
        if (ib >= 0) *at(&sh.c0[ib], lane) = vb;
      }
    });
    sync();
    pc.mark(2);
    for_my_pairs([&](int ia, int ib) {  // r = row - L c0
      double va, vb;
      row_dot_pair(a.L + tri_off(ia), ia + 1, a.L + tri_off(ib < 0 ? 0 : ib), ib < 0 ? 0 : ib + 1,
                   [&](int j) { return sh.c0[j]; }, lane, va, vb);
      if (lane < kClusterCTAs) {
        *at(&sh.r[ia], lane) = sh.row[ia] - va;
        if (ib >= 0) *at(&sh.r[ib], lane) = sh.row[ib] - vb;
      }
    });
    sync();
    pc.mark(3);
    double pcc = 0.0, pcy0 = 0.0, pcy1 = 0.0, pcy2 = 0.0;
    for_my_pairs([&](int ia, int ib) {  // c = c0 + Li r
      double va, vb;
      row_dot_pair(a.Li + tri_off(ia), ia + 1, a.Li + tri_off(ib < 0 ? 0 : ib), ib < 0 ? 0 : ib + 1,
                   [&](int j) { return sh.r[j]; }, lane, va, vb);
      const double ca = sh.c0[ia] + va;
      if (lane < kClusterCTAs) *at(&sh.c1[ia], lane) = ca;
      if (lane == 0) {
        a.L[tri_off(n) + ia] = ca;  // row n of L (global)
        pcc = fma(ca, ca, pcc);
        pcy0 = fma(ca, sh.y0[ia], pcy0);
        pcy1 = fma(ca, sh.y1[ia], pcy1);
        pcy2 = fma(ca, sh.y2[ia], pcy2);
      }
      if (ib >= 0) {
        const double cb = sh.c0[ib] + vb;
        if (lane < kClusterCTAs) *at(&sh.c1[ib], lane) = cb;
        if (lane == 0) {
          a.L[tri_off(n) + ib] = cb;
          pcc = fma(cb, cb, pcc);
          pcy0 = fma(cb, sh.y0[ib], pcy0);
          pcy1 = fma(cb, sh.y1[ib], pcy1);
          pcy2 = fma(cb, sh.y2[ib], pcy2);
        }
      }
    });
    Common& cm = sh.cm;
    if (lane == 0) {
      cm.wred[warp][0] = pcc;
      cm.wred[warp][1] = pcy0;
      cm.wred[warp][2] = pcy1;
      cm.wred[warp][3] = pcy2;
    }
    __syncthreads();
    if (tid < 4) {
      double t = 0.0;
      for (int w = 0; w < kLoopWarps; ++w) t += cm.wred[w][tid];
      for (int c = 0; c < kClusterCTAs; ++c) *at(&sh.rpart[rank][tid], c) = t;
    }
    sync();
    pc.mark(4);
    if (tid < 4) {  // fixed-order fold of the 16 CTA partials
      double t = 0.0;
      for (int c = 0; c < kClusterCTAs; ++c) t += sh.rpart[c][tid];
      cm.dbl[1 + tid] = t;
    }
    __syncthreads();
    const double pivot2 = 1.0 - cm.dbl[1];  // row[n] = phi(0) = 1 exactly
    *pivot2_out = pivot2;
    if (!(pivot2 > 0.0)) {
      __syncthreads();
      return kRejectPivot;
    }
    const double l = sqrt(pivot2);
    const double inv_l = 1.0 / l;  // one division; every later 1/l is a multiply
    const double yn0 = (__ldg(a.disp + 3 * (int64_t)pos) - cm.dbl[2]) * inv_l;
    const double yn1 = (__ldg(a.disp + 3 * (int64_t)pos + 1) - cm.dbl[3]) * inv_l;
    const double yn2 = (__ldg(a.disp + 3 * (int64_t)pos + 2) - cm.dbl[4]) * inv_l;
    // column partials of u = Li^T c, v = Li^T y over this CTA's own rows:
    // warp w owns 32-column chunks J = w, w + 16, ...; every load of a chunk
    // is issued before its FMAs
    const int nchunks = (n + 31) / 32;
    for (int J = warp; J < nchunks; J += kLoopWarps) {
      const int j = 32 * J + lane;
      double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
      for (int p0 = rank; p0 < npairs; p0 += 8 * kClusterCTAs) {
        double av[16];
        int iv[16];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int p = p0 + u * kClusterCTAs;
          const int ia = p < npairs ? p : -1;
          const int ib = (p < npairs && n - 1 - p != p) ? n - 1 - p : -1;
          iv[2 * u] = ia;
          iv[2 * u + 1] = ib;
          av[2 * u] = (ia >= 0 && j <= ia) ? __ldcg(a.Li + tri_off(ia) + j) : 0.0;
          av[2 * u + 1] = (ib >= 0 && j <= ib) ? __ldcg(a.Li + tri_off(ib) + j) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int i = iv[u];
          if (i >= 0 && j <= i) {
            acc0 = fma(av[u], sh.c1[i], acc0);
            acc1 = fma(av[u], sh.y0[i], acc1);
            acc2 = fma(av[u], sh.y1[i], acc2);
            acc3 = fma(av[u], sh.y2[i], acc3);
          }
        }
      }
      if (j < n) {
        sh.colp[j][0] = acc0;
        sh.colp[j][1] = acc1;
        sh.colp[j][2] = acc2;
        sh.colp[j][3] = acc3;
      }
    }
    sync();
    pc.mark(15);
    // CTA `rank` folds columns [jlo, jhi) over the 16 CTAs in fixed order
    const int per = (n + kClusterCTAs - 1) / kClusterCTAs;
    const int jlo = rank * per, jhi = min(n, jlo + per);
    for (int e = tid; e < (jhi - jlo) * 4; e += kLoopThreads) {
      const int j = jlo + (e >> 2), c = e & 3;
      double part[kClusterCTAs];
#pragma unroll
      for (int q = 0; q < kClusterCTAs; ++q) part[q] = *at(&sh.colp[j][c], q);
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < kClusterCTAs; ++q) t += part[q];
      cm.red[e] = t;
    }
    __syncthreads();
    double* Lirow = a.Li + tri_off(n);
    double* wgt = a.sup + 3 * (int64_t)cap;
    for (int e = tid; e < (jhi - jlo) * kClusterCTAs; e += kLoopThreads) {
      const int jj = e / kClusterCTAs, q = e % kClusterCTAs, j = jlo + jj;
      const double lij = -cm.red[4 * jj] * inv_l;
      const double w0 = fma(lij, yn0, cm.red[4 * jj + 1]);
      const double w1 = fma(lij, yn1, cm.red[4 * jj + 2]);
      const double w2 = fma(lij, yn2, cm.red[4 * jj + 3]);
      *at(&sh.wx[j], q) = w0;
      *at(&sh.wy[j], q) = w1;
      *at(&sh.wz[j], q) = w2;
      if (q == 0) {  // fresh weights (Li^T y): hi = w, lo = 0 for the compensated paths
        Lirow[j] = lij;
        wgt[j] = wgt[3 * cap + j] = w0;  // (wgt = sup row 3: rows 6-8 hi, 9-11 lo)
        wgt[cap + j] = wgt[4 * cap + j] = w1;
        wgt[2 * cap + j] = wgt[5 * cap + j] = w2;
        wgt[6 * cap + j] = wgt[7 * cap + j] = wgt[8 * cap + j] = 0.0;
      }
    }
    if (tid == 0) {  // the new support, in every CTA's resident copy
      sh.ux[n] = px;
      sh.uy[n] = py;
      sh.uz[n] = pz;
      sh.sx[n] = px * inv_r;
      sh.sy[n] = py * inv_r;
      sh.sz[n] = pz * inv_r;
      sh.wx[n] = yn0 * inv_l;
      sh.wy[n] = yn1 * inv_l;
      sh.wz[n] = yn2 * inv_l;
      sh.y0[n] = yn0;
      sh.y1[n] = yn1;
      sh.y2[n] = yn2;
      a.inel[pos] = 1;
      if (rank == 0) {  // and in the global state
        Lirow[n] = inv_l;
        a.L[tri_off(n) + n] = l;
        a.y[3 * (int64_t)n] = yn0;
        a.y[3 * (int64_t)n + 1] = yn1;
        a.y[3 * (int64_t)n + 2] = yn2;
        a.sup[n] = px;
        a.sup[cap + n] = py;
        a.sup[2 * cap + n] = pz;
        wgt[n] = wgt[3 * cap + n] = yn0 * inv_l;
        wgt[cap + n] = wgt[4 * cap + n] = yn1 * inv_l;
        wgt[2 * cap + n] = wgt[5 * cap + n] = yn2 * inv_l;
        wgt[6 * cap + n] = wgt[7 * cap + n] = wgt[8 * cap + n] = 0.0;
        a.sel[n] = pos;
      }
    }
    n += 1;
    sync();
    pc.mark(5);
    return kAccepted;
  }
};

// ================================================================== MsgPath
// 16-CTA cluster, everything a phase reads in shared memory, every
// cross-CTA value pushed with st.async into the consumer's smem and counted
// by the consumer's mbarrier (complete_tx). No cluster barrier and no
// MEMBAR in steady state: a phase costs its math plus one DSMEM hop (~420
// cycles measured, tools/barrier_bench.cu). Factor rows are owner-stable:
// row i of L and Li lives in CTA i % 16 (packed), so the n < kMsgMax rows of
// both factors fit next to the replicated vectors.
constexpr int kMsgMax = 384;
constexpr int kMsgOwnRows = kMsgMax / kClusterCTAs;                 // 24
constexpr int kMsgOwnElems = 8 * kMsgOwnRows * (kMsgOwnRows - 1) + kMsgOwnRows * kClusterCTAs;
// column-owned copy of Li: column j = 16 q + rank holds rows j .. kMsgMax-1
constexpr int kMsgColElems = kMsgOwnRows * kMsgMax - 8 * kMsgOwnRows * (kMsgOwnRows - 1);
constexpr int kMsgGoff = 512;   // group offsets cached in shared memory (else read from L2)
// Overlapped group scans (MsgPath::ov_scan_a / scan_ov): while warps
// 0..kAppWarps-1 append a support, the other kOvWarps warps (one per TMEM
// lane quadrant) evaluate the next group's kernel values phi(|p - s_j|) for
// every support including the one being appended and keep them in tensor
// memory; after the append the group scan is sum_j x'_j phi_j from TMEM
// (3 FMAs per pair instead of 18 FP64 instructions), shared by all warps.
constexpr int kAppWarps = 12;
constexpr int kOvWarps = kLoopWarps - kAppWarps;
static_assert(kOvWarps == 4, "one overlap-scan warp per TMEM lane quadrant");
constexpr int kOvRowsMax = 128;  // rows of a group per CTA
constexpr int kTmemCols = 512;   // 32-bit columns per TMEM lane (all of it)
#ifndef RBF_OV_R
#define RBF_OV_R 4
#endif
#ifndef RBF_OV_C
#define RBF_OV_C (8 / RBF_OV_R)
#endif
constexpr int kOvR = RBF_OV_R;   // rows per overlap row group
constexpr int kOvC = RBF_OV_C;   // support columns per ov_scan_a step: kOvR * kOvC pair chains per lane
constexpr int kOvLd = 16 / kOvR; // chunks per scan_ov TMEM load (16 doubles)
static_assert(kOvR * kOvC == 16 || kOvR * kOvC == 8, "one TMEM store per step");
#ifndef RBF_OV_SLEEP_NS
#define RBF_OV_SLEEP_NS 0
#endif
constexpr unsigned kOvSleepNs = RBF_OV_SLEEP_NS;

enum MsgBar { kMbScan0 = 0, kMbScan1, kMbC0, kMbR, kMbC1, kMbW, kMbCount };

struct MsgShared {
  Common cm;
  double ux[kMsgMax], uy[kMsgMax], uz[kMsgMax];  // support coordinates
  double sx[kMsgMax], sy[kMsgMax], sz[kMsgMax];  // ... scaled by 1/R
  double wx[kMsgMax], wy[kMsgMax], wz[kMsgMax];  // weights (hi + lo, what the scans read)
  double wh[3][kMsgMax], wl[3][kMsgMax];         // compensated weights: hi, lo (comp_add)
  double y0[kMsgMax], y1[kMsgMax], y2[kMsgMax];  // forward-substituted d
  double row[kMsgMax], c0[kMsgMax], r[kMsgMax], c1[kMsgMax];
  double Lown[kMsgOwnElems], Liown[kMsgOwnElems];  // owned rows i = 16 q + rank
  double Licol[kMsgColElems];                      // owned columns of Li
  double u_all[kMsgMax];                           // u = Li^T c, all-gathered
  double rpart[kClusterCTAs][4];                   // c.c, c.y partials
  double part_in[2][kClusterCTAs][2][2];           // scan partials (err, pos as double)
  double acc[kLoopWarps][4][4];
  int goff[kMsgGoff + 1];
  double ov_p[kOvRowsMax][3];        // overlap scan: this CTA's rows of the next group: scaled points,
  double ov_d[kOvRowsMax][3];        // displacements,
  int ov_pos[kOvRowsMax];            // positions
  unsigned char ov_el[kOvRowsMax];   // and eligibility (but for the node being appended, ov_added)
  int ov_added;                      // node appended while the rows were evaluated
  unsigned tmem_base;        // TMEM allocation (kTmemCols columns)
  int ov_res, ov_n;          // append result / n after it, for the scan warps
  int ov_group, ov_nold;     // overlap valid for group ov_group, computed at n = ov_nold
  unsigned ov_bits;          // mbarrier phase bits of the append warps
  alignas(8) unsigned long long mbar[kMbCount];
};
static_assert(sizeof(MsgShared) <= 227 * 1024, "MsgShared exceeds shared memory");
static_assert(sizeof(SmemShared) <= 227 * 1024, "SmemShared exceeds shared memory");
static_assert(sizeof(GlobalShared) <= 227 * 1024, "GlobalShared exceeds shared memory");
static_assert(6 * kSupTile >= kRowSmemMax, "stage_x uses sx..wz as one kRowSmemMax buffer");


__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ unsigned mapa(unsigned local, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async(unsigned raddr, double v, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
               "d"(v), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async2(unsigned raddr, double v0, double v1, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "d"(v0), "d"(v1), "r"(rbar)
               : "memory");
}

template <class Clock>
struct MsgPath {
  const rbf_gcb_args& a;
  const LoopScratch& s;
  MsgShared& sh;
  double inv_r;
  Clock& pc;
  unsigned phase_bits;  // parity of the next completion of each mbarrier

  static constexpr int kMaxN = kMsgMax;
  __device__ Best* best_cache() { return nullptr; }  // (the tail launch is a GlobalPath)
  __device__ static constexpr int best_cache_cap() { return 0; }
  __device__ Common& cm() { return sh.cm; }
  unsigned gathers;  // publications so far (cross-cluster sequence numbers)
  double min_p2 = 1.0;  // min over the factor's l_i * l_i (identical in every thread)
  __device__ bool refine() const { return (a.flags & RBF_GCB_REFINE) || !(min_p2 >= kRefineBelowP2); }
  __device__ void note_pivot(int res, double p2) {
    if (res == kAccepted) {
      const double l = sqrt(p2);
      min_p2 = fmin(min_p2, l * l);
    }
  }
  __device__ int rank() const { return blockIdx.x % kClusterCTAs; }
  __device__ int cluster() const { return blockIdx.x / kClusterCTAs; }
  __device__ int nclusters() const { return gridDim.x / kClusterCTAs; }

  __device__ static int own_off(int q, int rank) { return 8 * q * (q - 1) + q * (rank + 1); }
  // column j = 16 qc + rank, capacity kMsgMax - j entries (rows j ..)
  __device__ static int own_col_off(int qc, int rank) {
    return qc * (kMsgMax - rank) - 8 * qc * (qc - 1);
  }

  // -------------------------------------------------------------- mbarriers
  __device__ void expect(int bar, unsigned bytes) {
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&sh.mbar[bar])),
                   "r"(bytes)
                   : "memory");
  }
  __device__ void wait(int bar) {
    const unsigned parity = (phase_bits >> bar) & 1u;
    const unsigned addr = smem_u32(&sh.mbar[bar]);
    unsigned done = 0, spins = 0;
    uint64_t t0 = 0;
    while (true) {
      // suspend-time hint: the warp sleeps in the barrier unit (up to 1 ms)
      // instead of re-issuing try_wait -- spinning warps were ~15 % of the
      // kernel's issued instructions, taken from the warps doing the work
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(addr), "r"(parity), "r"(1000000u)
          : "memory");
      if (done) break;
      if ((++spins & 63u) == 0) {
        const uint64_t now = globaltimer_ns();
        if (t0 == 0) {
          t0 = now;
        } else if (now - t0 > 20ull * 1000000000ull) {
          atomicExch(s.fault, 2);
          __trap();
        }
      }
    }
    phase_bits ^= 1u << bar;
  }
  // address of `p` (a field of MsgShared) in CTA `dst` and that CTA's mbarrier
  __device__ __forceinline__ unsigned raddr(const void* p, int dst) { return mapa(smem_u32(p), dst); }
  __device__ __forceinline__ unsigned rbar(int bar, int dst) { return mapa(smem_u32(&sh.mbar[bar]), dst); }

  // rare-path / exit barrier: the whole team (all clusters) when there are
  // several (the launch is cooperative), else the cluster
  __device__ void sync() {
    if (nclusters() > 1)
      cg::this_grid().sync();
    else
      cg::this_cluster().sync();
  }

  __device__ void begin(int n) {
    const int cap = a.cap, rk = rank();
    if (threadIdx.x == 0) {
      for (int b = 0; b < kMbCount; ++b)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sh.mbar[b])) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    phase_bits = 0;
    for (int j = threadIdx.x; j < n; j += kLoopThreads) {
      const double x = __ldcg(a.sup + j), y = __ldcg(a.sup + cap + j), z = __ldcg(a.sup + 2 * cap + j);
      sh.ux[j] = x;
      sh.uy[j] = y;
      sh.uz[j] = z;
      sh.sx[j] = x * inv_r;
      sh.sy[j] = y * inv_r;
      sh.sz[j] = z * inv_r;
      sh.wx[j] = __ldcg(a.sup + 3 * cap + j);
      sh.wy[j] = __ldcg(a.sup + 4 * cap + j);
      sh.wz[j] = __ldcg(a.sup + 5 * cap + j);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        sh.wh[k][j] = __ldcg(a.sup + (6 + k) * (int64_t)cap + j);
        sh.wl[k][j] = __ldcg(a.sup + (9 + k) * (int64_t)cap + j);
      }
      sh.y0[j] = __ldcg(a.y + 3 * j);
      sh.y1[j] = __ldcg(a.y + 3 * j + 1);
      sh.y2[j] = __ldcg(a.y + 3 * j + 2);
    }
    // owned factor rows i = 16 q + rank < n, owned columns of Li
    for (int q = 0; 16 * q + rk < n; ++q) {
      const int i = 16 * q + rk, o = own_off(q, rk), oc = own_col_off(q, rk);
      for (int j = threadIdx.x; j <= i; j += kLoopThreads) {
        sh.Lown[o + j] = __ldcg(a.L + tri_off(i) + j);
        sh.Liown[o + j] = __ldcg(a.Li + tri_off(i) + j);
      }
      for (int r = i + threadIdx.x; r < n; r += kLoopThreads) sh.Licol[oc + (r - i)] = __ldcg(a.Li + tri_off(r) + i);
    }
    for (int g = threadIdx.x; g <= a.m && g <= kMsgGoff; g += kLoopThreads) sh.goff[g] = __ldg(a.group_off + g);
    // min l_i^2 of the rows already factored (a resumed run decides its
    // refinements exactly as an uninterrupted one: note_pivot squares the
    // same stored l)
    double mp = 1.0;
    for (int i = threadIdx.x; i < n; i += kLoopThreads) {
      const double l = __ldcg(a.L + tri_off(i) + i);
      mp = fmin(mp, l * l);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mp = fmin(mp, __shfl_xor_sync(0xffffffffu, mp, off));
    if ((threadIdx.x & 31) == 0) sh.cm.wred[threadIdx.x >> 5][0] = mp;
    __syncthreads();
    min_p2 = 1.0;
    for (int w = 0; w < kLoopWarps; ++w) min_p2 = fmin(min_p2, sh.cm.wred[w][0]);
    __syncthreads();
  }
  __device__ void finish() { sync(); }
  __device__ int group_off(int g) { return a.m <= kMsgGoff ? sh.goff[g] : __ldg(a.group_off + g); }

  // ---------------------------------------------------------------- partials
  // lanes 0..15 of warp 0 hold the CTA's (bu, br): push them to every CTA
  __device__ void publish2(Best bu, Best br, int par) {
    if (threadIdx.x < kClusterCTAs) {
      const int dst = threadIdx.x, bar = kMbScan0 + par;
      st_async2(raddr(&sh.part_in[par][rank()][0][0], dst), bu.err, (double)bu.pos, rbar(bar, dst));
      st_async2(raddr(&sh.part_in[par][rank()][1][0], dst), br.err, (double)br.pos, rbar(bar, dst));
    }
  }
  __device__ void publish(Best b, int slot, int par) {  // seeds: slot 0 only
    publish2(b, Best{-1.0, kNone}, par);
  }
  // wait for the 16 CTAs' partials of this parity and fold them (fixed order)
  __device__ void gather(int par, int nslots) {
    expect(kMbScan0 + par, kClusterCTAs * 32);
    wait(kMbScan0 + par);
    if (threadIdx.x < 32 * nslots) {
      const int slot = threadIdx.x >> 5, lane = threadIdx.x & 31;
      Best b{-1.0, kNone};
      if (lane < kClusterCTAs)
        b = Best{sh.part_in[par][lane][slot][0], (int)sh.part_in[par][lane][slot][1]};
      b = warp_best(b);
      if (lane == 0) sh.cm.bcast[slot] = b;
    }
    __syncthreads();
    const int ncl = nclusters();
    if (ncl > 1) {  // combine the clusters' results through L2
      const unsigned seq = ++gathers;
      if (rank() == 0 && threadIdx.x == 0) {
        double* slot = s.xc + (par * 16 + cluster()) * 4;
        slot[0] = sh.cm.bcast[0].err;
        slot[1] = (double)sh.cm.bcast[0].pos;
        slot[2] = sh.cm.bcast[1].err;
        slot[3] = (double)sh.cm.bcast[1].pos;
        __threadfence();
        st_release(s.xseq + par * 16 + cluster(), seq);
      }
      if (threadIdx.x < 32 * nslots) {
        const int slot = threadIdx.x >> 5, lane = threadIdx.x & 31;
        Best b{-1.0, kNone};
        if (lane < ncl) {
          uint64_t t0 = 0;
          unsigned spins = 0;
          while (ld_acquire(s.xseq + par * 16 + lane) != seq) {
            if ((++spins & 1023u) == 0) {
              const uint64_t now = globaltimer_ns();
              if (t0 == 0) {
                t0 = now;
              } else if (now - t0 > 20ull * 1000000000ull) {
                atomicExch(s.fault, 3);
                __trap();
              }
            }
          }
          const double* x = s.xc + (par * 16 + lane) * 4;
          b = Best{__ldcg(x + 2 * slot), (int)__ldcg(x + 2 * slot + 1)};
        }
        b = warp_best(b);
        if (lane == 0) sh.cm.bcast[slot] = b;
      }
      __syncthreads();
    }
  }

  // -------------------------------------------------------------------- scan
  // targets per lane chosen so the CTA's rows fill as many warps as possible
  __device__ __forceinline__ void scan(const int* gpos, const double* gpt, const double* gdisp, int card, int n,
                       int par) {
    // this CTA's rows [lo, hi): shifts for the one-cluster team (no integer
    // divisions in the scan prologue, which every warp executes)
    const unsigned b = blockIdx.x, G = gridDim.x;
    const int lo = G == kClusterCTAs ? (int)(((unsigned)card * b) >> 4) : (int)((int64_t)card * b / G);
    const int hi = G == kClusterCTAs ? (int)(((unsigned)card * (b + 1)) >> 4) : (int)((int64_t)card * (b + 1) / G);
    const int mine = hi - lo;
    if (mine <= kLoopWarps)
      scan_t<1>(gpos, gpt, gdisp, lo, hi, n, par);
    else if (mine <= 2 * kLoopWarps)
      scan_t<2>(gpos, gpt, gdisp, lo, hi, n, par);
    else if (mine <= 3 * kLoopWarps)
      scan_t<3>(gpos, gpt, gdisp, lo, hi, n, par);
    else
      scan_t<4>(gpos, gpt, gdisp, lo, hi, n, par);
  }

  template <int kTPT>
  __device__ __forceinline__ void scan_t(const int* gpos, const double* gpt, const double* gdisp, int lo, int hi, int n,
                         int par) {
    const int tid = threadIdx.x, lane = tid & 31;
    const int tgroups = (hi - lo + kTPT - 1) / kTPT;
    int lg = 5;  // S = 1 << lg lanes per target group: shifts and masks only
    while (lg > 0 && (tgroups << lg) > kLoopThreads) --lg;
    const int S = 1 << lg;
    const int per_round = kLoopThreads >> lg;
    const int rounds = (tgroups + per_round - 1) >> (9 - lg);  // kLoopThreads = 2^9
    const int sub = tid & (S - 1);
    Best bu{-1.0, kNone}, br{-1.0, kNone};
    for (int rd = 0; rd < rounds; ++rd) {
      const int tg = rd * per_round + (tid >> lg);
      double px[kTPT], py[kTPT], pz[kTPT];
      double v[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = 0.0;
#pragma unroll
      for (int q = 0; q < kTPT; ++q) {
        const int t = lo + kTPT * tg + q;
        const bool ok = tg < tgroups && t < hi;
        px[q] = ok ? __ldcg(gpt + 3 * (int64_t)t) * inv_r : 0.0;
        py[q] = ok ? __ldcg(gpt + 3 * (int64_t)t + 1) * inv_r : 0.0;
        pz[q] = ok ? __ldcg(gpt + 3 * (int64_t)t + 2) * inv_r : 0.0;
        v[4 * q] = v[4 * q + 1] = v[4 * q + 2] = v[4 * q + 3] = 0.0;
      }
      const int my_t = lo + kTPT * tg + (S == 32 ? lane : 0);
      const bool mine = S == 32 && lane < kTPT && tg < tgroups && my_t < hi;
      int my_pos = -1;
      bool my_elig = false;
      double dx = 0.0, dy = 0.0, dz = 0.0;
      if (mine) {
        my_pos = gpos ? __ldg(gpos + my_t) : my_t;
        my_elig = !__ldcg(reinterpret_cast<const unsigned char*>(a.inel) + my_pos);
        dx = __ldcg(gdisp + 3 * (int64_t)my_t);
        dy = __ldcg(gdisp + 3 * (int64_t)my_t + 1);
        dz = __ldcg(gdisp + 3 * (int64_t)my_t + 2);
      }
      if (tg < tgroups) {
#pragma unroll 1
        for (int j = sub; j < n; j += S) {
          const double sx = sh.sx[j], sy = sh.sy[j], sz = sh.sz[j];
          const double wx = sh.wx[j], wy = sh.wy[j], wz = sh.wz[j];
#pragma unroll
          for (int q = 0; q < kTPT; ++q)
            pair_accum(px[q], py[q], pz[q], sx, sy, sz, wx, wy, wz, v[4 * q], v[4 * q + 1], v[4 * q + 2]);
        }
      }
      if (rd == 0) pc.mark(11);
      if (S == 32) {
        int idx;
        const double tot = warp_reduce_scatter16(v, lane, idx);
        const int w = tid >> 5;
        if ((lane & 1) == 0 && (idx & 3) != 3) sh.acc[w][idx >> 2][idx & 3] = tot;
        __syncwarp();
        if (rd == 0) pc.mark(12);
        if (mine) {
          const double e = residual_norm(dx, dy, dz, sh.acc[w][lane][0], sh.acc[w][lane][1],
                                         sh.acc[w][lane][2]);
          s.err[my_t] = e;
          bu = Best{e, my_pos};
          if (my_elig) br = Best{e, my_pos};
        }
        __syncwarp();
      } else {
#pragma unroll
        for (int q = 0; q < kTPT; ++q) {
          for (int off = S >> 1; off > 0; off >>= 1) {
            v[4 * q] += __shfl_xor_sync(0xffffffffu, v[4 * q], off);
            v[4 * q + 1] += __shfl_xor_sync(0xffffffffu, v[4 * q + 1], off);
            v[4 * q + 2] += __shfl_xor_sync(0xffffffffu, v[4 * q + 2], off);
          }
        }
        if (rd == 0) pc.mark(12);
        if (sub == 0 && tg < tgroups) {
#pragma unroll
          for (int q = 0; q < kTPT; ++q) {
            const int t = lo + kTPT * tg + q;
            if (t >= hi) continue;
            const int pos = gpos ? __ldg(gpos + t) : t;
            const double e = residual_norm(__ldcg(gdisp + 3 * (int64_t)t), __ldcg(gdisp + 3 * (int64_t)t + 1),
                                           __ldcg(gdisp + 3 * (int64_t)t + 2), v[4 * q], v[4 * q + 1],
                                           v[4 * q + 2]);
            s.err[t] = e;
            if (better(e, pos, bu.err, bu.pos)) bu = Best{e, pos};
            if (!__ldcg(reinterpret_cast<const unsigned char*>(a.inel) + pos) && better(e, pos, br.err, br.pos))
              br = Best{e, pos};
          }
        }
      }
      if (rd == 0) pc.mark(13);
    }
    cta_best2(sh.cm, bu, br, S == 32 ? kTPT : 32);
    if (threadIdx.x < 32) publish2(bu, br, par);
    pc.mark(14);
  }

  // ------------------------------------------------------------- overlap
  static constexpr bool kHasOv = true;
  __device__ __forceinline__ void bar_ov() { asm volatile("bar.sync 2, %0;" ::"n"(kLoopThreads) : "memory"); }
  template <bool kOv>
  __device__ __forceinline__ void sync_a() {
    if (kOv)
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kAppWarps) : "memory");
    else
      __syncthreads();
  }
  __device__ __forceinline__ static void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  __device__ __forceinline__ static void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  // all of TMEM for this CTA (one CTA per SM), allocated by the last warp
  __device__ void tmem_alloc() {
    if ((threadIdx.x >> 5) == kLoopWarps - 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&sh.tmem_base)),
                   "n"(kTmemCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  __device__ void tmem_free() {
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if ((threadIdx.x >> 5) == kLoopWarps - 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sh.tmem_base), "n"(kTmemCols)
                   : "memory");
  }
  // 4 doubles of this thread <-> 8 consecutive 32-bit columns of its TMEM lane
  __device__ __forceinline__ static void tmem_st4(unsigned taddr, const double (&f)[4]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
        "r"(__double2loint(f[0])), "r"(__double2hiint(f[0])), "r"(__double2loint(f[1])), "r"(__double2hiint(f[1])),
        "r"(__double2loint(f[2])), "r"(__double2hiint(f[2])), "r"(__double2loint(f[3])), "r"(__double2hiint(f[3]))
        : "memory");
  }
  __device__ __forceinline__ static void tmem_st8(unsigned taddr, const double* f) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16};" ::"r"(taddr),
        "r"(__double2loint(f[0])), "r"(__double2hiint(f[0])), "r"(__double2loint(f[1])), "r"(__double2hiint(f[1])),
        "r"(__double2loint(f[2])), "r"(__double2hiint(f[2])), "r"(__double2loint(f[3])), "r"(__double2hiint(f[3])),
        "r"(__double2loint(f[4])), "r"(__double2hiint(f[4])), "r"(__double2loint(f[5])), "r"(__double2hiint(f[5])),
        "r"(__double2loint(f[6])), "r"(__double2hiint(f[6])), "r"(__double2loint(f[7])), "r"(__double2hiint(f[7]))
        : "memory");
  }
  __device__ __forceinline__ static void tmem_st16(unsigned taddr, const double* f) {
    unsigned r[32];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      r[2 * i] = (unsigned)__double2loint(f[i]);
      r[2 * i + 1] = (unsigned)__double2hiint(f[i]);
    }
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
  }
  __device__ __forceinline__ static void tmem_ld4(unsigned taddr, double (&f)[4]) {
    unsigned r0, r1, r2, r3, r4, r5, r6, r7;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3), "=r"(r4), "=r"(r5), "=r"(r6), "=r"(r7)
                 : "r"(taddr)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    f[0] = __hiloint2double((int)r1, (int)r0);
    f[1] = __hiloint2double((int)r3, (int)r2);
    f[2] = __hiloint2double((int)r5, (int)r4);
    f[3] = __hiloint2double((int)r7, (int)r6);
  }

  // 16 doubles (4 column chunks of 4) in one load, one wait
  __device__ __forceinline__ static void tmem_ld16(unsigned taddr, double (&f)[16]) {
    unsigned r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) f[i] = __hiloint2double((int)r[2 * i + 1], (int)r[2 * i]);
  }

  // can the next group (card rows) be scanned during an append at n supports
  __device__ bool ov_fits(int card, int n) {
    if ((a.flags & RBF_GCB_NO_OVERLAP) || nclusters() != 1 || n + 1 >= kMsgMax) return false;
    const int rows = (card + kClusterCTAs - 1) / kClusterCTAs;
    if (rows > kOvRowsMax) return false;
    const int rounds = ((rows + kOvR - 1) / kOvR + kOvWarps - 1) / kOvWarps;
    const int ji = (n + 1 + 31) >> 5;
    return 2 * kOvR * rounds * ov_stride(ji) <= kTmemCols;
  }

  // TMEM layout of the overlap: scan warp qd (lane quadrant qd) keeps the
  // row groups rg = qd, qd + 4, ... (round r = rg >> 2) of kOvR rows; its
  // lane holds, per round, chunks ji = 0 .. ji_n-1 (columns j = 32 ji +
  // lane) of kOvR doubles at 32-bit column 2 kOvR (r * stride + ji).
  __device__ __forceinline__ static int ov_stride(int ji_n) {
    constexpr int kQ = kOvC > kOvLd ? kOvC : kOvLd;
    return (ji_n + kQ - 1) / kQ * kQ;
  }

  // Scan warps, during the append of support n (coordinates s*, scaled):
  // phi of the next group's rows against supports 0 .. n (n: the new one),
  // kOvC columns at a time (kOvR * kOvC independent pair chains per lane:
  // one warp per SMSP keeps the FP64 pipe busy on its own), into TMEM; the
  // rows' positions and displacements into shared memory.
  __device__ void ov_scan_a(int off, int card, int n, double spx, double spy, double spz) {
    const int wq = (threadIdx.x >> 5) - kAppWarps, lane = threadIdx.x & 31;
    const unsigned b = blockIdx.x;
    const int lo = (int)(((unsigned)card * b) >> 4), hi = (int)(((unsigned)card * (b + 1)) >> 4);
    const int ng = (hi - lo + kOvR - 1) / kOvR, ji_n = (n + 1 + 31) >> 5, stride = ov_stride(ji_n);
    const unsigned tl = sh.tmem_base + ((unsigned)(32 * wq) << 16);
    const double* gpt = s.gpt + 3 * (int64_t)off;
    // this warp's rows (groups rg = wq + 4 r) -> shared memory in one round trip
    for (int k = lane; k < kOvRowsMax; k += 32) {
      const int i = kOvR * (wq + kOvWarps * (k / kOvR)) + k % kOvR, t = lo + i;
      if (t >= hi) break;
      const int pos = __ldg(a.group_pos + off + t);
      sh.ov_pos[i] = pos;
      // eligibility: only the node being appended can change before scan_ov
      // (rejected candidates are marked before the next attempt re-runs this)
      sh.ov_el[i] = !__ldcg(reinterpret_cast<const unsigned char*>(a.inel) + pos);
      sh.ov_p[i][0] = __ldcg(gpt + 3 * (int64_t)t) * inv_r;
      sh.ov_p[i][1] = __ldcg(gpt + 3 * (int64_t)t + 1) * inv_r;
      sh.ov_p[i][2] = __ldcg(gpt + 3 * (int64_t)t + 2) * inv_r;
      sh.ov_d[i][0] = __ldcg(s.gdisp + 3 * ((int64_t)off + t));
      sh.ov_d[i][1] = __ldcg(s.gdisp + 3 * ((int64_t)off + t) + 1);
      sh.ov_d[i][2] = __ldcg(s.gdisp + 3 * ((int64_t)off + t) + 2);
    }
    __syncwarp();
    int r = 0;
    for (int rg = wq; rg < ng; rg += kOvWarps, ++r) {
      double px[kOvR], py[kOvR], pz[kOvR];
#pragma unroll
      for (int q = 0; q < kOvR; ++q) {
        const int i = kOvR * rg + q;
        const bool ok = lo + i < hi;
        px[q] = ok ? sh.ov_p[i][0] : 0.0;
        py[q] = ok ? sh.ov_p[i][1] : 0.0;
        pz[q] = ok ? sh.ov_p[i][2] : 0.0;
      }
#pragma unroll 1
      for (int ji = 0; ji < ji_n; ji += kOvC) {
        double f[kOvR * kOvC];
#pragma unroll
        for (int h = 0; h < kOvC; ++h) {
          const int j = 32 * (ji + h) + lane;
          const bool old = j < n, add = j == n;
          const int jj = old ? j : 0;
          const double sx = add ? spx : sh.sx[jj], sy = add ? spy : sh.sy[jj], sz = add ? spz : sh.sz[jj];
#pragma unroll
          for (int q = 0; q < kOvR; ++q) {
            const double fq = pair_phi(px[q], py[q], pz[q], sx, sy, sz);
            f[kOvR * h + q] = (old || add) ? fq : 0.0;
          }
        }
        if constexpr (kOvR * kOvC == 16)
          tmem_st16(tl + 2u * kOvR * (unsigned)(r * stride + ji), f);
        else
          tmem_st8(tl + 2u * kOvR * (unsigned)(r * stride + ji), f);
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  // The scan of the group whose kernel values ov_scan_a stored, after the
  // append (n supports now, weights x'): every warp takes rounds of its lane
  // quadrant (warps w, w + 4, w + 8, w + 12 share quadrant w % 4), sums
  // x'_j phi_j over its lanes' columns in increasing j, butterfly-sums the
  // lanes and finishes errors, arg-max partials and publication as scan().
  __device__ void scan_ov(const int*, const double*, int card, int n, int par) {
    Best bu{-1.0, kNone}, br{-1.0, kNone};
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int qd = warp & 3, wr = warp >> 2;
    const unsigned b = blockIdx.x;
    const int lo = (int)(((unsigned)card * b) >> 4), hi = (int)(((unsigned)card * (b + 1)) >> 4);
    const int ng = (hi - lo + kOvR - 1) / kOvR, ji_n = (n + 31) >> 5, stride = ov_stride(ji_n);
    const unsigned tl = sh.tmem_base + ((unsigned)(32 * qd) << 16);
    // rounds of quadrant qd: rg = qd + 4 r < ng; this warp: r = wr, wr + 4, ..
    for (int r = wr; qd + 4 * r < ng; r += 4) {
      const int rg = qd + 4 * r;
      static_assert(kOvR == 4, "scan_ov reduce-scatters 4 rows x 4 slots");
      double v[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = 0.0;
#pragma unroll 1
      for (int j0 = 0; j0 < ji_n; j0 += kOvLd) {
        double f[16];
        tmem_ld16(tl + 2u * kOvR * (unsigned)(r * stride + j0), f);
#pragma unroll
        for (int h = 0; h < kOvLd; ++h) {
          const int j = 32 * (j0 + h) + lane;
          const bool in = j < n;
          const int jj = in ? j : 0;
          const double wx = in ? sh.wx[jj] : 0.0, wy = in ? sh.wy[jj] : 0.0, wz = in ? sh.wz[jj] : 0.0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            v[4 * q] = fma(wx, f[4 * h + q], v[4 * q]);
            v[4 * q + 1] = fma(wy, f[4 * h + q], v[4 * q + 1]);
            v[4 * q + 2] = fma(wz, f[4 * h + q], v[4 * q + 2]);
          }
        }
      }
      if (r == 0) pc.mark(12);
      int idx;
      const double tot = warp_reduce_scatter16(v, lane, idx);
      if ((lane & 1) == 0 && (idx & 3) != 3) sh.acc[warp][idx >> 2][idx & 3] = tot;
      __syncwarp();
      if (r == 0) pc.mark(13);
      const int i = 4 * rg + lane, t = lo + i;
      if (lane < 4 && t < hi) {
        const double e = residual_norm(sh.ov_d[i][0], sh.ov_d[i][1], sh.ov_d[i][2], sh.acc[warp][lane][0],
                                       sh.acc[warp][lane][1], sh.acc[warp][lane][2]);
        s.err[t] = e;
        const int pos = sh.ov_pos[i];
        if (better(e, pos, bu.err, bu.pos)) bu = Best{e, pos};
        if (sh.ov_el[i] && pos != sh.ov_added && better(e, pos, br.err, br.pos)) br = Best{e, pos};
      }
      __syncwarp();
    }
    pc.mark(11);
    cta_best2(sh.cm, bu, br, kOvR);
    if (threadIdx.x < 32) publish2(bu, br, par);
    pc.mark(14);
  }

  // append of `pos` with the scan of the next group (off, card) overlapped
  __device__ int append_ov(int pos, int& n, bool check_dup, double* pivot2_out, int off, int card) {
    const int n0 = n;
    int res = kAccepted;
    double p2 = 0.0;
    if ((threadIdx.x >> 5) < kAppWarps) {
      res = append_t<true>(pos, n, check_dup, &p2);
    } else {
      ov_scan_a(off, card, n0, __ldg(a.points + 3 * (int64_t)pos) * inv_r,
                __ldg(a.points + 3 * (int64_t)pos + 1) * inv_r, __ldg(a.points + 3 * (int64_t)pos + 2) * inv_r);
      bar_ov();
    }
    if (threadIdx.x == 0) {
      sh.ov_res = res;
      sh.ov_added = pos;
      sh.ov_n = n;
      sh.ov_bits = phase_bits;
      sh.cm.dbl[5] = p2;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    res = sh.ov_res;
    n = sh.ov_n;
    phase_bits = sh.ov_bits;  // the scan warps skipped the append's waits
    *pivot2_out = sh.cm.dbl[5];
    note_pivot(res, *pivot2_out);
    return res;
  }
  __device__ int append(int pos, int& n, bool check_dup, double* pivot2_out) {
    const int res = append_t<false>(pos, n, check_dup, pivot2_out);
    note_pivot(res, *pivot2_out);
    return res;
  }

  // ------------------------------------------------------------------ append
  // owned rows: q = 0.. with i = 16 q + rank < n (q < 24 here); warp w takes
  // q = w and q = w + 16 together, so no warp handles two rows one after the
  // other
  template <int kW, typename F>
  __device__ __forceinline__ void for_owned_row_pairs(int n, F&& body) {
    const int warp = threadIdx.x >> 5, rk = rank();
    for (int q = warp; 16 * q + rk < n; q += 2 * kW) {
      const int qb = q + kW;
      body(q, 16 * q + rk, 16 * qb + rk < n ? qb : -1, 16 * qb + rk);
    }
  }

  // dot products of packed owned rows (qa: length ia+1; qb < 0: none) with
  // x, loads of both rows issued before the FMAs, the two warp reductions
  // interleaved
  template <typename XL>
  __device__ __forceinline__ void own_dot2(const double* M, int qa, int ia, int qb, int ib, XL x,
                                           int lane, double& sa, double& sb) {
    const double* ra = M + own_off(qa, rank());
    const double* rb = M + own_off(qb < 0 ? 0 : qb, rank());
    const int la = ia + 1, lb = qb < 0 ? 0 : ib + 1;
    const int len = la > lb ? la : lb;
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
    for (int j0 = 0; j0 < len; j0 += 4 * kWarp) {
      double av[4], bv[4], xv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + u * kWarp + lane;
        xv[u] = j < len ? x(j) : 0.0;
        av[u] = j < la ? ra[j] : 0.0;
        bv[u] = j < lb ? rb[j] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; u += 2) {
        a0 = fma(av[u], xv[u], a0);
        a1 = fma(av[u + 1], xv[u + 1], a1);
        b0 = fma(bv[u], xv[u], b0);
        b1 = fma(bv[u + 1], xv[u + 1], b1);
      }
    }
    double va = a0 + a1, vb = b0 + b1;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      va += __shfl_xor_sync(0xffffffffu, va, off);
      vb += __shfl_xor_sync(0xffffffffu, vb, off);
    }
    sa = va;
    sb = vb;
  }

  // value v of owned row i -> vector `vec` in all 16 CTAs (lanes 0..15 send)
  __device__ __forceinline__ void bcast(double* vec, int i, double v, int bar, int lane) {
    if (lane < kClusterCTAs) st_async(raddr(&vec[i], lane), v, rbar(bar, lane));
  }

  // kOv: warps 0..kAppWarps-1 only (the others scan the next group
  // meanwhile, ov_scan_a); every path of the append passes bar_ov() exactly
  // once, before the weights are updated
  template <bool kOv>
  __device__ int append_t(int pos, int& n, bool check_dup, double* pivot2_out) {
    constexpr int kWA = kOv ? kAppWarps : kLoopWarps, kTA = 32 * kWA;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rk = rank();
    const int cap = a.cap;
    const double px = __ldg(a.points + 3 * (int64_t)pos), py = __ldg(a.points + 3 * (int64_t)pos + 1),
                 pz = __ldg(a.points + 3 * (int64_t)pos + 2);
    bool near;
    {  // exact_row() over the append warps
      if (tid == 0) sh.cm.dbl[0] = 0.0;
      sync_a<kOv>();
      bool nr = false;
      for (int j = tid; j < n; j += kTA) {
        const double d = cdist_exact(px, py, pz, sh.ux[j], sh.uy[j], sh.uz[j]);
        sh.row[j] = phi_exact(d, a.radius);
        nr |= d < a.dup_dist;
      }
      if (__any_sync(0xffffffffu, nr) && lane == 0) sh.cm.dbl[0] = 1.0;
      sync_a<kOv>();
      near = sh.cm.dbl[0] != 0.0;
    }
    if (check_dup && n > 0 && near) {
      if (kOv) bar_ov();
      return kRejectDup;
    }
    pc.mark(1);
    const bool ref = refine();
    if (ref) {
      // c0 = Li row
      expect(kMbC0, n * 8);
      for_owned_row_pairs<kWA>(n, [&](int qa, int ia, int qb, int ib) {
        double va, vb;
        own_dot2(sh.Liown, qa, ia, qb, ib, [&](int j) { return sh.row[j]; }, lane, va, vb);
        bcast(sh.c0, ia, va, kMbC0, lane);
        if (qb >= 0) bcast(sh.c0, ib, vb, kMbC0, lane);
      });
      wait(kMbC0);
      pc.mark(2);
      // r = row - L c0
      expect(kMbR, n * 8);
      for_owned_row_pairs<kWA>(n, [&](int qa, int ia, int qb, int ib) {
        double va, vb;
        own_dot2(sh.Lown, qa, ia, qb, ib, [&](int j) { return sh.c0[j]; }, lane, va, vb);
        bcast(sh.r, ia, sh.row[ia] - va, kMbR, lane);
        if (qb >= 0) bcast(sh.r, ib, sh.row[ib] - vb, kMbR, lane);
      });
      wait(kMbR);
    }
    pc.mark(3);
    // c = c0 + Li r (refined) or c = Li row, partial sums of c.c and c.y over
    // the owned rows
    expect(kMbC1, n * 8 + kClusterCTAs * 32);
    double pcc = 0.0, pcy0 = 0.0, pcy1 = 0.0, pcy2 = 0.0;
    const double* xv = ref ? sh.r : sh.row;
    for_owned_row_pairs<kWA>(n, [&](int qa, int ia, int qb, int ib) {
      double va, vb;
      own_dot2(sh.Liown, qa, ia, qb, ib, [&](int j) { return xv[j]; }, lane, va, vb);
      const double ca = ref ? sh.c0[ia] + va : va;
      bcast(sh.c1, ia, ca, kMbC1, lane);
      pcc = fma(ca, ca, pcc);
      pcy0 = fma(ca, sh.y0[ia], pcy0);
      pcy1 = fma(ca, sh.y1[ia], pcy1);
      pcy2 = fma(ca, sh.y2[ia], pcy2);
      if (qb >= 0) {
        const double cb = ref ? sh.c0[ib] + vb : vb;
        bcast(sh.c1, ib, cb, kMbC1, lane);
        pcc = fma(cb, cb, pcc);
        pcy0 = fma(cb, sh.y0[ib], pcy0);
        pcy1 = fma(cb, sh.y1[ib], pcy1);
        pcy2 = fma(cb, sh.y2[ib], pcy2);
      }
    });
    Common& cm = sh.cm;
    if (lane == 0) {
      cm.wred[warp][0] = pcc;
      cm.wred[warp][1] = pcy0;
      cm.wred[warp][2] = pcy1;
      cm.wred[warp][3] = pcy2;
    }
    sync_a<kOv>();
    if (tid < 4 * kClusterCTAs) {  // CTA partial (warp order) -> every CTA
      const int c = tid & 3, dst = tid >> 2;
      double t = 0.0;
      for (int w = 0; w < kWA; ++w) t += cm.wred[w][c];
      st_async(raddr(&sh.rpart[rk][c], dst), t, rbar(kMbC1, dst));
    }
    wait(kMbC1);
    pc.mark(4);
    if (tid < 4) {  // fixed-order fold of the 16 CTA partials
      double t = 0.0;
      for (int c = 0; c < kClusterCTAs; ++c) t += sh.rpart[c][tid];
      cm.dbl[1 + tid] = t;
    }
    sync_a<kOv>();
    const double pivot2 = 1.0 - cm.dbl[1];  // row[n] = phi(0) = 1 exactly
    *pivot2_out = pivot2;
    if (!(pivot2 > 0.0)) {
      sync_a<kOv>();
      if (kOv) bar_ov();
      return kRejectPivot;
    }
    const double l = sqrt(pivot2);
    const double inv_l = 1.0 / l;
    const double yn0 = (__ldg(a.disp + 3 * (int64_t)pos) - cm.dbl[2]) * inv_l;
    const double yn1 = (__ldg(a.disp + 3 * (int64_t)pos + 1) - cm.dbl[3]) * inv_l;
    const double yn2 = (__ldg(a.disp + 3 * (int64_t)pos + 2) - cm.dbl[4]) * inv_l;
    // u = Li^T c (the weights are updated incrementally,
    // x' = x - (u / l) y_n: as accurate as recomputing Li^T y).
    // Li is also kept column-owned (column j in CTA j % 16), so u_j is a
    // local dot product of column j with the replicated c; one all-gather
    // hands u to every CTA. The column owner appends Li[n][j] = -u_j / l.
    const double neg_inv_l = -inv_l;
    expect(kMbW, (unsigned)(n * 8));
    // warp w takes owned columns qc = w and w + 16 together
    for (int qa = warp; 16 * qa + rk < n; qa += 2 * kWA) {
      const int qb = qa + kWA;
      const int ja = 16 * qa + rk, jb = 16 * qb + rk;
      const bool has_b = jb < n;
      const double* ca = sh.Licol + own_col_off(qa, rk);
      const double* cb = sh.Licol + own_col_off(has_b ? qb : qa, rk);
      double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
      for (int i0 = ja; i0 < n; i0 += 4 * kWarp) {  // rows i >= ja (column b starts later)
        double av[4], bv[4], cv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * kWarp + lane;
          cv[u] = i < n ? sh.c1[i] : 0.0;
          av[u] = i < n ? ca[i - ja] : 0.0;
          bv[u] = (has_b && i < n && i >= jb) ? cb[i - jb] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; u += 2) {
          a0 = fma(av[u], cv[u], a0);
          a1 = fma(av[u + 1], cv[u + 1], a1);
          b0 = fma(bv[u], cv[u], b0);
          b1 = fma(bv[u + 1], cv[u + 1], b1);
        }
      }
      double ua = a0 + a1, ub = b0 + b1;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        ua += __shfl_xor_sync(0xffffffffu, ua, off);
        ub += __shfl_xor_sync(0xffffffffu, ub, off);
      }
      bcast(sh.u_all, ja, ua, kMbW, lane);
      if (lane == 0) sh.Licol[own_col_off(qa, rk) + (n - ja)] = ua * neg_inv_l;
      if (has_b) {
        bcast(sh.u_all, jb, ub, kMbW, lane);
        if (lane == 0) sh.Licol[own_col_off(qb, rk) + (n - jb)] = ub * neg_inv_l;
      }
    }
    if (n % kClusterCTAs == rk && tid == 0) sh.Licol[own_col_off(n / kClusterCTAs, rk)] = inv_l;
    pc.mark(15);
    const int owner = n % kClusterCTAs, qn = n / kClusterCTAs;
    double* Lirow_g = a.Li + tri_off(n);
    double* wgt = a.sup + 3 * (int64_t)cap;
    // the new support, in every CTA's resident copy
    if (tid == 0) {
      sh.ux[n] = px;
      sh.uy[n] = py;
      sh.uz[n] = pz;
      sh.sx[n] = px * inv_r;
      sh.sy[n] = py * inv_r;
      sh.sz[n] = pz * inv_r;
      sh.y0[n] = yn0;
      sh.y1[n] = yn1;
      sh.y2[n] = yn2;
      a.inel[pos] = 1;
      if (rk == 0 && cluster() == 0) {  // global copies
        a.y[3 * (int64_t)n] = yn0;
        a.y[3 * (int64_t)n + 1] = yn1;
        a.y[3 * (int64_t)n + 2] = yn2;
        a.sup[n] = px;
        a.sup[cap + n] = py;
        a.sup[2 * cap + n] = pz;
        wgt[n] = wgt[3 * cap + n] = yn0 * inv_l;  // (wgt = sup row 3: rows 6-8 hi, 9-11 lo)
        wgt[cap + n] = wgt[4 * cap + n] = yn1 * inv_l;
        wgt[2 * cap + n] = wgt[5 * cap + n] = yn2 * inv_l;
        wgt[6 * cap + n] = wgt[7 * cap + n] = wgt[8 * cap + n] = 0.0;
        a.sel[n] = pos;
        Lirow_g[n] = inv_l;
        a.L[tri_off(n) + n] = l;
      }
    }
    if (rk == owner) {  // row n of L = [c, l] (c replicated), diagonal of Li
      const int o = own_off(qn, owner);
      const bool global_copy = cluster() == 0;
      for (int j = tid; j < n; j += kTA) {
        sh.Lown[o + j] = sh.c1[j];
        if (global_copy) a.L[tri_off(n) + j] = sh.c1[j];
      }
      if (tid == 0) {
        sh.Lown[o + n] = l;
        sh.Liown[o + n] = inv_l;
      }
    }
    wait(kMbW);
    if (kOv) bar_ov();  // the next group's scan has read the old weights
    for (int j = tid; j < n; j += kTA) {  // x' = x + Li[n][j] y_n, compensated (comp_add)
      const double lij = sh.u_all[j] * neg_inv_l;
      double h0 = sh.wh[0][j], l0 = sh.wl[0][j], h1 = sh.wh[1][j], l1 = sh.wl[1][j];
      double h2 = sh.wh[2][j], l2 = sh.wl[2][j];
      sh.wx[j] = comp_add(h0, l0, lij, yn0);
      sh.wy[j] = comp_add(h1, l1, lij, yn1);
      sh.wz[j] = comp_add(h2, l2, lij, yn2);
      sh.wh[0][j] = h0;
      sh.wl[0][j] = l0;
      sh.wh[1][j] = h1;
      sh.wl[1][j] = l1;
      sh.wh[2][j] = h2;
      sh.wl[2][j] = l2;
      if (rk == owner) sh.Liown[own_off(qn, owner) + j] = lij;
      if (j % kClusterCTAs == rk && cluster() == 0) {  // my columns -> global copies
        wgt[j] = sh.wx[j];
        wgt[cap + j] = sh.wy[j];
        wgt[2 * cap + j] = sh.wz[j];
        wgt[3 * cap + j] = h0;
        wgt[4 * cap + j] = h1;
        wgt[5 * cap + j] = h2;
        wgt[6 * cap + j] = l0;
        wgt[7 * cap + j] = l1;
        wgt[8 * cap + j] = l2;
        Lirow_g[j] = lij;
      }
    }
    if (tid == 0) {
      sh.wx[n] = sh.wh[0][n] = yn0 * inv_l;
      sh.wy[n] = sh.wh[1][n] = yn1 * inv_l;
      sh.wz[n] = sh.wh[2][n] = yn2 * inv_l;
      sh.wl[0][n] = sh.wl[1][n] = sh.wl[2][n] = 0.0;
    }
    n += 1;
    sync_a<kOv>();
    pc.mark(5);
    return kAccepted;
  }
};

// ================================================================== driver
// Next candidate after a rejection: eligible arg-max over the stored group
// errors (rare path; every CTA scans the whole group redundantly).
__device__ Best rescan_candidate(const rbf_gcb_args& a, const LoopScratch& s, Common& cm,
                                 const int* gpos, int card) {
  Best b{-1.0, kNone};
  for (int t = threadIdx.x; t < card; t += kLoopThreads) {
    const int pos = gpos ? __ldg(gpos + t) : t;
    if (__ldcg(reinterpret_cast<const unsigned char*>(a.inel) + pos)) continue;
    const double e = __ldcg(s.err + t);
    if (better(e, pos, b.err, b.pos)) b = Best{e, pos};
  }
  __syncthreads();
  b = cta_best(cm, b, 1);
  if (threadIdx.x == 0) cm.bcast[1] = b;
  __syncthreads();
  return cm.bcast[1];
}

// Gather the boundary into group order (gpt/gdisp), once per launch.
__device__ void gather_groups(const rbf_gcb_args& a, const LoopScratch& s) {
  const int G = gridDim.x;
  for (int t = blockIdx.x * kLoopThreads + threadIdx.x; t < a.nb; t += G * kLoopThreads) {
    const int p = __ldg(a.group_pos + t);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      s.gpt[3 * (int64_t)t + c] = __ldg(a.points + 3 * (int64_t)p + c);
      s.gdisp[3 * (int64_t)t + c] = __ldg(a.disp + 3 * (int64_t)p + c);
    }
  }
}

// selection.py:198-212: argmax |d| (first occurrence), then twice
// argmax dmin with dmin = min(dmin, |P - P_next|); norms are
// sqrt((x0*x0 + x1*x1) + x2*x2), numpy's bits for a (n, 3) row norm.
template <class Path>
__device__ void device_seeds(Path& P, const rbf_gcb_args& a, const LoopScratch& s, int seeds[3],
                             int& par) {
  const int nb = a.nb, G = gridDim.x;
  const int lo = (int)((int64_t)nb * blockIdx.x / G), hi = (int)((int64_t)nb * (blockIdx.x + 1) / G);
  Best b{-1.0, kNone};
  for (int i = lo + threadIdx.x; i < hi; i += kLoopThreads) {
    const double m = residual_norm(__ldg(a.disp + 3 * (int64_t)i), __ldg(a.disp + 3 * (int64_t)i + 1),
                                   __ldg(a.disp + 3 * (int64_t)i + 2), 0.0, 0.0, 0.0);
    if (better(m, i, b.err, b.pos)) b = Best{m, i};
  }
  P.publish(cta_best(P.cm(), b, 0), 0, par);
  P.gather(par, 1);
  par ^= 1;
  seeds[0] = P.cm().bcast[0].pos;
  for (int q = 1; q < 3; ++q) {
    const int p = seeds[q - 1];
    const double qx = __ldg(a.points + 3 * (int64_t)p), qy = __ldg(a.points + 3 * (int64_t)p + 1),
                 qz = __ldg(a.points + 3 * (int64_t)p + 2);
    Best bb{-1.0, kNone};
    for (int i = lo + threadIdx.x; i < hi; i += kLoopThreads) {
      double d = residual_norm(__ldg(a.points + 3 * (int64_t)i), __ldg(a.points + 3 * (int64_t)i + 1),
                               __ldg(a.points + 3 * (int64_t)i + 2), qx, qy, qz);
      if (q == 2) d = fmin(s.dmin[i], d);
      s.dmin[i] = d;
      if (better(d, i, bb.err, bb.pos)) bb = Best{d, i};
    }
    __syncthreads();
    P.publish(cta_best(P.cm(), bb, 0), 0, par);
    P.gather(par, 1);
    par ^= 1;
    seeds[q] = P.cm().bcast[0].pos;
  }
}

template <class Path, class Clock>
__device__ void gcb_driver(Path& P, const rbf_gcb_args& a, const LoopScratch& s, Clock& pc,
                           int self_mode) {
  const int tid = threadIdx.x;
  const bool leader = blockIdx.x == 0 && tid == 0;
  rbf_gcb_state* st = a.state;
  Common& cm = P.cm();

  int n = __ldcg(&st->n);
  int k = __ldcg(&st->k);
  int streak_ok = __ldcg(&st->streak_ok);
  int streak_noadd = __ldcg(&st->streak_noadd);
  int nrec = __ldcg(&st->n_records);
  int done_loop = __ldcg(&st->done_loop);
  double t2_carry = __ldcg(&st->t2_carry);
  const int m = a.m;
  int par = 0;

  auto save = [&](int status, int want_mode, int handover = 0) {
    if (leader) {
      st->handover = handover;
      for (int i = 0; i < 16; ++i) st->phase_cycles[i] += cm.phase[i];
      st->n = n;
      st->k = k;
      st->streak_ok = streak_ok;
      st->streak_noadd = streak_noadd;
      st->n_records = nrec;
      st->done_loop = done_loop;
      st->t2_carry = t2_carry;
      st->want_mode = want_mode;
      st->status = status;
    }
  };

  // the tail launch after a one-cluster loop: proceed only if that loop
  // finished and handed its final sweep over (else the host decides)
  const bool tail = (a.flags & kFlagTailOnly) != 0;
  const int handover = tail ? __ldcg(&st->handover) : 0;
  if (tail && !((done_loop || handover) && __ldcg(&st->status) == RBF_EGROW &&
                __ldcg(&st->want_mode) == RBF_GCB_GRID))
    return;
  // the one-cluster launch queued behind the tail: continue only where the
  // tail handed a run back (or any pause that asks for this shape)
  if ((a.flags & kFlagResumeOnly) &&
      !(__ldcg(&st->status) == RBF_EGROW && __ldcg(&st->want_mode) == self_mode))
    return;
  if (!tail) {  // the final sweep and the run resolution read neither the group order nor the column copy
    gather_groups(a, s);
    P.begin(n);
  }
  P.sync();

  if (n == 0) {
    if (a.cap < 3 || a.rec_cap < 1) {
      save(RBF_EGROW, self_mode);
      return;
    }
    int seeds[3];
    device_seeds(P, a, s, seeds, par);
    pc.mark(7);
    // seed appends (selection.py:288-297): no near-duplicate guard, NotPD propagates
    for (int q = 0; q < 3; ++q) {
      double p2 = 0.0;
      const int res = P.append(seeds[q], n, false, &p2);
      if (res != kAccepted) {
        if (leader) {
          st->fail_row = n;
          st->fail_pivot2 = p2;
        }
        save(RBF_ENOTPD, self_mode);
        return;
      }
    }
    k = 3;
    streak_ok = streak_noadd = 0;
    nrec = 0;
    t2_carry = 0.0;
  }

  int gk = k % m;
  // the tail's whole-boundary pass is still valid when its run closes the loop
  // (same weights): the final sweep then folds its per-group bests
  const Best* swept = nullptr;
  if (tail && handover && !done_loop) {
    // A run of groups within tolerance handed over by a one-cluster launch:
    // the weights stay fixed until the next append, so one whole-boundary
    // pass gives every following group's (max error, lowest position); the
    // groups are then taken in order exactly as the loop below would, until
    // the run reaches m (loop done: the final sweep follows) or a group
    // exceeds the tolerance (hand back: the one-cluster launch rescans it
    // and appends). The pass time is the first resolved record's t1.
    const uint64_t t_a = leader_timer();
    P.scan(nullptr, a.points, a.disp, a.nb, n, par);
    P.gather(par, 1);
    par ^= 1;
    Best* gbest = reinterpret_cast<Best*>(s.gpt);  // 24 nb bytes >= 16 m
    for (int g = blockIdx.x; g < m; g += gridDim.x) {
      const int lo = P.group_off(g), hi = P.group_off(g + 1);
      Best b{-1.0, kNone};
      for (int t = lo + (int)threadIdx.x; t < hi; t += kLoopThreads) {
        const int pos = __ldg(a.group_pos + t);
        const double e = __ldcg(s.err + pos);
        if (better(e, pos, b.err, b.pos)) b = Best{e, pos};
      }
      b = cta_best(cm, b, 0);
      if (threadIdx.x == 0) gbest[g] = b;
      __syncthreads();
    }
    P.sync();
    // the walk below visits the groups one after another: their bests come
    // from shared memory, not one dependent L2 load per group (~40 % of the
    // launch, profiles/r02_ncu_summary.md)
    Best* gcache = P.best_cache();
    const int ncache = m < P.best_cache_cap() ? m : P.best_cache_cap();
    for (int g = tid; g < ncache; g += kLoopThreads) gcache[g] = Best{__ldcg(&gbest[g].err), __ldcg(&gbest[g].pos)};
    __syncthreads();
    const uint64_t t_b = leader_timer();
    bool first = true;
    while (true) {
      if (nrec >= a.rec_cap) {
        save(RBF_EGROW, handover);
        return;
      }
      const Best gb = gk < ncache ? gcache[gk] : Best{__ldcg(&gbest[gk].err), __ldcg(&gbest[gk].pos)};
      if (gb.err > a.tol) {  // the run ends here: back to the one-cluster loop
        save(RBF_EGROW, handover);
        return;
      }
      if (leader) {
        rbf_gcb_record rec;
        rec.group = gk;
        rec.node_pos = gb.pos;
        rec.added = 0;
        rec.n_before = n;
        rec.local_max = gb.err;
        rec.t1_s = first ? (double)(t_b - t_a) * 1e-9 : 0.0;
        rec.t2_s = t2_carry;
        a.records[nrec] = rec;
      }
      first = false;
      nrec += 1;
      t2_carry = 0.0;
      streak_noadd += 1;
      streak_ok += 1;
      if (streak_ok >= m) {
        done_loop = 1;
        swept = gbest;
        break;
      }
      if (streak_noadd >= m) {
        save(RBF_ESTALL, self_mode);
        return;
      }
      k += 1;
      gk = gk + 1 == m ? 0 : gk + 1;
    }
  }

  const int card_max = (a.nb + m - 1) / m;
  int ov_group = -1;  // group whose scan ran during the last append (MsgPath)
  while (!done_loop) {
    if (n >= a.max_supports) {
      done_loop = 1;
      break;
    }
    // one-cluster paths hand over to the whole-GPU grid once a group scan
    // (card x n pairs on 16 SMs) costs more than the grid's extra barriers
    if (self_mode != RBF_GCB_GRID && self_mode != RBF_GCB_CLUSTER &&
        (int64_t)card_max * n > kClusterScanPairs) {
      save(RBF_EGROW, RBF_GCB_GRID);
      return;
    }
    if (n >= Path::kMaxN - 1) {  // beyond this path's resident capacity
      const bool big_scans = (int64_t)card_max * n > kSmemScanPairs;
      // past the shared-memory paths the factor passes need every SM's
      // bandwidth: SMEM hands over to the grid (CLUSTER only when forced)
      save(RBF_EGROW, self_mode == RBF_GCB_MSG ? (big_scans ? RBF_GCB_GRID : RBF_GCB_SMEM)
                      : self_mode == RBF_GCB_SMEM ? RBF_GCB_GRID : self_mode);
      return;
    }
    if (n >= a.cap || nrec >= a.rec_cap) {
      save(RBF_EGROW, self_mode);
      return;
    }
    const uint64_t t_a = leader_timer();
    const int gi = gk;  // == k % m, advanced with k (no division per iteration)
    const int off = P.group_off(gi);
    const int card = P.group_off(gi + 1) - off;
    const int* gpos = a.group_pos + off;
    pc.mark(6);
    if (ov_group == gi)  // rows evaluated during the last append
      P.scan_ov(gpos, s.gdisp + 3 * (int64_t)off, card, n, par);
    else
      P.scan(gpos, s.gpt + 3 * (int64_t)off, s.gdisp + 3 * (int64_t)off, card, n, par);
    ov_group = -1;
    P.gather(par, 2);
    pc.mark(0);
    pc.count(10);
    par ^= 1;
    const Best bu = cm.bcast[0];
    Best cand = cm.bcast[1];
    const uint64_t t_b = leader_timer();
    const int n_before = n;
    const double local_max = bu.err;
    bool added = false;
    int added_pos = -1;
    if (local_max > a.tol) {
      // the next group's scan runs during the append when it fits
      const int gn = gk + 1 == m ? 0 : gk + 1;
      int ov_g = -1, ov_off = 0, ov_card = 0;
      if (Path::kHasOv) {
        ov_off = P.group_off(gn);
        ov_card = P.group_off(gn + 1) - ov_off;
        if (P.ov_fits(ov_card, n)) ov_g = gn;
      }
      while (cand.pos != kNone && cand.err > a.tol) {
        double p2;
        const int res = ov_g >= 0 ? P.append_ov(cand.pos, n, true, &p2, ov_off, ov_card)
                                  : P.append(cand.pos, n, true, &p2);
        pc.count(9);
        if (res == kAccepted) {
          added = true;
          added_pos = cand.pos;
          ov_group = ov_g;
          break;
        }
        if (tid == 0) {
          a.inel[cand.pos] = 1;
          __threadfence();
        }
        P.sync();  // rare path: every CTA's errors (global) visible
        cand = rescan_candidate(a, s, cm, gpos, card);
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
        save(RBF_ESTALL, self_mode);
        return;
      }
      if ((a.flags & kFlagTailSweep) && self_mode != RBF_GCB_GRID && streak_ok >= kStreakHandover &&
          m >= 2 * kStreakHandover) {  // likely the closing run: the tail launch resolves it
        k += 1;
        save(RBF_EGROW, RBF_GCB_GRID, self_mode);
        return;
      }
    } else {
      streak_noadd = 0;
      streak_ok = 0;
    }
    k += 1;
    gk = gk + 1 == m ? 0 : gk + 1;
  }

  // RBF_GCB_NO_SWEEP: the caller runs the final sweep itself (multi-GPU: one
  // boundary shard per rank, multi.py); the loop ends here
  if (a.flags & RBF_GCB_NO_SWEEP) {
    if (leader) {
      st->final_max = -1.0;
      st->final_pos = -1;
    }
    save(1, self_mode);
    return;
  }
  // final verification sweep (selection.py:388-412), natural order: one
  // cluster's 16 SMs would take Nb x n pairs at 1/9 of the GPU, so the
  // one-cluster paths hand it to the tail launch queued behind them
  if ((a.flags & kFlagTailSweep) && self_mode != RBF_GCB_GRID) {
    save(RBF_EGROW, RBF_GCB_GRID);
    return;
  }
  if (nrec >= a.rec_cap) {
    save(RBF_EGROW, self_mode);
    return;
  }
  const uint64_t t_a = leader_timer();
  pc.mark(6);
  Best bu{-1.0, kNone};
  if (swept) {  // the groups partition the boundary: the best group best is the sweep's
    if (blockIdx.x == 0) {
      Best b{-1.0, kNone};
      for (int g = tid; g < m; g += kLoopThreads) {
        const Best q{__ldcg(&swept[g].err), __ldcg(&swept[g].pos)};
        if (better(q.err, q.pos, b.err, b.pos)) b = q;
      }
      bu = cta_best(cm, b, 0);
    }
  } else {
    P.scan(nullptr, a.points, a.disp, a.nb, n, par);
    P.gather(par, 1);
    par ^= 1;
    bu = cm.bcast[0];
  }
  pc.mark(8);
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
  save(1, self_mode);
}

extern __shared__ __align__(16) unsigned char g_smem[];

template <class Team, bool kPh>
__device__ void run_global(const rbf_gcb_args& a, const LoopScratch& s, Team team, int mode) {
  GlobalShared& sh = *reinterpret_cast<GlobalShared*>(g_smem);
  PhaseClockT<kPh> pc;
  pc.start(sh.cm.phase);
  GlobalPath<Team, PhaseClockT<kPh>> P{a, s, sh, team, 1.0 / a.radius, pc};
  gcb_driver(P, a, s, pc, mode);
}

// kPh: with the per-phase clock (rbf_gcb_args.flags & RBF_GCB_PHASES)
template <bool kPh>
__global__ void __launch_bounds__(kLoopThreads, 1) gcb_cluster_kernel(rbf_gcb_args a, LoopScratch s) {
  run_global<ClusterTeam, kPh>(a, s, ClusterTeam{}, RBF_GCB_CLUSTER);
}

template <bool kPh>
__global__ void __launch_bounds__(kLoopThreads, 1) gcb_grid_kernel(rbf_gcb_args a, LoopScratch s) {
  run_global<GridTeam, kPh>(a, s, GridTeam{s.bar, s.fault}, RBF_GCB_GRID);
}

template <bool kPh>
__global__ void __launch_bounds__(kLoopThreads, 1) gcb_smem_kernel(rbf_gcb_args a, LoopScratch s) {
  SmemShared& sh = *reinterpret_cast<SmemShared*>(g_smem);
  PhaseClockT<kPh> pc;
  pc.start(sh.cm.phase);
  SmemPath<PhaseClockT<kPh>> P{a, s, sh, 1.0 / a.radius, pc};
  gcb_driver(P, a, s, pc, RBF_GCB_SMEM);
  P.finish();
}

template <bool kPh>
__global__ void __launch_bounds__(kLoopThreads, 1) gcb_msg_kernel(rbf_gcb_args a, LoopScratch s) {
  MsgShared& sh = *reinterpret_cast<MsgShared*>(g_smem);
  PhaseClockT<kPh> pc;
  pc.start(sh.cm.phase);
  MsgPath<PhaseClockT<kPh>> P{a, s, sh, 1.0 / a.radius, pc, 0u, 0u};
  P.tmem_alloc();
  gcb_driver(P, a, s, pc, RBF_GCB_MSG);
  P.finish();
  P.tmem_free();
}

// Kernel attributes (dynamic shared memory, non-portable cluster size) are
// per function and device: set them once per process instead of on every
// launch (a host call each, on the path before the first loop launch).
static cudaError_t func_attrs_once(const void* fn, size_t smem, bool cluster) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({fn, dev})) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess && cluster) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e == cudaSuccess) done.insert({fn, dev});
  return e;
}

// The whole-GPU launch queued behind a one-cluster launch: the final sweep of
// a finished loop, or the resolution of a run of groups within tolerance
// (gcb_driver); it returns at once otherwise.
static cudaError_t launch_tail(const rbf_gcb_args& a, LoopScratch& s, int ctas, bool ph, cudaStream_t st) {
  rbf_gcb_args t = a;
  t.flags = (a.flags & 0xffff) | kFlagTailOnly;
  t.mode = RBF_GCB_GRID;
  const size_t smem = sizeof(GlobalShared);
  auto grid_kernel = ph ? gcb_grid_kernel<true> : gcb_grid_kernel<false>;
  cudaError_t e = func_attrs_once((const void*)grid_kernel, smem, false);
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeCooperative;
  at.val.cooperative = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(kLoopThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, grid_kernel, t, s);
}

static int resolve_mode(int mode, int nb, int m) {
  if (mode != RBF_GCB_AUTO) return mode;
  const int card = (nb + m - 1) / m;
  return card <= kAutoClusterMaxCard ? RBF_GCB_MSG : RBF_GCB_GRID;
}

static cudaError_t launch_cluster(const void* fn, rbf_gcb_args& a, LoopScratch& s, size_t smem,
                                  cudaStream_t st, int nclusters = 1) {
  cudaError_t e = func_attrs_once(fn, smem, true);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kClusterCTAs * nclusters);
  cfg.blockDim = dim3(kLoopThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kClusterCTAs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;  // several clusters wait on each other
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = nclusters > 1 ? 2 : 1;
  void* args[] = {&a, &s};
  return cudaLaunchKernelExC(&cfg, fn, args);
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
  if (mode < RBF_GCB_AUTO || mode > RBF_GCB_MSG) return set_error(RBF_EARG, "bad mode %d", mode);
  int dev = 0;
  RBF_CUDA_TRY(cudaGetDevice(&dev));
  const int r = resolve_mode(mode, nb, m);
  const int sms = sm_count(dev);
  if (sms <= 0) return set_error(RBF_ECUDA, "no CUDA device");
  // scratch is sized for the widest team so a run can switch paths
  if (ctas_host) *ctas_host = sms;
  if (resolved_mode_host) *resolved_mode_host = r;
  return RBF_OK;
}

extern "C" size_t rbf_gcb_scratch_bytes(int32_t nb, int32_t cap, int32_t ctas) {
  size_t total = 0;
  carve(nullptr, nb, cap, ctas, &total);
  return total;
}

// Persisting-L2 set-aside for the L2 path (0: unavailable or disabled with
// RBF_L2_PERSIST=0). The device limit is raised once, to the device maximum.
static size_t l2_persist_bytes() {
  static size_t bytes = [] {
    const char* e = getenv("RBF_L2_PERSIST");
    if (e && e[0] == '0') return (size_t)0;
    int dev = 0, persist = 0, window = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return (size_t)0;
    cudaDeviceGetAttribute(&persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    if (persist <= 0 || window <= 0) return (size_t)0;
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)persist) != cudaSuccess) {
      cudaGetLastError();
      return (size_t)0;
    }
    return (size_t)(persist < window ? persist : window);
  }();
  return bytes;
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
  rbf_gcb_args acopy = a;
  acopy.flags &= 0xffff;
  const bool ph = (a.flags & RBF_GCB_PHASES) != 0;
  // one-cluster paths: the final sweep runs in a whole-GPU launch queued
  // right behind (it returns at once unless the loop finished)
  const bool tail = (mode == RBF_GCB_MSG || mode == RBF_GCB_SMEM) && !(a.flags & RBF_GCB_NO_TAIL);
  // with runs handed to the tail (m >= 2 kStreakHandover), a second
  // one-cluster launch and a second tail are queued too, so a run that ends
  // in an append resumes without a host round trip
  const int rounds = tail && a.m >= 2 * kStreakHandover ? 2 : 1;
  if (mode == RBF_GCB_MSG || mode == RBF_GCB_SMEM) {
    int ncl = 1;
    if (mode == RBF_GCB_MSG) {
      int dev = 0;
      RBF_CUDA_TRY(cudaGetDevice(&dev));
      const int max_cl = sm_count(dev) / kClusterCTAs;
      ncl = a.clusters > 0 ? a.clusters : kMsgDefaultClusters;
      ncl = ncl < 1 ? 1 : (ncl > max_cl ? max_cl : (ncl > 16 ? 16 : ncl));
    }
    if (tail) acopy.flags |= kFlagTailSweep;
    for (int r = 0; r < rounds; ++r) {
      rbf_gcb_args x = acopy;
      if (r > 0) x.flags |= kFlagResumeOnly;
      // every MSG launch counts its cross-cluster publications from 0
      // (MsgPath::gathers): clear the sequence words before each one
      if (mode == RBF_GCB_MSG) RBF_CUDA_TRY(cudaMemsetAsync(s.xseq, 0, sizeof(unsigned) * 2 * 16, st));
      if (mode == RBF_GCB_MSG)
        RBF_CUDA_TRY(launch_cluster(ph ? (const void*)gcb_msg_kernel<true> : (const void*)gcb_msg_kernel<false>,
                                    x, s, sizeof(MsgShared), st, ncl));
      else
        RBF_CUDA_TRY(launch_cluster(ph ? (const void*)gcb_smem_kernel<true> : (const void*)gcb_smem_kernel<false>,
                                    x, s, sizeof(SmemShared), st));
      if (tail) RBF_CUDA_TRY(launch_tail(a, s, ctas, ph, st));
    }
  } else if (mode == RBF_GCB_CLUSTER) {
    RBF_CUDA_TRY(launch_cluster(ph ? (const void*)gcb_cluster_kernel<true> : (const void*)gcb_cluster_kernel<false>,
                                acopy, s, sizeof(GlobalShared), st));
  } else {
    const size_t smem = sizeof(GlobalShared);
    auto grid_kernel = ph ? gcb_grid_kernel<true> : gcb_grid_kernel<false>;
    RBF_CUDA_TRY(func_attrs_once((const void*)grid_kernel, smem, false));
    // Li is read twice per append (c0 = Li row, c = c0 + Li r): keep its first
    // persisting-L2 share resident (an access-policy window on this launch),
    // while L and the column copy stream from HBM. rbf_l2_release() returns
    // the lines to normal once the selection is over.
    cudaLaunchAttribute attrs[2];
    attrs[0].id = cudaLaunchAttributeCooperative;
    attrs[0].val.cooperative = 1;
    int nattr = 1;
    const size_t persist = l2_persist_bytes();
    if (persist > 0) {
      const size_t li_bytes = sizeof(double) * (size_t)a.cap * (a.cap + 1) / 2;
      attrs[1].id = cudaLaunchAttributeAccessPolicyWindow;
      attrs[1].val.accessPolicyWindow.base_ptr = a.Li;
      attrs[1].val.accessPolicyWindow.num_bytes = li_bytes < persist ? li_bytes : persist;
      attrs[1].val.accessPolicyWindow.hitRatio = 1.0f;
      attrs[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      attrs[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      nattr = 2;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(kLoopThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attrs;
    cfg.numAttrs = nattr;
    RBF_CUDA_TRY(cudaLaunchKernelEx(&cfg, grid_kernel, acopy, s));
  }
  return RBF_OK;
}

extern "C" int rbf_l2_release(void) {
  if (l2_persist_bytes() > 0) RBF_CUDA_TRY(cudaCtxResetPersistingL2Cache());
  return RBF_OK;
}
