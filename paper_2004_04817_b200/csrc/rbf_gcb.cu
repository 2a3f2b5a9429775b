// Device-resident GCB / greedy selection loop (replaces reference
// selection.py:274-421 `_gcb_run`, statement for statement; see
// SURVEY.md Appendix A for the exact semantics reproduced here).
//
// One cooperative persistent kernel, one 512-thread CTA per SM. Every CTA
// runs the same control flow: decisions (arg-max, accept/reject, streaks,
// termination) are recomputed redundantly by every CTA from the same
// global data in the same order, so they agree bit for bit and the only
// synchronisation is a grid barrier between data-parallel phases:
//
//   scan   group errors + (err, lowest id) arg-max partials         | B1
//   append row phi(|p - s_j|/R) in shared memory (each CTA), then
//          c0 = Li row                                               | B2
//          r  = row - L c0                                           | B3
//          c  = c0 + Li r, partial sums c.c and c.y                  | B4
//          pivot^2 = 1 - c.c; l; y_n = (d - c.y)/l;
//          u = Li^T c, v = Li^T y  ->  Li[n] = -u/l, weights v + Li[n] y_n,
//          L[n] = [c, l]                                              | B5
//
// The host only computes what must match numpy bit for bit (the PCG64
// partition, selection.py:177-185, and the seeds, selection.py:198-212)
// and reads the records once at the end.
#include <cmath>
#include <cstdint>

#include "rbf_common.cuh"
#include "rbf_internal.h"
#include "rbf_tri.cuh"

namespace rbf {

constexpr int kLoopThreads = 512;
constexpr int kLoopWarps = kLoopThreads / 32;
constexpr int kRowSmemMax = 24576;  // supports held in the shared-memory row
constexpr int kSupStride = 8;       // doubles per support record

struct LoopScratch {
  GridBarrier* bar;
  int* fault;
  Best* part;    // [ctas][2]: unrestricted, eligible-only
  double* red;   // [ctas][4]: c.c, c.y(3)
  double* err;   // [nb]   errors of the group being scanned
  double* c0;    // [cap]
  double* r;     // [cap]
  double* c1;    // [cap]
};

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

static LoopScratch carve(void* base, int nb, int cap, int ctas, size_t* total) {
  char* p = static_cast<char*>(base);
  size_t off = 0;
  LoopScratch s{};
  auto take = [&](size_t bytes) {
    char* q = p ? p + off : nullptr;
    off += align256(bytes);
    return q;
  };
  s.bar = reinterpret_cast<GridBarrier*>(take(sizeof(GridBarrier) + sizeof(int)));
  s.fault = reinterpret_cast<int*>(s.bar ? reinterpret_cast<char*>(s.bar) + sizeof(GridBarrier) : nullptr);
  s.part = reinterpret_cast<Best*>(take(sizeof(Best) * 2 * ctas));
  s.red = reinterpret_cast<double*>(take(sizeof(double) * 4 * ctas));
  s.err = reinterpret_cast<double*>(take(sizeof(double) * (size_t)nb));
  s.c0 = reinterpret_cast<double*>(take(sizeof(double) * (size_t)cap));
  s.r = reinterpret_cast<double*>(take(sizeof(double) * (size_t)cap));
  s.c1 = reinterpret_cast<double*>(take(sizeof(double) * (size_t)cap));
  if (total) *total = off;
  return s;
}

struct Shared {
  Best wb[kLoopWarps][2];
  double wred[kLoopWarps][4];
  double red[kLoopWarps * 32 * 4];
  Best bcast[2];
  double dmin[kLoopWarps];
  double dbl[8];
};

__device__ __forceinline__ uint64_t cta0_timer() {
  return (blockIdx.x == 0 && threadIdx.x == 0) ? globaltimer_ns() : 0ull;
}

// ----------------------------------------------------------------- scan
// errors of `card` targets (positions gpos[t], or t if gpos == null) against
// the n current supports; writes err[t] and the CTA's two arg-max partials.
__device__ void scan_phase(const rbf_gcb_args& a, const LoopScratch& s, Shared& sh,
                           const int* gpos, int card, int n, double inv_r) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t total = (int64_t)gridDim.x * kLoopThreads;
  int S = 32;
  while (S > 1 && (int64_t)card * (S / 2) >= total) S >>= 1;
  while (S > 1 && S / 2 >= n) S >>= 1;
  const int64_t gthread = (int64_t)blockIdx.x * kLoopThreads + tid;
  const int64_t ngroups = total / S;
  const int64_t g = gthread / S;
  const int sub = (int)(gthread % S);
  const double2* sup = reinterpret_cast<const double2*>(a.sup);

  Best bu{-1.0, 0x7fffffff}, br{-1.0, 0x7fffffff};
  for (int64_t base = 0; base < card; base += ngroups) {
    const int64_t t = base + g;
    const bool active = t < card;
    int pos = 0;
    double px = 0.0, py = 0.0, pz = 0.0;
    if (active) {
      pos = gpos ? __ldg(gpos + t) : (int)t;
      px = __ldg(a.points + 3 * (int64_t)pos) * inv_r;
      py = __ldg(a.points + 3 * (int64_t)pos + 1) * inv_r;
      pz = __ldg(a.points + 3 * (int64_t)pos + 2) * inv_r;
    }
    double ax = 0.0, ay = 0.0, az = 0.0;
    if (active) {
      for (int j = sub; j < n; j += S) {
        const double2 q0 = __ldcg(sup + 4 * j);
        const double2 q1 = __ldcg(sup + 4 * j + 1);
        const double2 q2 = __ldcg(sup + 4 * j + 2);
        pair_accum(px, py, pz, q0.x, q0.y, q1.x, q1.y, q2.x, q2.y, ax, ay, az);
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
  bu = warp_best(bu);
  br = warp_best(br);
  if (lane == 0) {
    sh.wb[warp][0] = bu;
    sh.wb[warp][1] = br;
  }
  __syncthreads();
  if (tid == 0) {
    Best u = sh.wb[0][0], r = sh.wb[0][1];
    for (int w = 1; w < kLoopWarps; ++w) {
      u = best_of(u, sh.wb[w][0]);
      r = best_of(r, sh.wb[w][1]);
    }
    s.part[2 * blockIdx.x] = u;
    s.part[2 * blockIdx.x + 1] = r;
  }
}

// every CTA folds the per-CTA partials in CTA order (identical result everywhere)
__device__ void fold_partials(const LoopScratch& s, Shared& sh) {
  if (threadIdx.x < 32) {
    Best u{-1.0, 0x7fffffff}, r{-1.0, 0x7fffffff};
    for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) {
      const Best pu{__ldcg(&s.part[2 * b].err), __ldcg(&s.part[2 * b].pos)};
      const Best pr{__ldcg(&s.part[2 * b + 1].err), __ldcg(&s.part[2 * b + 1].pos)};
      u = best_of(u, pu);
      r = best_of(r, pr);
    }
    u = warp_best(u);
    r = warp_best(r);
    if (threadIdx.x == 0) {
      sh.bcast[0] = u;
      sh.bcast[1] = r;
    }
  }
  __syncthreads();
}

// next candidate after a rejection: eligible arg-max over the stored group
// errors (rare path; every CTA scans the group redundantly).
__device__ Best rescan_candidate(const rbf_gcb_args& a, const LoopScratch& s, Shared& sh,
                                 const int* gpos, int card) {
  Best b{-1.0, 0x7fffffff};
  for (int t = threadIdx.x; t < card; t += kLoopThreads) {
    const int pos = gpos ? __ldg(gpos + t) : t;
    if (__ldcg(reinterpret_cast<const unsigned char*>(a.inel) + pos)) continue;
    const double e = __ldcg(s.err + t);
    if (better(e, pos, b.err, b.pos)) b = Best{e, pos};
  }
  b = warp_best(b);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh.wb[threadIdx.x >> 5][1] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    Best r = sh.wb[0][1];
    for (int w = 1; w < kLoopWarps; ++w) r = best_of(r, sh.wb[w][1]);
    sh.bcast[1] = r;
  }
  __syncthreads();
  return sh.bcast[1];
}

enum AppendResult { kAccepted = 0, kRejectDup = 1, kRejectPivot = 2 };

// Bordered append of boundary position `pos` (reference core.py:153-185 via
// selection.py:288-297 / 341-356). All CTAs call it; the result is uniform.
__device__ int append_node(const rbf_gcb_args& a, const LoopScratch& s, Shared& sh, double* row,
                           int pos, int& n, bool check_dup, double inv_r, double* pivot2_out) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x;
  const double px = __ldg(a.points + 3 * (int64_t)pos), py = __ldg(a.points + 3 * (int64_t)pos + 1),
               pz = __ldg(a.points + 3 * (int64_t)pos + 2);
  // row[j] = phi(cdist(p, s_j) / R), bitwise the reference's chain; min distance
  double dmin = INFINITY;
  for (int j = tid; j < n; j += kLoopThreads) {
    const int q = __ldcg(a.sel + j);
    const double d = cdist_exact(px, py, pz, __ldg(a.points + 3 * (int64_t)q),
                                 __ldg(a.points + 3 * (int64_t)q + 1), __ldg(a.points + 3 * (int64_t)q + 2));
    row[j] = phi_exact(d, a.radius);
    dmin = fmin(dmin, d);
  }
  dmin = warp_min(dmin);
  if (lane == 0) sh.dmin[warp] = dmin;
  __syncthreads();
  if (tid == 0) {
    double m = sh.dmin[0];
    for (int w = 1; w < kLoopWarps; ++w) m = fmin(m, sh.dmin[w]);
    sh.dbl[0] = m;
  }
  __syncthreads();
  if (check_dup && n > 0 && sh.dbl[0] < a.dup_dist) return kRejectDup;

  const int gw = blockIdx.x * kLoopWarps + warp, nw = G * kLoopWarps;
  // c0 = Li row
  tri_rows<1>(a.Li, n, [&](int j, int) { return row[j]; },
              [&](int i, const double* acc) { s.c0[i] = acc[0]; }, gw, nw, lane);
  grid_sync(s.bar, G, s.fault);
  // r = row - L c0
  tri_rows<1>(a.L, n, [&](int j, int) { return __ldcg(s.c0 + j); },
              [&](int i, const double* acc) { s.r[i] = row[i] - acc[0]; }, gw, nw, lane);
  grid_sync(s.bar, G, s.fault);
  // c = c0 + Li r, with per-warp partial sums of c.c and c.y
  double pcc = 0.0, pcy0 = 0.0, pcy1 = 0.0, pcy2 = 0.0;
  tri_rows<1>(a.Li, n, [&](int j, int) { return __ldcg(s.r + j); },
              [&](int i, const double* acc) {
                const double c = __ldcg(s.c0 + i) + acc[0];
                s.c1[i] = c;
                pcc = fma(c, c, pcc);
                pcy0 = fma(c, __ldcg(a.y + 3 * (int64_t)i), pcy0);
                pcy1 = fma(c, __ldcg(a.y + 3 * (int64_t)i + 1), pcy1);
                pcy2 = fma(c, __ldcg(a.y + 3 * (int64_t)i + 2), pcy2);
              },
              gw, nw, lane);
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
  grid_sync(s.bar, G, s.fault);
  if (tid < 4) {
    double t = 0.0;
    for (int b = 0; b < G; ++b) t += __ldcg(s.red + 4 * b + tid);
    sh.dbl[1 + tid] = t;
  }
  __syncthreads();
  const double cc = sh.dbl[1];
  const double pivot2 = 1.0 - cc;  // row[n] = phi(0) = 1 exactly
  *pivot2_out = pivot2;
  __syncthreads();
  if (!(pivot2 > 0.0)) return kRejectPivot;
  const double l = sqrt(pivot2);
  const double yn0 = (__ldg(a.disp + 3 * (int64_t)pos) - sh.dbl[2]) / l;
  const double yn1 = (__ldg(a.disp + 3 * (int64_t)pos + 1) - sh.dbl[3]) / l;
  const double yn2 = (__ldg(a.disp + 3 * (int64_t)pos + 2) - sh.dbl[4]) / l;
  // u = Li^T c, v = Li^T y -> new Li row, new L row, refreshed weights
  double* Lrow = a.L + tri_off(n);
  double* Lirow = a.Li + tri_off(n);
  tri_cols<4, kLoopWarps>(
      a.Li, n,
      [&](int i, int c) {
        return c == 0 ? __ldcg(s.c1 + i) : __ldcg(a.y + 3 * (int64_t)i + (c - 1));
      },
      (int)blockIdx.x, G, sh.red, [&](int j, const double* sum) {
        const double lij = -sum[0] / l;
        Lirow[j] = lij;
        Lrow[j] = __ldcg(s.c1 + j);
        double* w = a.sup + (int64_t)kSupStride * j;
        w[3] = fma(lij, yn0, sum[1]);
        w[4] = fma(lij, yn1, sum[2]);
        w[5] = fma(lij, yn2, sum[3]);
      });
  if (blockIdx.x == 0 && tid == 0) {
    Lirow[n] = 1.0 / l;
    Lrow[n] = l;
    a.y[3 * (int64_t)n] = yn0;
    a.y[3 * (int64_t)n + 1] = yn1;
    a.y[3 * (int64_t)n + 2] = yn2;
    double* w = a.sup + (int64_t)kSupStride * n;
    w[0] = px * inv_r;
    w[1] = py * inv_r;
    w[2] = pz * inv_r;
    w[3] = yn0 / l;
    w[4] = yn1 / l;
    w[5] = yn2 / l;
    w[6] = 0.0;
    w[7] = 0.0;
    a.sel[n] = pos;
  }
  if (tid == 0) a.inel[pos] = 1;
  n += 1;
  grid_sync(s.bar, G, s.fault);
  return kAccepted;
}

__global__ void __launch_bounds__(kLoopThreads, 1) gcb_kernel(rbf_gcb_args a, LoopScratch s) {
  extern __shared__ double row[];
  __shared__ Shared sh;
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

  auto save = [&](int status) {
    if (leader) {
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
    // seeds (selection.py:288-297): no near-duplicate guard, NotPD propagates
    if (a.cap < 3 || a.rec_cap < 1) {
      save(RBF_EGROW);
      return;
    }
    for (int q = 0; q < 3; ++q) {
      double p2 = 0.0;
      const int res = append_node(a, s, sh, row, a.seeds[q], n, false, inv_r, &p2);
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
    const uint64_t t_a = cta0_timer();
    const int gi = k % m;
    const int off = __ldg(a.group_off + gi);
    const int card = __ldg(a.group_off + gi + 1) - off;
    const int* gpos = a.group_pos + off;
    scan_phase(a, s, sh, gpos, card, n, inv_r);
    grid_sync(s.bar, gridDim.x, s.fault);
    fold_partials(s, sh);
    const Best bu = sh.bcast[0];
    Best cand = sh.bcast[1];
    const uint64_t t_b = cta0_timer();
    const int n_before = n;
    const double local_max = bu.err;
    bool added = false;
    int added_pos = -1;
    if (local_max > a.tol) {
      while (cand.pos != 0x7fffffff && cand.err > a.tol) {
        double p2;
        const int res = append_node(a, s, sh, row, cand.pos, n, true, inv_r, &p2);
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
    const uint64_t t_c = cta0_timer();
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
  const uint64_t t_a = cta0_timer();
  scan_phase(a, s, sh, nullptr, a.nb, n, inv_r);
  grid_sync(s.bar, gridDim.x, s.fault);
  fold_partials(s, sh);
  const Best bu = sh.bcast[0];
  const uint64_t t_b = cta0_timer();
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

}  // namespace rbf

using namespace rbf;

extern "C" int rbf_device_info(int device, int* sm_count_host, int* loop_ctas_host) {
  int sms = sm_count(device);
  if (sms <= 0) return set_error(RBF_ECUDA, "no CUDA device %d", device);
  if (sm_count_host) *sm_count_host = sms;
  int per_sm = 0;
  RBF_CUDA_TRY(cudaFuncSetAttribute(gcb_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kRowSmemMax * (int)sizeof(double)));
  RBF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gcb_kernel, kLoopThreads,
                                                             kRowSmemMax * sizeof(double)));
  if (per_sm < 1) return set_error(RBF_ECUDA, "selection kernel does not fit on an SM");
  if (loop_ctas_host) *loop_ctas_host = sms;  // one CTA per SM
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
  int dev = 0;
  RBF_CUDA_TRY(cudaGetDevice(&dev));
  int sms = 0, ctas = 0;
  int rc = rbf_device_info(dev, &sms, &ctas);
  if (rc != RBF_OK) return rc;
  size_t need = 0;
  LoopScratch s = carve(a.scratch, a.nb, a.cap, ctas, &need);
  if (a.scratch_bytes < need) return set_error(RBF_EARG, "scratch too small (%zu < %zu)", a.scratch_bytes, need);
  cudaStream_t st = as_stream(stream);
  RBF_CUDA_TRY(cudaMemsetAsync(s.bar, 0, sizeof(GridBarrier) + sizeof(int), st));
  const int rows = a.cap < kRowSmemMax ? a.cap : kRowSmemMax;
  const size_t smem = (size_t)(rows < 1 ? 1 : rows) * sizeof(double);
  rbf_gcb_args acopy = a;
  void* kargs[] = {&acopy, &s};
  RBF_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)gcb_kernel, dim3(ctas), dim3(kLoopThreads),
                                           kargs, smem, st));
  return RBF_OK;
}
