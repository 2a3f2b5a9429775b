// Volume evaluation and boundary error scan (throughput kernels).
//
// Replaces reference core.py:301-334 `_eval_displacements` (2048-row spans x
// 512-column tiles on a CPU thread pool, supports padded to a tile multiple
// by core.py:284-298) with one CUDA grid: every thread owns TPT targets in
// registers, support tiles (coordinates pre-scaled by 1/R, weights) are
// staged through shared memory and read as warp-wide broadcasts, partial
// tiles are handled by the loop bound (no padding sentinels). The summation
// order per target is support order, independent of the launch geometry, so
// any sharding of the targets reproduces single-GPU results bit for bit.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstdio>

#include "rbf_common.cuh"
#include "rbf_internal.h"

namespace rbf {

constexpr int kEvalThreads = 128;
constexpr int kEvalTPT = 4;
constexpr int kEvalTile = 128;
enum EvalMode { kModeEval = 0, kModeDeform = 1, kModeError = 2 };

// Where the supports are: element (support g, component c) of the points
// and of the weights at ptr[g * row + c * comp] -- (n, 3) AoS arrays
// (row 3, comp 1) or the selection loop's SoA buffer (row 1, comp cap);
// with n_dev the support count is read on the device (a launch queued
// behind the loop before the host knows it), and with status_dev the
// launch does nothing unless the loop finished (status 1).
struct SupLayout {
  int64_t row = 3, comp = 1;
  const int32_t* n_dev = nullptr;
  const int32_t* status_dev = nullptr;
};

template <int MODE, int kEvalThreads = rbf::kEvalThreads, int kEvalTPT = rbf::kEvalTPT,
          int kEvalTile = rbf::kEvalTile, int kMinBlocks = 4>
__global__ void __launch_bounds__(kEvalThreads, kMinBlocks)
eval_kernel(const double* __restrict__ tpts, const double* __restrict__ tdisp,
            const int64_t* __restrict__ pos, int64_t nt,
            const double* __restrict__ spts, const double* __restrict__ sw, int nsup,
            double inv_r, double* __restrict__ out, Best* __restrict__ partials, SupLayout lay = {}) {
  constexpr int kEvalTargetsPerBlock = kEvalThreads * kEvalTPT;
  __shared__ double4 s_a[kEvalTile];  // scaled x, y, z, wx
  __shared__ double2 s_b[kEvalTile];  // wy, wz
  if (lay.status_dev && __ldcg(lay.status_dev) != 1) return;
  if (lay.n_dev) nsup = __ldcg(lay.n_dev);
  const int64_t srow = lay.row, scomp = lay.comp;

  const int64_t base = (int64_t)blockIdx.x * kEvalTargetsPerBlock + threadIdx.x;
  double px[kEvalTPT], py[kEvalTPT], pz[kEvalTPT];
  double ax[kEvalTPT], ay[kEvalTPT], az[kEvalTPT];
  int64_t row[kEvalTPT];
#pragma unroll
  for (int k = 0; k < kEvalTPT; ++k) {
    int64_t idx = base + (int64_t)k * kEvalThreads;
    int64_t r = -1;
    if (idx < nt) r = (MODE == kModeError && pos) ? pos[idx] : idx;
    row[k] = r;
    if (r >= 0) {
      px[k] = tpts[3 * r] * inv_r;
      py[k] = tpts[3 * r + 1] * inv_r;
      pz[k] = tpts[3 * r + 2] * inv_r;
    } else {
      px[k] = py[k] = pz[k] = 0.0;
    }
    ax[k] = ay[k] = az[k] = 0.0;
  }

  for (int t0 = 0; t0 < nsup; t0 += kEvalTile) {
    const int cnt = min(kEvalTile, nsup - t0);
    __syncthreads();
    for (int j = threadIdx.x; j < cnt; j += kEvalThreads) {
      const int64_t g = (t0 + j) * srow;
      s_a[j] = make_double4(spts[g] * inv_r, spts[g + scomp] * inv_r, spts[g + 2 * scomp] * inv_r, sw[g]);
      s_b[j] = make_double2(sw[g + scomp], sw[g + 2 * scomp]);
    }
    __syncthreads();
#pragma unroll 2
    for (int j = 0; j < cnt; ++j) {
      const double4 a = s_a[j];
      const double2 b = s_b[j];
#pragma unroll
      for (int k = 0; k < kEvalTPT; ++k)
        pair_accum(px[k], py[k], pz[k], a.x, a.y, a.z, a.w, b.x, b.y, ax[k], ay[k], az[k]);
    }
  }

  if (MODE == kModeError) {
    Best best{-1.0, 0x7fffffff};
#pragma unroll
    for (int k = 0; k < kEvalTPT; ++k) {
      const int64_t r = row[k];
      if (r < 0) continue;
      const double e = residual_norm(tdisp[3 * r], tdisp[3 * r + 1], tdisp[3 * r + 2],
                                     ax[k], ay[k], az[k]);
      if (out) out[base + (int64_t)k * kEvalThreads] = e;
      if (better(e, (int)r, best.err, best.pos)) best = Best{e, (int)r};
    }
    best = warp_best(best);
    __shared__ Best s_best[kEvalThreads / kWarp];
    if ((threadIdx.x & 31) == 0) s_best[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
      Best b = s_best[0];
      for (int w = 1; w < kEvalThreads / kWarp; ++w) b = best_of(b, s_best[w]);
      partials[blockIdx.x] = b;
    }
  } else {
#pragma unroll
    for (int k = 0; k < kEvalTPT; ++k) {
      const int64_t r = row[k];
      if (r < 0) continue;
      if (MODE == kModeDeform) {
        out[3 * r] = tpts[3 * r] + ax[k];
        out[3 * r + 1] = tpts[3 * r + 1] + ay[k];
        out[3 * r + 2] = tpts[3 * r + 2] + az[k];
      } else {
        out[3 * r] = ax[k];
        out[3 * r + 1] = ay[k];
        out[3 * r + 2] = az[k];
      }
    }
  }
}

// One block folds the per-block (err, pos) partials in block order.
__global__ void best_reduce_kernel(const Best* __restrict__ partials, int n, double* __restrict__ result,
                                   int64_t pos_offset) {
  Best b{-1.0, 0x7fffffff};
  for (int i = threadIdx.x; i < n; i += blockDim.x) b = best_of(b, partials[i]);
  b = warp_best(b);
  __shared__ Best s[32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    Best r = s[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = best_of(r, s[w]);
    result[0] = r.err;
    result[1] = (double)(r.pos + pos_offset);
  }
}

// Fold of n (err, pos) records (pos held exactly as a double), larger error
// first, exact ties to the lowest position: the combine step of a sharded
// sweep (one record per rank, all-gathered) -- reference selection.py:231-234.
__global__ void best_fold_kernel(const double* __restrict__ recs, int64_t n, double* __restrict__ out) {
  double be = -1.0, bp = 0.0;
  bool have = false;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double e = recs[2 * i], p = recs[2 * i + 1];
    if (!have || e > be || (e == be && p < bp)) {
      be = e;
      bp = p;
      have = true;
    }
  }
  __shared__ double s_e[256], s_p[256];
  __shared__ bool s_h[256];
  s_e[threadIdx.x] = be;
  s_p[threadIdx.x] = bp;
  s_h[threadIdx.x] = have;
  __syncthreads();
  if (threadIdx.x == 0) {
    bool h = false;
    double e0 = -1.0, p0 = -1.0;
    for (int t = 0; t < (int)blockDim.x; ++t) {
      if (!s_h[t]) continue;
      if (!h || s_e[t] > e0 || (s_e[t] == e0 && s_p[t] < p0)) {
        e0 = s_e[t];
        p0 = s_p[t];
        h = true;
      }
    }
    out[0] = e0;
    out[1] = p0;
  }
}

// Launch variants of the volume kernel: 1-5 launch geometries (threads,
// targets per thread, support tile, min resident blocks), 7-8 64 x 6 (6 CTAs
// per SM; support tile 128 / 64), 10-11 short-grid shapes (128 x 2 and 64 x 4:
// more CTAs when the targets fill less than one wave). RBF_EVAL_VARIANT
// selects one for experiments (tools/eval_variants.py). The expanded pair form
// r^2 = |p|^2 + |s|^2 - 2 p.s (16 instead of 18 FP64 instructions) was removed
// in round 2: with the one-instruction clamp it is no faster than the
// difference form (19.3-20.0 vs 19.4 TFLOP/s) and less accurate.
template <int MODE, int NT, int TPT, int TILE, int MINB>
static void launch_eval_variant(const double* targets, int64_t n, const double* sp, const double* sw,
                                int ns, double inv_r, double* out, cudaStream_t s) {
  const int64_t nblk = (n + NT * TPT - 1) / (NT * TPT);
  eval_kernel<MODE, NT, TPT, TILE, MINB><<<(unsigned)nblk, NT, 0, s>>>(
      targets, nullptr, nullptr, n, sp, sw, ns, inv_r, out, nullptr);
}

template <int MODE>
static void launch_eval(int variant, const double* t, int64_t n, const double* sp, const double* sw, int ns,
                        double inv_r, double* out, cudaStream_t s) {
  switch (variant) {
    case 1: launch_eval_variant<MODE, 128, 8, 128, 2>(t, n, sp, sw, ns, inv_r, out, s); break;
    case 2: launch_eval_variant<MODE, 256, 4, 256, 2>(t, n, sp, sw, ns, inv_r, out, s); break;
    case 3: launch_eval_variant<MODE, 64, 8, 128, 4>(t, n, sp, sw, ns, inv_r, out, s); break;
    case 4: launch_eval_variant<MODE, 128, 6, 128, 3>(t, n, sp, sw, ns, inv_r, out, s); break;
    case 5: launch_eval_variant<MODE, 128, 4, 256, 4>(t, n, sp, sw, ns, inv_r, out, s); break;
    case 7: launch_eval_variant<MODE, 64, 6, 128, 6>(t, n, sp, sw, ns, inv_r, out, s); break;
    case 8: launch_eval_variant<MODE, 64, 6, 64, 6>(t, n, sp, sw, ns, inv_r, out, s); break;
    case 10: launch_eval_variant<MODE, 128, 2, 128, 8>(t, n, sp, sw, ns, inv_r, out, s); break;
    case 11: launch_eval_variant<MODE, 64, 4, 128, 6>(t, n, sp, sw, ns, inv_r, out, s); break;
    default: launch_eval_variant<MODE, 128, 4, 128, 4>(t, n, sp, sw, ns, inv_r, out, s); break;
  }
}

// Default: variant 4, 128 threads x 6 targets, 3 CTAs per SM (19.4 FP64
// TFLOP/s algorithmic on configs[1]; tools/eval_variants.py).
static int eval_variant() {
  static int v = [] {
    const char* e = getenv("RBF_EVAL_VARIANT");
    return e ? atoi(e) : 4;
  }();
  return v;
}

}  // namespace rbf

using namespace rbf;

extern "C" int rbf_eval(const double* targets, int64_t n_targets, const double* sup_points,
                        const double* sup_weights, int64_t n_sup, double radius, int deform,
                        double* out, void* stream) {
  if (n_targets < 0 || n_sup < 0) return set_error(RBF_EARG, "negative size");
  if (!(radius > 0.0)) return set_error(RBF_EARG, "radius must be positive, got %g", radius);
  if (n_sup > INT32_MAX) return set_error(RBF_EARG, "too many supports");
  if (n_targets == 0) return RBF_OK;
  if (!targets || !out || (n_sup > 0 && (!sup_points || !sup_weights)))
    return set_error(RBF_EARG, "null pointer");
  const double inv_r = 1.0 / radius;
  cudaStream_t s = as_stream(stream);
  if (deform)
    launch_eval<kModeDeform>(eval_variant(), targets, n_targets, sup_points, sup_weights, (int)n_sup, inv_r, out, s);
  else
    launch_eval<kModeEval>(eval_variant(), targets, n_targets, sup_points, sup_weights, (int)n_sup, inv_r, out, s);
  RBF_LAUNCH_CHECK("eval_kernel");
  return RBF_OK;
}

// The volume evaluation queued behind the selection loop on its stream, with
// the supports and weights read from the loop's own buffers (SoA rows 0-5 of
// rbf_gcb_args.sup, capacity `cap`) and their count from the loop state: the
// host enqueues it before it has read the loop's result, so the volume
// kernel runs while the host reads and unpacks the selection. A no-op (and
// the caller re-runs it) unless the loop finished (state->status == 1).
extern "C" int rbf_eval_loop(const double* targets, int64_t n_targets, const double* sup, int64_t cap,
                             const rbf_gcb_state* state, double radius, int deform, double* out, void* stream) {
  if (n_targets < 0 || cap < 1) return set_error(RBF_EARG, "bad size");
  if (!(radius > 0.0)) return set_error(RBF_EARG, "radius must be positive, got %g", radius);
  if (n_targets == 0) return RBF_OK;
  if (!targets || !out || !sup || !state) return set_error(RBF_EARG, "null pointer");
  SupLayout lay;
  lay.row = 1;
  lay.comp = cap;
  lay.n_dev = &state->n;
  lay.status_dev = &state->status;
  constexpr int NT = 128, TPT = 6;
  const int64_t nblk = (n_targets + NT * TPT - 1) / (NT * TPT);
  cudaStream_t s = as_stream(stream);
  if (deform)
    eval_kernel<kModeDeform, NT, TPT, 128, 3><<<(unsigned)nblk, NT, 0, s>>>(
        targets, nullptr, nullptr, n_targets, sup, sup + 3 * cap, 0, 1.0 / radius, out, nullptr, lay);
  else
    eval_kernel<kModeEval, NT, TPT, 128, 3><<<(unsigned)nblk, NT, 0, s>>>(
        targets, nullptr, nullptr, n_targets, sup, sup + 3 * cap, 0, 1.0 / radius, out, nullptr, lay);
  RBF_LAUNCH_CHECK("eval_kernel (loop supports)");
  return RBF_OK;
}

// Host targets -> host results through caller-provided device buffers, the
// targets streamed in `chunks` pieces so the host->device copy of piece k+1
// and the device->host copy of piece k-1 overlap the kernel on piece k (PCIe
// is full duplex: 48 MB each way in 1.0 ms together vs 0.87 ms alone). The
// copy and kernel streams and the events are the library's own (created
// once per device and host thread); they start after the work pending on
// `stream`, and `stream` waits for the last copy, so the caller synchronises
// `stream` before reading `host_out`. Per-target results
// are bitwise those of one rbf_eval launch.
namespace {
// Chunk kernels rotate over kPipeCompute library-owned streams so the
// partial last wave of chunk k runs beside the first wave of chunk k+1 (one
// stream serialises them: 8 chunks of 250k targets cost 8 full-wave times).
constexpr int kPipeCompute = 3;
struct PipeStreams {
  int device = -1;
  cudaStream_t in = nullptr, out = nullptr;
  cudaStream_t comp[kPipeCompute] = {};
  cudaEvent_t ev[3 * 64] = {};
};
}  // namespace

// host_targets == nullptr: the targets are already in dev_in (copied there
// ahead of time by the caller, in stream order): only kernel + D2H per chunk
template <class Launch>
static int eval_pipeline(const double* host_targets, int64_t n_targets, double* dev_in, double* dev_out,
                         double* host_out, int chunks, void* stream, Launch launch_chunk) {
  if (chunks < 1) chunks = 1;
  if (chunks > 63) chunks = 63;  // events 3c+1, 3c+2 per chunk; 191 marks the end
  static thread_local PipeStreams ps;
  int dev = 0;
  RBF_CUDA_TRY(cudaGetDevice(&dev));
  if (ps.device != dev) {
    RBF_CUDA_TRY(cudaStreamCreateWithFlags(&ps.in, cudaStreamNonBlocking));
    RBF_CUDA_TRY(cudaStreamCreateWithFlags(&ps.out, cudaStreamNonBlocking));
    for (auto& c : ps.comp) RBF_CUDA_TRY(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking));
    for (auto& e : ps.ev) RBF_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ps.device = dev;
  }
  cudaStream_t compute = as_stream(stream);
  // start the copies only after the caller's pending work (e.g. the weights)
  RBF_CUDA_TRY(cudaEventRecord(ps.ev[0], compute));
  RBF_CUDA_TRY(cudaStreamWaitEvent(ps.in, ps.ev[0], 0));
  RBF_CUDA_TRY(cudaStreamWaitEvent(ps.out, ps.ev[0], 0));
  for (auto& cs : ps.comp) RBF_CUDA_TRY(cudaStreamWaitEvent(cs, ps.ev[0], 0));
  // Chunk schedule: chunks - 1 equal pieces, then the last one halved
  // `tail` times (1/2, 1/4, .., the rest), so what runs after the final
  // host->device copy -- the last kernel (its CTAs alone on their SMs) and
  // the last device->host copy -- is a small piece.
  constexpr int64_t kBlock = 768;  // targets per volume-kernel CTA (128 x 6)
  static const int tail = [] {
    const char* e = getenv("RBF_PIPE_TAIL");
    return e ? atoi(e) : 2;
  }();
  int64_t sizes[63];
  int nchunks = 0;
  {
    int64_t step = (n_targets + chunks - 1) / chunks;
    step = (step + kBlock - 1) / kBlock * kBlock;
    int64_t lo = 0;
    while (lo < n_targets && nchunks < 63) {
      int64_t rest = n_targets - lo, cnt = std::min(step, rest);
      if (rest <= step) {  // the last piece: split it
        for (int t = 0; t < tail && nchunks < 62 && rest > 2 * kBlock; ++t) {
          const int64_t half = (rest / 2 + kBlock - 1) / kBlock * kBlock;
          sizes[nchunks++] = half;
          lo += half;
          rest -= half;
        }
        cnt = rest;
      }
      sizes[nchunks++] = cnt;
      lo += cnt;
    }
  }
  // RBF_PIPE_TRACE=1 (diagnostic): per-chunk device timeline on stderr
  static const bool trace = getenv("RBF_PIPE_TRACE") != nullptr;
  cudaEvent_t tev[4 * 63 + 1] = {};
  if (trace) {
    for (auto& e : tev) RBF_CUDA_TRY(cudaEventCreate(&e));
    RBF_CUDA_TRY(cudaEventRecord(tev[0], compute));
  }
  int64_t lo = 0;
  for (int c = 0; c < nchunks; lo += sizes[c], ++c) {
    const int64_t cnt = sizes[c];
    cudaEvent_t in_done = ps.ev[3 * c + 1], k_done = ps.ev[3 * c + 2];
    cudaStream_t cs = ps.comp[c % kPipeCompute];
    if (host_targets) {
      RBF_CUDA_TRY(cudaMemcpyAsync(dev_in + 3 * lo, host_targets + 3 * lo, 24 * cnt, cudaMemcpyHostToDevice, ps.in));
      RBF_CUDA_TRY(cudaEventRecord(in_done, ps.in));
      RBF_CUDA_TRY(cudaStreamWaitEvent(cs, in_done, 0));
    }
    const int rc = launch_chunk(dev_in + 3 * lo, cnt, dev_out + 3 * lo, cs);
    if (rc != RBF_OK) return rc;
    RBF_CUDA_TRY(cudaEventRecord(k_done, cs));
    RBF_CUDA_TRY(cudaStreamWaitEvent(ps.out, k_done, 0));
    RBF_CUDA_TRY(cudaMemcpyAsync(host_out + 3 * lo, dev_out + 3 * lo, 24 * cnt, cudaMemcpyDeviceToHost, ps.out));
    if (trace) {
      RBF_CUDA_TRY(cudaEventRecord(tev[4 * c + 1], ps.in));
      RBF_CUDA_TRY(cudaEventRecord(tev[4 * c + 2], cs));
      RBF_CUDA_TRY(cudaEventRecord(tev[4 * c + 3], ps.out));
    }
  }
  if (trace) {
    RBF_CUDA_TRY(cudaDeviceSynchronize());
    for (int c = 0; c < nchunks; ++c) {
      float h = 0.f, k = 0.f, d = 0.f;
      cudaEventElapsedTime(&h, tev[0], tev[4 * c + 1]);
      cudaEventElapsedTime(&k, tev[0], tev[4 * c + 2]);
      cudaEventElapsedTime(&d, tev[0], tev[4 * c + 3]);
      fprintf(stderr, "pipe chunk %d n=%lld h2d_end %.3f kernel_end %.3f d2h_end %.3f ms\n", c,
              (long long)sizes[c], h, k, d);
    }
    for (auto& e : tev) cudaEventDestroy(e);
  }
  RBF_CUDA_TRY(cudaEventRecord(ps.ev[3 * 63 + 2], ps.out));
  RBF_CUDA_TRY(cudaStreamWaitEvent(compute, ps.ev[3 * 63 + 2], 0));
  return RBF_OK;
}

extern "C" int rbf_eval_host(const double* host_targets, int64_t n_targets, const double* sup_points,
                             const double* sup_weights, int64_t n_sup, double radius, int deform,
                             double* dev_in, double* dev_out, double* host_out, int chunks, void* stream) {
  if (n_targets < 0 || n_sup < 0) return set_error(RBF_EARG, "negative size");
  if (!(radius > 0.0)) return set_error(RBF_EARG, "radius must be positive, got %g", radius);
  if (n_targets == 0) return RBF_OK;
  if (!host_out || !dev_in || !dev_out || (n_sup > 0 && (!sup_points || !sup_weights)))
    return set_error(RBF_EARG, "null pointer");
  return eval_pipeline(host_targets, n_targets, dev_in, dev_out, host_out, chunks, stream,
                       [&](const double* in, int64_t cnt, double* out, cudaStream_t cs) {
                         return rbf_eval(in, cnt, sup_points, sup_weights, n_sup, radius, deform, out, cs);
                       });
}

// rbf_eval_host with the supports read from a selection run's buffers on
// the device (rbf_eval_loop): the whole chunked copy / kernel / copy
// pipeline is queued behind the selection loop before the host has read
// its result. The kernels do nothing unless the loop finished; the copies
// always run.
extern "C" int rbf_eval_host_loop(const double* host_targets, int64_t n_targets, const double* sup, int64_t cap,
                                  const rbf_gcb_state* state, double radius, int deform, double* dev_in,
                                  double* dev_out, double* host_out, int chunks, void* stream) {
  if (n_targets < 0 || cap < 1) return set_error(RBF_EARG, "bad size");
  if (!(radius > 0.0)) return set_error(RBF_EARG, "radius must be positive, got %g", radius);
  if (n_targets == 0) return RBF_OK;
  if (!host_out || !dev_in || !dev_out || !sup || !state) return set_error(RBF_EARG, "null pointer");
  return eval_pipeline(host_targets, n_targets, dev_in, dev_out, host_out, chunks, stream,
                       [&](const double* in, int64_t cnt, double* out, cudaStream_t cs) {
                         return rbf_eval_loop(in, cnt, sup, cap, state, radius, deform, out, cs);
                       });
}

// Error scans use the volume kernel's launch shape (128 threads x 6 rows, 3
// CTAs per SM); 2 / 4 rows per thread and 64-thread blocks measured within
// 5 % of it on configs[3]'s boundary (tools/err_kernel_time.py).
constexpr int kErrThreads = 128, kErrTPT = 6, kErrMinBlocks = 3;
constexpr int kErrRowsPerBlock = kErrThreads * kErrTPT;

// Small scans (a GCB group: a few hundred rows) would occupy a handful of
// SMs with one row per thread; they are split over S slices of the supports
// instead (grid = row blocks x S, partial sums through scratch, then one
// fixed-order pass sums the slices per row and finishes residual + arg-max):
// deterministic for a given (rows, supports).
constexpr int kSplitThreads = 128, kSplitTPT = 2;
constexpr int kSplitRowsPerBlock = kSplitThreads * kSplitTPT;
constexpr int64_t kSplitBound = 148LL * 4 * kSplitRowsPerBlock;  // rows x slices held in scratch
constexpr int kFinishThreads = 128;

static int split_slices(int64_t nt, int64_t ns) {
  if (nt >= kSplitBound / 2 || ns < 128) return 1;
  const int64_t blocks = (nt + kSplitRowsPerBlock - 1) / kSplitRowsPerBlock;
  int64_t S = (2 * 148 * 4 + blocks - 1) / blocks;  // ~2 waves of 4 CTAs per SM
  S = std::min<int64_t>(S, ns / 64);                 // >= 64 supports per slice
  S = std::min<int64_t>(S, kSplitBound / nt);
  return (int)std::max<int64_t>(S, 1);
}

__global__ void __launch_bounds__(kSplitThreads, 4)
err_partial_kernel(const double* __restrict__ tpts, const int64_t* __restrict__ pos, int64_t nt,
                   const double* __restrict__ spts, const double* __restrict__ sw, int nsup, int per_slice,
                   double inv_r, double* __restrict__ part) {
  __shared__ double4 s_a[128];
  __shared__ double2 s_b[128];
  const int slice = blockIdx.y;
  const int j0 = slice * per_slice, j1 = min(nsup, j0 + per_slice);
  const int64_t base = (int64_t)blockIdx.x * kSplitRowsPerBlock + threadIdx.x;
  double px[kSplitTPT], py[kSplitTPT], pz[kSplitTPT], ax[kSplitTPT], ay[kSplitTPT], az[kSplitTPT];
#pragma unroll
  for (int k = 0; k < kSplitTPT; ++k) {
    const int64_t idx = base + (int64_t)k * kSplitThreads;
    const int64_t r = idx < nt ? (pos ? pos[idx] : idx) : -1;
    px[k] = r >= 0 ? tpts[3 * r] * inv_r : 0.0;
    py[k] = r >= 0 ? tpts[3 * r + 1] * inv_r : 0.0;
    pz[k] = r >= 0 ? tpts[3 * r + 2] * inv_r : 0.0;
    ax[k] = ay[k] = az[k] = 0.0;
  }
  for (int t0 = j0; t0 < j1; t0 += 128) {
    const int cnt = min(128, j1 - t0);
    __syncthreads();
    for (int j = threadIdx.x; j < cnt; j += kSplitThreads) {
      const int g = t0 + j;
      s_a[j] = make_double4(spts[3 * g] * inv_r, spts[3 * g + 1] * inv_r, spts[3 * g + 2] * inv_r, sw[3 * g]);
      s_b[j] = make_double2(sw[3 * g + 1], sw[3 * g + 2]);
    }
    __syncthreads();
#pragma unroll 2
    for (int j = 0; j < cnt; ++j) {
      const double4 a = s_a[j];
      const double2 b = s_b[j];
#pragma unroll
      for (int k = 0; k < kSplitTPT; ++k)
        pair_accum(px[k], py[k], pz[k], a.x, a.y, a.z, a.w, b.x, b.y, ax[k], ay[k], az[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < kSplitTPT; ++k) {
    const int64_t idx = base + (int64_t)k * kSplitThreads;
    if (idx >= nt) continue;
    double* o = part + 3 * ((int64_t)slice * nt + idx);
    o[0] = ax[k];
    o[1] = ay[k];
    o[2] = az[k];
  }
}

__global__ void __launch_bounds__(kFinishThreads)
err_finish_kernel(const double* __restrict__ tdisp, const int64_t* __restrict__ pos, int64_t nt,
                  const double* __restrict__ part, int S, double* __restrict__ err_out,
                  Best* __restrict__ partials) {
  const int64_t idx = (int64_t)blockIdx.x * kFinishThreads + threadIdx.x;
  Best best{-1.0, 0x7fffffff};
  if (idx < nt) {
    double ux = 0.0, uy = 0.0, uz = 0.0;
    for (int sl = 0; sl < S; ++sl) {  // slices in order: deterministic
      const double* p = part + 3 * ((int64_t)sl * nt + idx);
      ux += p[0];
      uy += p[1];
      uz += p[2];
    }
    const int64_t r = pos ? pos[idx] : idx;
    const double e = residual_norm(tdisp[3 * r], tdisp[3 * r + 1], tdisp[3 * r + 2], ux, uy, uz);
    if (err_out) err_out[idx] = e;
    best = Best{e, (int)r};
  }
  best = warp_best(best);
  __shared__ Best s_best[kFinishThreads / kWarp];
  if ((threadIdx.x & 31) == 0) s_best[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    Best b = s_best[0];
    for (int w = 1; w < kFinishThreads / kWarp; ++w) b = best_of(b, s_best[w]);
    partials[blockIdx.x] = b;
  }
}

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

extern "C" size_t rbf_errors_scratch_bytes(int64_t n_targets) {
  const int64_t nt = n_targets < 1 ? 1 : n_targets;
  const int64_t blocks = std::max((nt + kErrRowsPerBlock - 1) / kErrRowsPerBlock,
                                  (nt + kFinishThreads - 1) / kFinishThreads);
  size_t bytes = 256 + align256((size_t)blocks * sizeof(Best));
  if (nt < kSplitBound / 2) bytes += (size_t)kSplitBound * 3 * sizeof(double);
  return bytes;
}

static int errors_argmax(const double* bnd_points, const double* bnd_disp, const int64_t* positions,
                         int64_t n_targets, const double* sup_points, const double* sup_weights, int64_t n_sup,
                         double radius, double* err_out, double* best_host, double* best_dev,
                         int64_t pos_offset, void* scratch, size_t scratch_bytes, void* stream) {
  if (n_targets <= 0) return set_error(RBF_EARG, "group is empty");
  if (!(radius > 0.0)) return set_error(RBF_EARG, "radius must be positive, got %g", radius);
  if (n_sup > INT32_MAX || n_targets > INT32_MAX) return set_error(RBF_EARG, "size too large");
  if (!bnd_points || !bnd_disp || !scratch) return set_error(RBF_EARG, "null pointer");
  if (scratch_bytes < rbf_errors_scratch_bytes(n_targets))
    return set_error(RBF_EARG, "scratch too small");
  int64_t nblk = 0;
  cudaStream_t s = as_stream(stream);
  double* result = best_dev ? best_dev : reinterpret_cast<double*>(scratch);
  Best* partials = reinterpret_cast<Best*>(static_cast<char*>(scratch) + 256);
  const double inv_r = 1.0 / radius;
  const int S = split_slices(n_targets, n_sup);
  if (S > 1) {
    const int64_t blocks = (n_targets + kErrRowsPerBlock - 1) / kErrRowsPerBlock;
    const int64_t fin = (n_targets + kFinishThreads - 1) / kFinishThreads;
    double* part = reinterpret_cast<double*>(static_cast<char*>(scratch) + 256 +
                                             align256((size_t)std::max(blocks, fin) * sizeof(Best)));
    const int per_slice = (int)((n_sup + S - 1) / S);
    const dim3 grid((unsigned)((n_targets + kSplitRowsPerBlock - 1) / kSplitRowsPerBlock), (unsigned)S);
    err_partial_kernel<<<grid, kSplitThreads, 0, s>>>(bnd_points, positions, n_targets, sup_points, sup_weights,
                                                       (int)n_sup, per_slice, inv_r, part);
    RBF_LAUNCH_CHECK("err_partial_kernel");
    nblk = fin;
    err_finish_kernel<<<(unsigned)nblk, kFinishThreads, 0, s>>>(bnd_disp, positions, n_targets, part, S, err_out,
                                                                 partials);
    RBF_LAUNCH_CHECK("err_finish_kernel");
  } else {
    nblk = (n_targets + kErrRowsPerBlock - 1) / kErrRowsPerBlock;
    eval_kernel<kModeError, kErrThreads, kErrTPT, 128, kErrMinBlocks><<<(unsigned)nblk, kErrThreads, 0, s>>>(
        bnd_points, bnd_disp, positions, n_targets, sup_points, sup_weights, (int)n_sup, inv_r, err_out,
        partials);
    RBF_LAUNCH_CHECK("eval_kernel<error>");
  }
  best_reduce_kernel<<<1, 256, 0, s>>>(partials, (int)nblk, result, pos_offset);
  RBF_LAUNCH_CHECK("best_reduce_kernel");
  if (best_host) {
    RBF_CUDA_TRY(cudaMemcpyAsync(best_host, result, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    RBF_CUDA_TRY(cudaStreamSynchronize(s));
  }
  return RBF_OK;
}

extern "C" int rbf_errors_argmax(const double* bnd_points, const double* bnd_disp,
                                 const int64_t* positions, int64_t n_targets,
                                 const double* sup_points, const double* sup_weights, int64_t n_sup,
                                 double radius, double* err_out, double* best_host, void* scratch,
                                 size_t scratch_bytes, void* stream) {
  return errors_argmax(bnd_points, bnd_disp, positions, n_targets, sup_points, sup_weights, n_sup, radius,
                       err_out, best_host, nullptr, 0, scratch, scratch_bytes, stream);
}

extern "C" int rbf_errors_argmax_dev(const double* bnd_points, const double* bnd_disp,
                                     const int64_t* positions, int64_t n_targets,
                                     const double* sup_points, const double* sup_weights, int64_t n_sup,
                                     double radius, double* err_out, int64_t pos_offset, double* best_dev,
                                     void* scratch, size_t scratch_bytes, void* stream) {
  if (!best_dev) return set_error(RBF_EARG, "null pointer");
  if (n_targets == 0) {  // an empty shard contributes the neutral record {-1, INT32_MAX}
    best_reduce_kernel<<<1, 256, 0, as_stream(stream)>>>(nullptr, 0, best_dev, 0);
    RBF_LAUNCH_CHECK("best_reduce_kernel");
    return RBF_OK;
  }
  return errors_argmax(bnd_points, bnd_disp, positions, n_targets, sup_points, sup_weights, n_sup, radius,
                       err_out, nullptr, best_dev, pos_offset, scratch, scratch_bytes, stream);
}

extern "C" int rbf_best_fold(const double* recs, int64_t n, double* out, void* stream) {
  if (n <= 0 || !recs || !out) return set_error(RBF_EARG, "rbf_best_fold: empty input or null pointer");
  best_fold_kernel<<<1, 256, 0, as_stream(stream)>>>(recs, n, out);
  RBF_LAUNCH_CHECK("best_fold_kernel");
  return RBF_OK;
}

// ------------------------------------------------------------ nearest support
// out[k] = min_i |t_k - s_i|_2 with scipy cdist's rounding (reference
// metrics.py:45-48 `_nearest_distances`, metrics.py:51-60
// `nearest_support_distance`): squared distance (dx*dx + dy*dy) + dz*dz
// without contraction, the minimum over supports, one correctly rounded
// sqrt at the end (sqrt is monotone and correctly rounded, so
// sqrt(min d^2) == min sqrt(d^2) bit for bit). Coordinates are not scaled.
constexpr int kNearThreads = 128, kNearTPT = 4, kNearTile = 256;

__global__ void __launch_bounds__(kNearThreads)
nearest_kernel(const double* __restrict__ tpts, int64_t nt, const double* __restrict__ spts, int nsup,
               double* __restrict__ out) {
  __shared__ double s_x[kNearTile], s_y[kNearTile], s_z[kNearTile];
  const int64_t base = (int64_t)blockIdx.x * (kNearThreads * kNearTPT) + threadIdx.x;
  double px[kNearTPT], py[kNearTPT], pz[kNearTPT], dmin[kNearTPT];
#pragma unroll
  for (int k = 0; k < kNearTPT; ++k) {
    const int64_t r = base + (int64_t)k * kNearThreads;
    const bool ok = r < nt;
    px[k] = ok ? tpts[3 * r] : 0.0;
    py[k] = ok ? tpts[3 * r + 1] : 0.0;
    pz[k] = ok ? tpts[3 * r + 2] : 0.0;
    dmin[k] = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  }
  for (int t0 = 0; t0 < nsup; t0 += kNearTile) {
    const int cnt = min(kNearTile, nsup - t0);
    __syncthreads();
    for (int j = threadIdx.x; j < cnt; j += kNearThreads) {
      s_x[j] = spts[3 * (int64_t)(t0 + j)];
      s_y[j] = spts[3 * (int64_t)(t0 + j) + 1];
      s_z[j] = spts[3 * (int64_t)(t0 + j) + 2];
    }
    __syncthreads();
#pragma unroll 4
    for (int j = 0; j < cnt; ++j) {
      const double sx = s_x[j], sy = s_y[j], sz = s_z[j];
#pragma unroll
      for (int k = 0; k < kNearTPT; ++k) {
        const double dx = __dsub_rn(px[k], sx), dy = __dsub_rn(py[k], sy), dz = __dsub_rn(pz[k], sz);
        const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
        dmin[k] = fmin(dmin[k], d2);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kNearTPT; ++k) {
    const int64_t r = base + (int64_t)k * kNearThreads;
    if (r < nt) out[r] = __dsqrt_rn(dmin[k]);
  }
}

extern "C" int rbf_nearest(const double* targets, int64_t n_targets, const double* sup_points, int64_t n_sup,
                           double* out, void* stream) {
  if (n_targets < 0 || n_sup < 0) return set_error(RBF_EARG, "negative size");
  if (n_sup == 0) return set_error(RBF_EARG, "support set is empty");
  if (n_sup > INT32_MAX) return set_error(RBF_EARG, "too many supports");
  if (n_targets == 0) return RBF_OK;
  if (!targets || !sup_points || !out) return set_error(RBF_EARG, "null pointer");
  const int64_t per = (int64_t)kNearThreads * kNearTPT;
  nearest_kernel<<<(unsigned)((n_targets + per - 1) / per), kNearThreads, 0, as_stream(stream)>>>(
      targets, n_targets, sup_points, (int)n_sup, out);
  RBF_LAUNCH_CHECK("nearest_kernel");
  return RBF_OK;
}
