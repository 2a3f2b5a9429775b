/*
 * rbf_b200.h -- C ABI of the B200 (sm_100a) hot path for GCB-greedy RBF mesh
 * deformation (Fang et al., arXiv 2004.04817).
 *
 * The reference (`rbfdeform`, pure Python) has no FFI layer: its only
 * interface is the Python API. Each entry point below replaces the
 * reference function named beside it; the Python package
 * `paper_2004_04817_b200` binds them with ctypes and keeps the reference's
 * names, argument meaning and exceptions.
 *
 * Conventions
 *  - Every pointer argument is a DEVICE pointer (caller-owned, e.g. torch
 *    tensors) unless its name ends in `_host`. Arrays of points,
 *    displacements and weights are C-contiguous (n, 3) float64 (AoS), the
 *    reference's layout (core.py:227-265, selection.py:46-83).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream). Calls are
 *    stream-ordered and asynchronous unless documented otherwise.
 *  - The library never allocates or frees caller memory; scratch buffers
 *    are passed in and sized by rbf_*_scratch_bytes().
 *  - Return value: RBF_OK or an RBF_E* code; rbf_last_error() gives a
 *    thread-local message. No CPU fallback exists: without a CUDA device
 *    every compute entry point returns RBF_ECUDA.
 */
#ifndef RBF_B200_H
#define RBF_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define RBF_API __attribute__((visibility("default")))
#else
#define RBF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define RBF_ABI_VERSION 1

enum {
  RBF_OK = 0,
  RBF_EARG = 1,     /* bad argument -> ValueError family                    */
  RBF_ECUDA = 2,    /* CUDA runtime error / no device                       */
  RBF_ENOTPD = 3,   /* NotPositiveDefiniteError (errors.py:13-15)            */
  RBF_EGROW = 5,    /* selection loop paused: factor/record capacity full    */
  RBF_ESTALL = 6,   /* SelectionStalledError (errors.py:44-46)               */
  RBF_EPARSE = 7,   /* text not parsed natively: the caller re-parses it with
                       the reference grammar for the exact ParseError      */
  RBF_ENCCL = 4     /* reserved: collective error                            */
};

RBF_API int rbf_abi_version(void);
RBF_API const char* rbf_last_error(void);
/* Number of SMs and cooperative CTAs the selection loop uses on `device`. */
RBF_API int rbf_device_info(int device, int* sm_count_host, int* loop_ctas_host);

/* ---------------------------------------------------------------------
 * Volume / boundary evaluation.
 * Replaces core.py:301-334 `_eval_displacements` (called by
 * evaluate_displacements core.py:337-351, evaluate_displacement
 * core.py:354-356 and deform_points core.py:359-367):
 *   out[k] = sum_i w_i * phi(|p_k - s_i| / radius)          (deform == 0)
 *   out[k] = p_k + sum_i w_i * phi(|p_k - s_i| / radius)    (deform == 1)
 * The per-target summation order is fixed (independent of n_targets and of
 * how targets are sharded), so shards are bitwise identical to a single
 * call. `out` may not alias `targets`.
 */
RBF_API int rbf_eval(const double* targets, int64_t n_targets,
             const double* sup_points, const double* sup_weights, int64_t n_sup,
             double radius, int deform, double* out, void* stream);

/* Host-resident variant of rbf_eval for inputs that live in host memory
 * (the public numpy API: core.py:337-367): `host_targets` (n,3) are streamed
 * through the caller's device buffers `dev_in` / `dev_out` (n,3 each) in
 * `chunks` pieces (<= 63) on library-owned copy streams, so the
 * host->device copy, the kernel and the device->host copy of consecutive
 * pieces overlap (PCIe is full duplex). Results land in `host_out` (pinned
 * memory for asynchronous copies) once `stream` is synchronised; bitwise
 * equal to rbf_eval on the whole array. Support arrays are device pointers.
 * host_targets == NULL: the targets are already in dev_in (copied there
 * ahead of time in stream order); only the kernels and result copies run.
 */
RBF_API int rbf_eval_host(const double* host_targets, int64_t n_targets,
                  const double* sup_points, const double* sup_weights, int64_t n_sup,
                  double radius, int deform, double* dev_in, double* dev_out,
                  double* host_out, int chunks, void* stream);

/* ---------------------------------------------------------------------
 * Interpolation error at boundary rows, fused with the (err, lowest id)
 * arg-max.  Replaces selection.py:215-221 `_errors_at` +
 * selection.py:231-234 `_argmax_lowest_id` (as used by
 * group_arg_max_error selection.py:237-254 and the final sweep
 * selection.py:394-402):
 *   err[t] = | disp[pos[t]] - sum_i w_i phi(|pts[pos[t]] - s_i| / R) |_2
 * `positions` may be NULL (then pos[t] = t). `err_out` may be NULL.
 * `best_host` (may be NULL) receives {max_err, (double)pos_of_max} after a
 * stream synchronisation; ties go to the lowest position.
 * `scratch` must hold rbf_errors_scratch_bytes(n_targets) bytes.
 */
RBF_API size_t rbf_errors_scratch_bytes(int64_t n_targets);
RBF_API int rbf_errors_argmax(const double* bnd_points, const double* bnd_disp,
                      const int64_t* positions, int64_t n_targets,
                      const double* sup_points, const double* sup_weights, int64_t n_sup,
                      double radius, double* err_out, double* best_host,
                      void* scratch, size_t scratch_bytes, void* stream);

/* Device-resident variant for sharded sweeps (multi-GPU final sweep and
 * error_summary): no synchronisation; `best_dev` (device,
 * 2 doubles) receives {max_err, pos_of_max + pos_offset}, the rank's 16-byte
 * record for the all-gather. n_targets == 0 (an empty shard) writes the
 * neutral record {-1, INT32_MAX}. The per-row summation order is the one
 * rbf_errors_argmax uses for the same (n_targets, n_sup).
 */
RBF_API int rbf_errors_argmax_dev(const double* bnd_points, const double* bnd_disp,
                          const int64_t* positions, int64_t n_targets,
                          const double* sup_points, const double* sup_weights, int64_t n_sup,
                          double radius, double* err_out, int64_t pos_offset, double* best_dev,
                          void* scratch, size_t scratch_bytes, void* stream);

/* Fold n (err, pos) records (n x 2 doubles, device) into out[2] (device):
 * the largest error, exact ties to the lowest position (selection.py:231-234).
 * The combine step of a sharded sweep after the all-gather of the per-rank
 * records. */
RBF_API int rbf_best_fold(const double* recs, int64_t n, double* out, void* stream);

/* ---------------------------------------------------------------------
 * Nearest-support distances.  Replaces metrics.py:45-48
 * `_nearest_distances` (cdist + row min, used by kl_divergence
 * metrics.py:63-74) and metrics.py:51-60 `nearest_support_distance`:
 *   out[k] = min_i | t_k - s_i |_2
 * with cdist's rounding, sqrt((dx*dx + dy*dy) + dz*dz) uncontracted, so the
 * distances are bit-identical to the reference's. Device pointers, AoS
 * (n,3) float64; n_sup = 0 -> RBF_EARG ("support set is empty").
 */
RBF_API int rbf_nearest(const double* targets, int64_t n_targets,
                const double* sup_points, int64_t n_sup, double* out, void* stream);

/* ---------------------------------------------------------------------
 * Growing Cholesky factor.  Replaces core.py:115-205 `CholeskyState`.
 * The factor L and its inverse Li are stored as PACKED lower triangles,
 * row-major (row i starts at i*(i+1)/2), so capacity growth is a prefix
 * copy. `n` is the current order.
 *
 * rbf_chol_append (core.py:153-185): given row[0..n] (the new matrix row
 * against the n prior indices plus itself), computes c = L^-1 row[:n]
 * (inverse product plus one step of residual refinement) and
 * pivot^2 = row[n] - c.c. If pivot^2 > 0 it writes row n of L and Li and
 * returns RBF_OK; otherwise it returns RBF_ENOTPD and leaves the state
 * unchanged. `pivot2_host` receives pivot^2 in both cases. Synchronous.
 * L and Li must have room for (n+1)(n+2)/2 doubles. `scratch` holds
 * rbf_chol_scratch_bytes(n+1) bytes.
 */
RBF_API size_t rbf_chol_scratch_bytes(int64_t n);
RBF_API int rbf_chol_append(double* L, double* Li, int64_t n, const double* row,
                    double* pivot2_host, void* scratch, size_t scratch_bytes,
                    void* stream);

/* rbf_chol_append_points: rbf_chol_append for rows n0 .. n0+k-1 at once,
 * the rows built on the device from the supports' coordinates (sup: device
 * (n0+k, 3) AoS; row i = phi(|s_i - s_j| / radius), j <= i, the reference's
 * kernel_matrix rounding, core.py:82-88) -- no host round trip between the
 * rows (solve_support_weights core.py:268-281, metrics.error_history
 * metrics.py:91-115). Stops at the first non-positive pivot: returns
 * RBF_ENOTPD with *appended_host = rows appended before it (the state has
 * order n0 + *appended_host) and *fail_pivot2_host its pivot^2. Synchronous
 * (one host read at the end). L and Li must have room for order n0 + k.
 * `scratch` holds rbf_chol_points_scratch_bytes(n0 + k + 1) bytes. */
RBF_API size_t rbf_chol_points_scratch_bytes(int64_t n_total);
RBF_API int rbf_chol_append_points(double* L, double* Li, int64_t n0, int64_t k, const double* sup,
                                   double radius, int64_t* appended_host, double* fail_pivot2_host,
                                   void* scratch, size_t scratch_bytes, void* stream);

/* rbf_chol_solve (core.py:187-205): x = (L L^T)^-1 rhs for rhs (n, k)
 * row-major, k >= 1. out may alias rhs. */
RBF_API int rbf_chol_solve(const double* L, const double* Li, int64_t n,
                   const double* rhs, int64_t k, double* out,
                   void* scratch, size_t scratch_bytes, void* stream);

/* ---------------------------------------------------------------------
 * The GCB / greedy selection loop, fully device resident.
 * Replaces selection.py:274-421 `_gcb_run` (entry points gcb_select
 * selection.py:257-271 and greedy_select selection.py:424-428), including
 * the seeds (selection.py:198-212, bit-exact norms and first-occurrence
 * arg-max) and the final sweep.
 *
 * The host does what must stay bit-identical to numpy's PCG64: the
 * partition (selection.py:177-185); it passes the groups in. One
 * persistent kernel then runs everything else. Two launch shapes share the
 * code: a single 16-CTA thread-block cluster synchronised by hardware
 * cluster barriers (small and medium problems: every phase is latency
 * bound), or a cooperative grid of one CTA per SM with a software grid
 * barrier (large group scans). It returns RBF_EGROW when the factor or
 * record buffers are full: the host grows them (packed prefixes are
 * capacity independent) and calls again with the same state, which resumes
 * the same iteration.
 */
typedef struct rbf_gcb_record {
  int32_t group;      /* group visited (-1 for the final sweep)             */
  int32_t node_pos;   /* position of the added node, else of the arg-max   */
  int32_t added;      /* 1 if a node was appended this iteration           */
  int32_t n_before;   /* support count during the scan                     */
  double local_max;   /* max error in the group (ineligible nodes included) */
  double t1_s;        /* scan time (device clock)                          */
  double t2_s;        /* factor/weights time carried into this record      */
} rbf_gcb_record;

typedef struct rbf_gcb_state {
  int32_t n;            /* current support count                          */
  int32_t k;            /* iteration counter (starts at 3, selection.py:307) */
  int32_t streak_ok;    /* selection.py:373-386                            */
  int32_t streak_noadd;
  int32_t n_records;
  int32_t status;       /* 0 running, 1 done, RBF_E* on failure            */
  int32_t fail_row;     /* NotPD: row index of the failing seed append     */
  int32_t done_loop;    /* 1 once the loop ended (final sweep pending/done) */
  double fail_pivot2;
  double t2_carry;
  double final_max;     /* final sweep */
  int32_t final_pos;
  int32_t fault;        /* watchdog flag                                   */
  int32_t want_mode;    /* on RBF_EGROW: mode the kernel asks to resume in  */
  int32_t handover;     /* on RBF_EGROW to GRID: 0, or the one-cluster mode whose
                           run without appends the whole-GPU tail launch resolves */
  /* diagnostics: SM cycles CTA 0 spent per phase, summed over the run:
   * [0] scan+barrier, [1] fold+row, [2] c0, [3] r, [4] c, [5] pivot+cols,
   * [6] bookkeeping, [7] seeds, [8] final sweep, [9] appends, [10] iterations,
   * [11..14] scan sub-phases: targets+compute, reduce, epilogue, partials,
   * [15] column partials of Li^T [c, y] */
  double phase_cycles[16];
} rbf_gcb_state;

/* rbf_gcb_args.flags */
#define RBF_GCB_PHASES 1
#define RBF_GCB_NO_OVERLAP 2 /* MSG path: no next-group scan during appends (A/B tests) */
#define RBF_GCB_NO_TAIL 4    /* one-cluster paths: final sweep in the cluster instead of a
                                stream-ordered whole-GPU tail launch (A/B tests) */
#define RBF_GCB_NO_SWEEP 8   /* end the loop without the final sweep (state->final_pos = -1,
                                no final record): the caller sweeps the boundary itself, e.g.
                                sharded over GPUs with rbf_errors_argmax_dev + rbf_best_fold */
#define RBF_GCB_REFINE 16    /* MSG path: the refinement step in every append (by default it
                                starts once min l_i^2 < 1e-7; A/B tests) */

/* Launch shapes of the selection kernel:
 *  MSG     one 16-CTA cluster, n < 384: the factor rows (owner-stable, row
 *          i in CTA i % 16) and all vectors resident in shared memory; every
 *          cross-CTA value is pushed with st.async into the consumer's
 *          mbarrier -- no cluster barriers in steady state;
 *  SMEM    one 16-CTA cluster; supports, weights and the Cholesky work
 *          vectors replicated in every CTA's shared memory (written through
 *          distributed shared memory), the factor rows in L2 (n < 1024);
 *  CLUSTER one 16-CTA cluster, all state in global memory (L2);
 *  GRID    one CTA per SM (cooperative), all state in global memory.
 * AUTO picks MSG for group sizes up to 2048 and GRID above. The kernel
 * pauses (RBF_EGROW) and names the shape to resume in: MSG -> SMEM when n
 * reaches 383 with group scans of at most 1.5e5 pairs (card * n), else ->
 * GRID; SMEM -> GRID when n reaches 1023; any one-cluster shape -> GRID as
 * soon as a group scan exceeds 8e5 pairs. CLUSTER runs only when forced
 * (DESIGN.md §4.2). */
enum { RBF_GCB_AUTO = 0, RBF_GCB_CLUSTER = 1, RBF_GCB_GRID = 2, RBF_GCB_SMEM = 3, RBF_GCB_MSG = 4 };

typedef struct rbf_gcb_args {
  /* boundary (device) */
  const double* points;     /* (nb, 3) */
  const double* disp;       /* (nb, 3) */
  const int32_t* group_pos; /* (nb) positions, groups concatenated        */
  const int32_t* group_off; /* (m + 1) offsets into group_pos              */
  int32_t nb, m;
  int32_t mode;             /* RBF_GCB_AUTO / _CLUSTER / _GRID / ...       */
  int32_t max_supports;
  int32_t clusters;         /* MSG path: 16-CTA clusters sharing the group
                               scans (0 = library default); each computes the
                               appends redundantly, scan partials meet in L2 */
  int32_t flags;            /* RBF_GCB_PHASES: record per-phase SM cycles (costs
                               ~4 % of the loop; off by default)              */
  double radius, tol;
  double dup_dist;          /* NEAR_DUPLICATE_FRACTION * radius            */
  /* factor state (device), capacity in rows */
  double* L;                /* packed, cap*(cap+1)/2 */
  double* Li;               /* packed, cap*(cap+1)/2 */
  double* y;                /* (cap, 3) forward-substituted displacements */
  double* sup;              /* (12, cap) SoA: x, y, z, wx, wy, wz (weights), then the
                               compensated weights' hi (3 rows) and lo (3 rows): the
                               loop carries each weight as hi + lo */
  int32_t* sel;             /* (cap) selected positions in order          */
  uint8_t* inel;            /* (nb) ineligible flags                       */
  int32_t cap;
  /* records (device) */
  rbf_gcb_record* records;
  int32_t rec_cap;
  /* state + scratch (device) */
  rbf_gcb_state* state;
  void* scratch;            /* rbf_gcb_scratch_bytes(nb, cap, ctas) bytes */
  size_t scratch_bytes;
} rbf_gcb_args;

/* Team width to size the selection scratch for (rbf_gcb_scratch_bytes):
 * the SM count in every mode, since a one-cluster launch is followed by a
 * whole-GPU launch for its final sweep and a run can move between shapes;
 * *resolved_mode_host is the shape `mode` resolves to (AUTO picks MSG for
 * group sizes up to 2048, GRID above). */
RBF_API int rbf_gcb_ctas(int32_t mode, int32_t nb, int32_t m, int32_t* ctas_host,
                         int32_t* resolved_mode_host);
RBF_API size_t rbf_gcb_scratch_bytes(int32_t nb, int32_t cap, int32_t ctas);
/* Launch (asynchronous). The caller zero-initialises *state (n = 0) and
 * inel before the first call. */
RBF_API int rbf_gcb_run(const rbf_gcb_args* args, void* stream);

/* rbf_eval with the supports taken from a selection run's own buffers:
 * `sup` = rbf_gcb_args.sup (SoA rows x, y, z, wx, wy, wz of capacity `cap`),
 * the support count from state->n, read on the device. Meant to be queued
 * on the selection's stream right behind rbf_gcb_run, before the host has
 * read the result (the volume kernel then overlaps the host's unpacking of
 * the selection: gcb_select + deform_points as one device sequence, the
 * reference's cmd_deform, cli.py:158-182). Does nothing unless the loop
 * finished (state->status == 1); the caller re-queues it otherwise. */
RBF_API int rbf_eval_loop(const double* targets, int64_t n_targets, const double* sup, int64_t cap,
                          const rbf_gcb_state* state, double radius, int deform, double* out,
                          void* stream);
/* rbf_eval_host (host targets, chunked copy / kernel / copy pipeline) with
 * the supports of rbf_eval_loop: the selection's result goes straight into
 * the volume pipeline queued behind the loop. The copies always run; the
 * kernels only if the loop finished. host_targets == NULL: the targets are
 * already in dev_in (the caller copied them ahead, in stream order, e.g.
 * while the loop ran), and only the kernels and the result copies run. */
RBF_API int rbf_eval_host_loop(const double* host_targets, int64_t n_targets, const double* sup,
                               int64_t cap, const rbf_gcb_state* state, double radius, int deform,
                               double* dev_in, double* dev_out, double* host_out, int chunks,
                               void* stream);


/* ---------------------------------------------------------------------
 * Group partition on the host (replaces selection.py:177-185
 * `partition_boundary`'s arithmetic): numpy's PCG64 permutation of nb dealt
 * round-robin into m groups, bit for bit. (state, inc) are the 128-bit
 * words of numpy.random.default_rng(seed).bit_generator.state, split
 * hi/lo. Writes group_pos_host[nb] (positions, groups concatenated) and
 * group_off_host[m + 1]. Host memory, no GPU needed.
 */
RBF_API int rbf_partition(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                          int64_t nb, int64_t m, int32_t* group_pos_host, int32_t* group_off_host);

/* ---------------------------------------------------------------------
 * Diagnostics (no reference counterpart): an FP64 DFMA throughput probe
 * used to measure the FP64 peak the roofline fractions are quoted against.
 * `scratch` holds rbf_fp64_probe_scratch_bytes(device) bytes; `flops_host`
 * receives the FP64 operations the launch performs (time it with events).
 */
/* ---------------------------------------------------------------------
 * MDK1 / MDK1-DISP text codec (host, multi-threaded).  Replaces the bulk
 * of meshio.py:135-250 (`read_mesh`, `write_mesh`, `read_displacements`,
 * `write_displacements`). Readers accept exactly the inputs the reference
 * parses the same way and return RBF_EPARSE for everything else (malformed
 * text, and tokens outside the plain numeric grammar), on which the Python
 * layer re-parses with the reference grammar to raise its ParseError /
 * InvariantViolationError with the line number. `threads` <= 0: all cores.
 *
 * rbf_mdk1_counts: node / boundary / cell counts (counts[3]).
 * rbf_mdk1_parse:  nodes (nv,3), boundary (nb, file order), cells (ne,5):
 *                  arity then 3-4 node indices.
 * rbf_disp_parse:  (nb,3) displacements aligned with the sorted boundary.
 * rbf_mdk1_format_nodes / rbf_disp_format: canonical "%.17g" rows into
 *                  `out` (100 / 124 bytes per row suffice); bytes written
 *                  or -1.
 */
RBF_API int rbf_mdk1_counts(const char* text, size_t len, int64_t* counts, int threads);
RBF_API int rbf_mdk1_parse(const char* text, size_t len, int64_t nv, int64_t nb, int64_t ne,
                   double* nodes, int64_t* boundary, int64_t* cells, int threads);
RBF_API int rbf_disp_parse(const char* text, size_t len, const int64_t* boundary, int64_t nb,
                   double* disp, int threads);
RBF_API int64_t rbf_mdk1_format_nodes(const double* xyz, int64_t n, char* out, int64_t cap,
                              int threads);
RBF_API int64_t rbf_disp_format(const int64_t* idx, const double* xyz, int64_t n, char* out,
                        int64_t cap, int threads);

/* Return the persisting-L2 lines the L2-path selection launch keeps for Li
 * (an access-policy window) to normal status; call once a selection has
 * finished (bound by the Python layer after rbf_gcb_run). */
RBF_API int rbf_l2_release(void);

RBF_API size_t rbf_fp64_probe_scratch_bytes(int device);
RBF_API int rbf_fp64_probe(int iters, double* scratch, double* flops_host, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RBF_B200_H */
