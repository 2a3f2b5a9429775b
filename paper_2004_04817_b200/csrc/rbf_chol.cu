// Standalone growing Cholesky factor behind `CholeskyState`
// (reference core.py:115-205, cholesky_append core.py:208-210,
// solve_weights core.py:213-224, solve_support_weights core.py:268-281).
//
// The reference appends row n by forward substitution c = L^-1 row[:n]
// (LAPACK, padded to 256-row blocks: core.py:139-151) and solves with two
// triangular substitutions. Here the factor keeps its inverse Li alongside
// L (both packed), so each substitution is a parallel product:
//   c0 = Li row,  c = c0 + Li (row - L c0)        (one refinement step)
//   pivot^2 = row[n] - c.c ;  L[n] = [c, l],  Li[n] = [-(c^T Li)/l, 1/l]
// The refinement step brings c to substitution accuracy (tests/ and
// DESIGN.md §4 quantify it against the reference).
#include <cmath>
#include <cstdint>

#include "rbf_common.cuh"
#include "rbf_internal.h"
#include "rbf_tri.cuh"

namespace rbf {

constexpr int kTriThreads = 256;
constexpr int kTriWarps = kTriThreads / 32;

// y[i] = b[i] + s * sum_{j<=i} A[i][j] x[j]   (b may be null)
template <int K>
__global__ void __launch_bounds__(kTriThreads) k_tri_rows(const double* A, int n, const double* x,
                                                          int ldx, const double* b, int ldb,
                                                          double s, double* y, int ldy) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kTriWarps + (threadIdx.x >> 5);
  tri_rows<K>(
      A, n, [&](int j, int c) { return x[(int64_t)j * ldx + c]; },
      [&](int i, const double* acc) {
#pragma unroll
        for (int c = 0; c < K; ++c) {
          const double base = b ? b[(int64_t)i * ldb + c] : 0.0;
          y[(int64_t)i * ldy + c] = fma(s, acc[c], base);
        }
      },
      gw, gridDim.x * kTriWarps, lane);
}

// y[j] = b[j] + s * sum_{i>=j} A[i][j] x[i]
template <int K>
__global__ void __launch_bounds__(kTriThreads) k_tri_cols(const double* A, int n, const double* x,
                                                          int ldx, const double* b, int ldb,
                                                          double s, double* y, int ldy) {
  __shared__ double red[kTriWarps * 32 * K];
  tri_cols<K, kTriWarps>(
      A, n, [&](int i, int c) { return x[(int64_t)i * ldx + c]; }, (int)blockIdx.x,
      (int)gridDim.x, red, [&](int j, const double* sum) {
#pragma unroll
        for (int c = 0; c < K; ++c) {
          const double base = b ? b[(int64_t)j * ldb + c] : 0.0;
          y[(int64_t)j * ldy + c] = fma(s, sum[c], base);
        }
      });
}

// pivot^2 = row[n] - c.c, written to out[0]; one block, fixed order.
__global__ void k_pivot(const double* row, const double* c, int n, double* out) {
  double acc = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) acc = fma(c[j], c[j], acc);
  acc = warp_sum(acc);
  __shared__ double s[32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    out[0] = row[n] - t;
  }
}

// Write row n of L and Li once the pivot is accepted.
__global__ void k_commit(double* L, double* Li, int n, const double* c, const double* u,
                         double l) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) {
    L[tri_off(n) + j] = c[j];
    Li[tri_off(n) + j] = -u[j] / l;
  } else if (j == n) {
    L[tri_off(n) + n] = l;
    Li[tri_off(n) + n] = 1.0 / l;
  }
}

// Batched appends (rbf_chol_append_points): the kernel row of support i
// against supports 0..i with the reference's rounding (kernel_matrix,
// core.py:82-88: phi(cdist / R), phi(0) = 1), skipped once an earlier row of
// the batch failed.
__global__ void k_exact_row(const double* sup, int i, double radius, const int* status, double* row) {
  if (*status) return;
  const double px = sup[3 * (int64_t)i], py = sup[3 * (int64_t)i + 1], pz = sup[3 * (int64_t)i + 2];
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= i; j += gridDim.x * blockDim.x)
    row[j] = j == i ? 1.0 : phi_exact(cdist_exact(px, py, pz, sup[3 * (int64_t)j], sup[3 * (int64_t)j + 1],
                                                  sup[3 * (int64_t)j + 2]), radius);
}
// pivot^2 as k_pivot; a non-positive one records (row, pivot^2) and stops the
// rest of the batch (status = 1)
__global__ void k_pivot_status(const double* row, const double* c, int n, double* piv, int* status,
                               double* fail) {
  if (*status) return;
  double acc = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) acc = fma(c[j], c[j], acc);
  acc = warp_sum(acc);
  __shared__ double s[32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    const double p2 = row[n] - t;
    piv[0] = p2;
    if (!(p2 > 0.0)) {
      fail[0] = p2;
      fail[1] = (double)n;
      *status = 1;
    }
  }
}
// k_commit with l = sqrt(pivot^2) taken on the device (correctly rounded, as
// the host's std::sqrt in rbf_chol_append)
__global__ void k_commit_dev(double* L, double* Li, int n, const double* c, const double* u,
                             const double* piv, const int* status) {
  if (*status) return;
  const double l = sqrt(piv[0]);
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) {
    L[tri_off(n) + j] = c[j];
    Li[tri_off(n) + j] = -u[j] / l;
  } else if (j == n) {
    L[tri_off(n) + n] = l;
    Li[tri_off(n) + n] = 1.0 / l;
  }
}

static inline unsigned row_blocks(int n) {
  int b = (n + kTriWarps - 1) / kTriWarps;
  return (unsigned)(b < 1 ? 1 : (b > 4096 ? 4096 : b));
}
static inline unsigned col_blocks(int n) {
  int b = (n + 31) / 32;
  return (unsigned)(b < 1 ? 1 : (b > 4096 ? 4096 : b));
}

template <int K>
static void launch_rows(const double* A, int n, const double* x, int ldx, const double* b,
                        int ldb, double s, double* y, int ldy, cudaStream_t st) {
  k_tri_rows<K><<<row_blocks(n), kTriThreads, 0, st>>>(A, n, x, ldx, b, ldb, s, y, ldy);
}
template <int K>
static void launch_cols(const double* A, int n, const double* x, int ldx, const double* b,
                        int ldb, double s, double* y, int ldy, cudaStream_t st) {
  k_tri_cols<K><<<col_blocks(n), kTriThreads, 0, st>>>(A, n, x, ldx, b, ldb, s, y, ldy);
}

using GemvFn = void (*)(const double*, int, const double*, int, const double*, int, double,
                        double*, int, cudaStream_t);
static GemvFn rows_fn(int k) {
  static const GemvFn f[4] = {launch_rows<1>, launch_rows<2>, launch_rows<3>, launch_rows<4>};
  return f[k - 1];
}
static GemvFn cols_fn(int k) {
  static const GemvFn f[4] = {launch_cols<1>, launch_cols<2>, launch_cols<3>, launch_cols<4>};
  return f[k - 1];
}

}  // namespace rbf

using namespace rbf;

extern "C" size_t rbf_chol_scratch_bytes(int64_t n) {
  // c0, r, c, u (n each) + pivot slot, 256-byte aligned pieces
  size_t v = ((size_t)(n < 1 ? 1 : n) * sizeof(double) + 255) & ~(size_t)255;
  return 4 * v + 256;
}

extern "C" int rbf_chol_append(double* L, double* Li, int64_t n64, const double* row,
                               double* pivot2_host, void* scratch, size_t scratch_bytes,
                               void* stream) {
  if (n64 < 0 || n64 >= INT32_MAX) return set_error(RBF_EARG, "bad order");
  if (!L || !Li || !row || !scratch) return set_error(RBF_EARG, "null pointer");
  if (scratch_bytes < rbf_chol_scratch_bytes(n64 + 1)) return set_error(RBF_EARG, "scratch too small");
  const int n = (int)n64;
  cudaStream_t st = as_stream(stream);
  size_t v = ((size_t)((n + 1) < 1 ? 1 : (n + 1)) * sizeof(double) + 255) & ~(size_t)255;
  char* base = static_cast<char*>(scratch);
  double* c0 = reinterpret_cast<double*>(base);
  double* r = reinterpret_cast<double*>(base + v);
  double* c = reinterpret_cast<double*>(base + 2 * v);
  double* u = reinterpret_cast<double*>(base + 3 * v);
  double* piv = reinterpret_cast<double*>(base + 4 * v);
  if (n > 0) {
    launch_rows<1>(Li, n, row, 1, nullptr, 0, 1.0, c0, 1, st);   // c0 = Li row
    launch_rows<1>(L, n, c0, 1, row, 1, -1.0, r, 1, st);         // r = row - L c0
    launch_rows<1>(Li, n, r, 1, c0, 1, 1.0, c, 1, st);           // c = c0 + Li r
  }
  k_pivot<<<1, 256, 0, st>>>(row, c, n, piv);
  RBF_LAUNCH_CHECK("chol append");
  double p2 = 0.0;
  RBF_CUDA_TRY(cudaMemcpyAsync(&p2, piv, sizeof(double), cudaMemcpyDeviceToHost, st));
  RBF_CUDA_TRY(cudaStreamSynchronize(st));
  if (pivot2_host) *pivot2_host = p2;
  if (!(p2 > 0.0))
    return set_error(RBF_ENOTPD, "pivot^2 = %.3e appending row %d; support nodes may coincide or be nearly coincident", p2, n);
  const double l = std::sqrt(p2);
  if (n > 0) launch_cols<1>(Li, n, c, 1, nullptr, 0, 1.0, u, 1, st);  // u = Li^T c
  k_commit<<<(n + 1 + 255) / 256, 256, 0, st>>>(L, Li, n, c, u, l);
  RBF_LAUNCH_CHECK("chol commit");
  return RBF_OK;
}

extern "C" int rbf_chol_solve(const double* L, const double* Li, int64_t n64, const double* rhs,
                              int64_t k, double* out, void* scratch, size_t scratch_bytes,
                              void* stream) {
  if (n64 < 0 || n64 >= INT32_MAX || k < 1) return set_error(RBF_EARG, "bad shape");
  if (n64 == 0) return RBF_OK;
  if (!L || !Li || !rhs || !out || !scratch) return set_error(RBF_EARG, "null pointer");
  const int n = (int)n64;
  const size_t need = 3 * (size_t)n * (size_t)k * sizeof(double);
  if (scratch_bytes < need) return set_error(RBF_EARG, "scratch too small");
  cudaStream_t st = as_stream(stream);
  double* y0 = static_cast<double*>(scratch);
  double* t = y0 + (size_t)n * k;
  double* y = t + (size_t)n * k;
  const int ld = (int)k;
  for (int64_t c0 = 0; c0 < k; c0 += 4) {
    const int kc = (int)((k - c0) < 4 ? (k - c0) : 4);
    // forward: y = Li rhs refined;  back: x = Li^T y refined
    rows_fn(kc)(Li, n, rhs + c0, ld, nullptr, 0, 1.0, y0 + c0, ld, st);
    rows_fn(kc)(L, n, y0 + c0, ld, rhs + c0, ld, -1.0, t + c0, ld, st);
    rows_fn(kc)(Li, n, t + c0, ld, y0 + c0, ld, 1.0, y + c0, ld, st);
    cols_fn(kc)(Li, n, y + c0, ld, nullptr, 0, 1.0, y0 + c0, ld, st);
    cols_fn(kc)(L, n, y0 + c0, ld, y + c0, ld, -1.0, t + c0, ld, st);
    cols_fn(kc)(Li, n, t + c0, ld, y0 + c0, ld, 1.0, out + c0, ld, st);
  }
  RBF_LAUNCH_CHECK("chol solve");
  return RBF_OK;
}

extern "C" size_t rbf_chol_points_scratch_bytes(int64_t n_total) {
  const size_t v = ((size_t)(n_total < 1 ? 1 : n_total) * sizeof(double) + 255) & ~(size_t)255;
  return 5 * v + 256;
}

// Append rows n0 .. n0+k-1 (supports sup[n0 .. n0+k) against every support
// before them) with no host round trip between them: the same kernels as
// rbf_chol_append per row, the pivot test on the device; a failing row stops
// the batch (its kernels and every later row's return at once) and the host
// reads (status, row, pivot^2) once at the end.
extern "C" int rbf_chol_append_points(double* L, double* Li, int64_t n0, int64_t k, const double* sup,
                                      double radius, int64_t* appended_host, double* fail_pivot2_host,
                                      void* scratch, size_t scratch_bytes, void* stream) {
  if (n0 < 0 || k < 0 || n0 + k >= INT32_MAX) return set_error(RBF_EARG, "bad order");
  if (!(radius > 0.0)) return set_error(RBF_EARG, "radius must be positive");
  if (appended_host) *appended_host = 0;
  if (k == 0) return RBF_OK;
  if (!L || !Li || !sup || !scratch) return set_error(RBF_EARG, "null pointer");
  const int ntot = (int)(n0 + k);
  if (scratch_bytes < rbf_chol_points_scratch_bytes(ntot + 1)) return set_error(RBF_EARG, "scratch too small");
  cudaStream_t st = as_stream(stream);
  const size_t v = ((size_t)(ntot + 1) * sizeof(double) + 255) & ~(size_t)255;
  char* base = static_cast<char*>(scratch);
  double* c0 = reinterpret_cast<double*>(base);
  double* r = reinterpret_cast<double*>(base + v);
  double* c = reinterpret_cast<double*>(base + 2 * v);
  double* u = reinterpret_cast<double*>(base + 3 * v);
  double* row = reinterpret_cast<double*>(base + 4 * v);
  double* piv = reinterpret_cast<double*>(base + 5 * v);  // [0] pivot^2, [1..2] failing (pivot^2, row)
  int* status = reinterpret_cast<int*>(base + 5 * v + 64);
  RBF_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int), st));
  for (int n = (int)n0; n < ntot; ++n) {
    k_exact_row<<<(n + 256) / 256, 256, 0, st>>>(sup, n, radius, status, row);
    if (n > 0) {
      launch_rows<1>(Li, n, row, 1, nullptr, 0, 1.0, c0, 1, st);   // c0 = Li row
      launch_rows<1>(L, n, c0, 1, row, 1, -1.0, r, 1, st);         // r = row - L c0
      launch_rows<1>(Li, n, r, 1, c0, 1, 1.0, c, 1, st);           // c = c0 + Li r
    }
    k_pivot_status<<<1, 256, 0, st>>>(row, c, n, piv, status, piv + 1);
    if (n > 0) launch_cols<1>(Li, n, c, 1, nullptr, 0, 1.0, u, 1, st);  // u = Li^T c
    k_commit_dev<<<(n + 1 + 255) / 256, 256, 0, st>>>(L, Li, n, c, u, piv, status);
  }
  RBF_LAUNCH_CHECK("chol append points");
  struct {
    double fail[2];
    int status;
  } h{};
  RBF_CUDA_TRY(cudaMemcpyAsync(&h.fail, piv + 1, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  RBF_CUDA_TRY(cudaMemcpyAsync(&h.status, status, sizeof(int), cudaMemcpyDeviceToHost, st));
  RBF_CUDA_TRY(cudaStreamSynchronize(st));
  if (h.status) {
    if (appended_host) *appended_host = (int64_t)h.fail[1] - n0;
    if (fail_pivot2_host) *fail_pivot2_host = h.fail[0];
    return set_error(RBF_ENOTPD, "pivot^2 = %.3e appending row %d; support nodes may coincide or be nearly coincident",
                     h.fail[0], (int)h.fail[1]);
  }
  if (appended_host) *appended_host = k;
  return RBF_OK;
}
