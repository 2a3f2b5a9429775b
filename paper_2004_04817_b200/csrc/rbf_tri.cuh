// Packed lower-triangular matrix-vector products for the growing Cholesky
// factor (reference core.py:115-205 keeps a dense capacity buffer and calls
// LAPACK trsv/trsm; here L and its inverse Li are packed row-major lower
// triangles, row i at offset i*(i+1)/2, so every substitution becomes a
// parallel product with Li and an append is a prefix write).
//
// Matrix loads go through L2 (ld.global.cg): these helpers also run inside
// the persistent selection kernel, where rows are produced by other CTAs
// between grid barriers and must not be served from a stale L1 line. The
// vector operand is read through a caller functor (shared or global memory).
#pragma once
#include "rbf_common.cuh"

namespace rbf {

__host__ __device__ __forceinline__ int64_t tri_off(int64_t i) { return i * (i + 1) / 2; }

// Row products, rows i = gw, gw + nw, ... < n, one warp per row:
//   acc[c] = sum_{j<=i} A[i][j] * xload(j, c),  c < K
// lanes stride j, xor-tree reduction (fixed order: deterministic); lane 0
// then calls finish(i, acc).
template <int K, typename XL, typename F>
__device__ __forceinline__ void tri_rows(const double* A, int n, XL xload, F finish, int gw, int nw,
                                         int lane) {
  for (int i = gw; i < n; i += nw) {
    const double* a = A + tri_off(i);
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.0;
    for (int j = lane; j <= i; j += kWarp) {
      const double aij = __ldcg(a + j);
#pragma unroll
      for (int c = 0; c < K; ++c) acc[c] = fma(aij, xload(j, c), acc[c]);
    }
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = warp_sum(acc[c]);
    if (lane == 0) finish(i, acc);
  }
}

// Column products over 32-column slabs J = slab0, slab0 + nslab, ...:
//   sum[c] = sum_{i=j}^{n-1} A[i][j] * xload(i, c),  c < K
// computed by one CTA per slab: its NW warps split the rows, the partials are
// folded in warp order through shared memory `red` (NW*32*K doubles); warp 0
// lane (j - 32J) then calls emit(j, sum).
template <int K, int NW, typename XL, typename Emit>
__device__ __forceinline__ void tri_cols(const double* A, int n, XL xload, int slab0, int nslab,
                                         double* red, Emit emit) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nslabs_total = (n + 31) / 32;
  for (int J = slab0; J < nslabs_total; J += nslab) {
    const int j = 32 * J + lane;
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.0;
    // U rows per batch: every load of the batch is issued before its FMAs
    constexpr int U = K >= 4 ? 4 : 8;
    for (int i0 = 32 * J + warp; i0 < n; i0 += U * NW) {
      double av[U], xv[U][K];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * NW;
        const bool ok = i < n && j <= i;
        av[u] = ok ? __ldcg(A + tri_off(i) + j) : 0.0;
#pragma unroll
        for (int c = 0; c < K; ++c) xv[u][c] = (i < n) ? xload(i, c) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int c = 0; c < K; ++c) acc[c] = fma(av[u], xv[u][c], acc[c]);
      }
    }
#pragma unroll
    for (int c = 0; c < K; ++c) red[(warp * 32 + lane) * K + c] = acc[c];
    __syncthreads();
    if (warp == 0 && j < n) {
      double sum[K];
#pragma unroll
      for (int c = 0; c < K; ++c) sum[c] = red[lane * K + c];
      for (int w = 1; w < NW; ++w) {
#pragma unroll
        for (int c = 0; c < K; ++c) sum[c] += red[(w * 32 + lane) * K + c];
      }
      emit(j, sum);
    }
    __syncthreads();
  }
}

}  // namespace rbf
