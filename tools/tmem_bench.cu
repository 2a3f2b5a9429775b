// TMEM access latency from a plain (non-MMA) kernel: tcgen05.st / tcgen05.ld
// of 32x32b.x{8,16,32} followed by the matching wait, per warp, clock64.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_bench tools/tmem_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int W>
__global__ void k(long long* out, int iters) {
  __shared__ unsigned base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&base)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tl = base + ((unsigned)(32 * (warp & 3)) << 16) + (warp >> 2) * 64;
  unsigned r[32];
  for (int i = 0; i < 32; ++i) r[i] = threadIdx.x * 32 + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (W == 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tl), "r"(r[0]), "r"(r[1]),
                   "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    r[0] += 1;
  }
  long long t1 = clock64();
  for (int it = 0; it < iters; ++it) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tl + (r[7] & 1)) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  }
  long long t2 = clock64();
  for (int it = 0; it < iters; ++it) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(tl + (r[31] & 1)) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  }
  long long t3 = clock64();
  unsigned acc = 0;
  for (int i = 0; i < 32; ++i) acc += r[i];
  if ((threadIdx.x & 31) == 0) {
    out[4 * warp] = (t1 - t0) / iters;
    out[4 * warp + 1] = (t2 - t1) / iters;
    out[4 * warp + 2] = (t3 - t2) / iters;
    out[4 * warp + 3] = acc;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base) : "memory");
}

int main() {
  long long* d;
  cudaMalloc(&d, 64 * 8);
  long long h[64];
  for (int warps : {1, 4, 16}) {
    k<8><<<1, 32 * warps>>>(d, 1000);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 64 * 8, cudaMemcpyDeviceToHost);
    printf("warps %2d: st.x8+wait %lld cyc, ld.x8+wait %lld cyc, ld.x32+wait %lld cyc  (%s)\n", warps, h[0], h[1], h[2],
           cudaGetErrorString(e));
  }
  return 0;
}
