// Microbenchmark: grid-wide software barrier (as in rbf_common.cuh) vs.
// hardware cluster barrier, on the B200. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier_bench barrier_bench.cu
#include <cstdio>
#include <cooperative_groups.h>
#include "../paper_2004_04817_b200/csrc/rbf_common.cuh"
namespace cg = cooperative_groups;

__global__ void grid_bar_kernel(rbf::GridBarrier* bar, int* fault, int iters, unsigned long long* out) {
  unsigned long long t0 = rbf::globaltimer_ns();
  for (int i = 0; i < iters; ++i) rbf::grid_sync(bar, gridDim.x, fault);
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = rbf::globaltimer_ns() - t0;
}

__global__ void cg_grid_kernel(int iters, unsigned long long* out) {
  cg::grid_group g = cg::this_grid();
  unsigned long long t0 = rbf::globaltimer_ns();
  for (int i = 0; i < iters; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[1] = rbf::globaltimer_ns() - t0;
}

__global__ void cluster_bar_kernel(int iters, unsigned long long* out, int slot) {
  cg::cluster_group c = cg::this_cluster();
  unsigned long long t0 = rbf::globaltimer_ns();
  for (int i = 0; i < iters; ++i) c.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[slot] = rbf::globaltimer_ns() - t0;
}

// L2 latency: dependent pointer chase over a small array (stays in L2)
__global__ void chase_kernel(const int* next, int steps, unsigned long long* out, int* sink) {
  int p = 0;
  unsigned long long t0 = rbf::globaltimer_ns();
  for (int i = 0; i < steps; ++i) p = __ldcg(next + p);
  out[5] = rbf::globaltimer_ns() - t0;
  sink[0] = p;
}

__global__ void timer_kernel(unsigned long long* out, int iters) {
  unsigned long long acc = 0;
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) acc += rbf::globaltimer_ns();
  long long c1 = clock64();
  for (int i = 0; i < iters; ++i) acc += clock64();
  long long c2 = clock64();
  out[6] = (unsigned long long)(c1 - c0);
  out[7] = (unsigned long long)(c2 - c1) + (acc & 1);
}

// DSMEM: each CTA stores 1 double into every CTA of the cluster, then syncs
__global__ void dsmem_kernel(int iters, unsigned long long* out) {
  __shared__ double buf[16];
  cg::cluster_group c = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x < 16) *c.map_shared_rank(&buf[blockIdx.x % 16], threadIdx.x) = (double)i;
    c.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[4] = (unsigned long long)(clock64() - t0);
}

// st.async + mbarrier: each CTA pushes one double into every CTA (16 x 8 B
// per CTA per round) and waits on its own mbarrier for the 16 incoming.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__global__ void stasync_kernel(int iters, unsigned long long* out) {
  __shared__ double buf[2][16];
  __shared__ __align__(8) unsigned long long mbar[2];
  cg::cluster_group c = cg::this_cluster();
  const unsigned rank = c.block_rank();
  if (threadIdx.x < 2) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&mbar[threadIdx.x])));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  c.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const int b = i & 1;
    const unsigned parity = (i >> 1) & 1;
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&mbar[b])), "r"(16 * 8) : "memory");
    }
    if (threadIdx.x < 16) {
      // remote addresses of buf[b][rank] and mbar[b] in CTA threadIdx.x
      unsigned laddr = smem_u32(&buf[b][rank]);
      unsigned lbar = smem_u32(&mbar[b]);
      unsigned raddr, rbar;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(laddr), "r"(threadIdx.x));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(lbar), "r"(threadIdx.x));
      double v = (double)i;
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
                   :: "r"(raddr), "d"(v), "r"(rbar) : "memory");
    }
    // wait for this round's 16 values
    unsigned done = 0;
    while (!done) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(smem_u32(&mbar[b])), "r"(parity) : "memory");
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[3] = (unsigned long long)(clock64() - t0);
  c.sync();
}

// all-to-all volume test: each CTA pushes `per` values (8 B each, or 16 B
// pairs) to every CTA per round, spread over threads; waits for its own.
template <bool V2>
__global__ void stasync_volume_kernel(int iters, int per, unsigned long long* out, int slot) {
  __shared__ double buf[16 * 64];
  __shared__ __align__(8) unsigned long long mbar[2];
  cg::cluster_group c = cg::this_cluster();
  const unsigned rank = c.block_rank();
  if (threadIdx.x < 2) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&mbar[threadIdx.x])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  c.sync();
  const int msgs = V2 ? per / 2 : per;   // per destination
  const unsigned bytes_in = 16 * per * 8;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const int b = i & 1;
    const unsigned parity = (i >> 1) & 1;
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&mbar[b])), "r"(bytes_in) : "memory");
    for (int e = threadIdx.x; e < 16 * msgs; e += blockDim.x) {
      const int dst = e % 16, k = e / 16;
      unsigned raddr, rbar;
      const unsigned laddr = smem_u32(&buf[rank * 64 + (V2 ? 2 * k : k)]);
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(laddr), "r"(dst));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(&mbar[b])), "r"(dst));
      const double v = (double)i;
      if (V2)
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" :: "r"(raddr), "d"(v), "d"(v), "r"(rbar) : "memory");
      else
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" :: "r"(raddr), "d"(v), "r"(rbar) : "memory");
    }
    unsigned done = 0;
    while (!done) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(smem_u32(&mbar[b])), "r"(parity) : "memory");
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[slot] = (unsigned long long)(clock64() - t0);
  c.sync();
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  rbf::GridBarrier* bar; int* fault; unsigned long long* out;
  cudaMalloc(&bar, 64); cudaMemset(bar, 0, 64); cudaMalloc(&fault, 4); cudaMalloc(&out, 64);
  cudaMemset(out, 0, 64);
  int iters = 20000;
  void* a1[] = {&bar, &fault, &iters, &out};
  cudaLaunchCooperativeKernel((void*)grid_bar_kernel, sms, 512, a1, 0, 0);
  void* a2[] = {&iters, &out};
  cudaLaunchCooperativeKernel((void*)cg_grid_kernel, sms, 512, a2, 0, 0);
  for (int cs : {8, 16}) {
    cudaFuncSetAttribute(cluster_bar_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs); cfg.blockDim = dim3(512);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int slot = cs == 8 ? 2 : 3;
    cudaError_t e = cudaLaunchKernelEx(&cfg, cluster_bar_kernel, iters, out, slot);
    if (e != cudaSuccess) printf("cluster %d launch: %s\n", cs, cudaGetErrorString(e));
  }
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16); cfg.blockDim = dim3(512);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaFuncSetAttribute(dsmem_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchKernelEx(&cfg, dsmem_kernel, iters, out);
  }
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16); cfg.blockDim = dim3(512);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaFuncSetAttribute(stasync_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaError_t e2 = cudaLaunchKernelEx(&cfg, stasync_kernel, iters, out);
    if (e2 != cudaSuccess) printf("stasync launch: %s\n", cudaGetErrorString(e2));
  }
  unsigned long long* out2; cudaMalloc(&out2, 16 * 8); cudaMemset(out2, 0, 16 * 8);
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16); cfg.blockDim = dim3(512);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaFuncSetAttribute(stasync_volume_kernel<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(stasync_volume_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int pers[4] = {2, 8, 18, 28};
    for (int q = 0; q < 4; ++q) {
      cudaLaunchKernelEx(&cfg, stasync_volume_kernel<false>, 2000, pers[q], out2, q);
      cudaLaunchKernelEx(&cfg, stasync_volume_kernel<true>, 2000, pers[q], out2, 4 + q);
    }
  }
  timer_kernel<<<1, 1>>>(out, 1000);
  int n = 1 << 16; int* next; cudaMalloc(&next, n * 4);
  int* h = new int[n]; for (int i = 0; i < n; ++i) h[i] = (i * 7919 + 13) % n;
  cudaMemcpy(next, h, n * 4, cudaMemcpyHostToDevice);
  int* sink; cudaMalloc(&sink, 4);
  chase_kernel<<<1, 1>>>(next, 20000, out, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long r[8]; cudaMemcpy(r, out, 64, cudaMemcpyDeviceToHost);
  printf("status %s\n", cudaGetErrorString(e));
  printf("grid barrier (ours, %d CTAs x 512): %.3f us/barrier\n", sms, r[0] / 1e3 / iters);
  printf("grid barrier (cg::grid.sync):        %.3f us/barrier\n", r[1] / 1e3 / iters);
  printf("cluster barrier (8 CTAs):            %.3f us/barrier\n", r[2] / 1e3 / iters);
  printf("st.async x16 + mbarrier wait:        %.1f cycles/round\n", r[3] / (double)iters);
  printf("L2 dependent load latency:           %.1f ns\n", r[5] / 20000.0);
  printf("DSMEM store x16 + cluster sync:      %.1f cycles\n", r[4] / (double)iters);
  {
    unsigned long long r2[16]; cudaMemcpy(r2, out2, 16 * 8, cudaMemcpyDeviceToHost);
    int pers[4] = {2, 8, 18, 28};
    for (int q = 0; q < 4; ++q)
      printf("all-to-all %2d doubles/CTA-pair: b64 %.0f cyc, v2 %.0f cyc per round\n", pers[q], r2[q] / 2000.0, r2[4 + q] / 2000.0);
  }
  printf("globaltimer read:                    %.1f cycles\n", r[6] / 1000.0);
  printf("clock64 read:                        %.1f cycles\n", r[7] / 1000.0);
  return 0;
}
