// Grid-wide barrier variants on 148 CTAs x 512 threads (the selection
// kernel's L2-path team). Build:
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gridbar_bench tools/gridbar_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_release(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

template <int V>
__device__ __forceinline__ void bar(unsigned* word) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned add = blockIdx.x == 0 ? (0x80000000u - (gridDim.x - 1)) : 1u;
    unsigned old;
    if (V == 0) { __threadfence(); old = atomicAdd(word, add); }
    else if (V == 1) { old = atom_add_release(word, add); }
    else { old = atom_add_acqrel(word, add); }
    while (((old ^ ld_acq(word)) & 0x80000000u) == 0) {
      if (V == 3) __nanosleep(32);
    }
    if (V == 0) __threadfence();
  }
  __syncthreads();
}

// fire-and-forget arrival (red.release): the expected bit-31 state is tracked
// locally (a parity flip per barrier), so the poll starts right away
__device__ __forceinline__ void bar_red(unsigned* word, unsigned& parity) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned add = blockIdx.x == 0 ? (0x80000000u - (gridDim.x - 1)) : 1u;
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(word), "r"(add) : "memory");
    parity ^= 0x80000000u;
    while ((ld_acq(word) & 0x80000000u) != parity) __nanosleep(32);
  }
  __syncthreads();
}

__global__ void kbar_red(unsigned* word, int iters, unsigned long long* out) {
  unsigned parity = 0;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) bar_red(word, parity);
  if (blockIdx.x == 0 && threadIdx.x == 0) out[4] = clock64() - t0;
}

template <int V>
__global__ void kbar(unsigned* word, int iters, unsigned long long* out) {
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) bar<V>(word);
  if (blockIdx.x == 0 && threadIdx.x == 0) out[V] = clock64() - t0;
}
__global__ void kcg(int iters, unsigned long long* out) {
  cg::grid_group g = cg::this_grid();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[7] = clock64() - t0;
}

int main(int argc, char** argv) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (argc > 1) sms = atoi(argv[1]);  // CTA count to test
  unsigned* word; unsigned long long* out;
  cudaMalloc(&word, 64); cudaMalloc(&out, 64); cudaMemset(out, 0, 64);
  int iters = 20000;
  auto run = [&](void* k, int slot) {
    cudaMemset(word, 0, 64);
    void* args[] = {&word, &iters, &out};
    cudaError_t e = cudaLaunchCooperativeKernel(k, sms, 512, args, 0, 0);
    if (e) printf("launch %d: %s\n", slot, cudaGetErrorString(e));
  };
  run((void*)kbar<0>, 0); run((void*)kbar<1>, 1); run((void*)kbar<2>, 2); run((void*)kbar<3>, 3);
  run((void*)kbar_red, 4);
  void* a2[] = {&iters, &out};
  cudaLaunchCooperativeKernel((void*)kcg, sms, 512, a2, 0, 0);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long r[8]; cudaMemcpy(r, out, 64, cudaMemcpyDeviceToHost);
  printf("status %s (cycles per barrier, %d CTAs x 512)\n", cudaGetErrorString(e), sms);
  const char* names[] = {"fence+atomicAdd (GridTeam)", "atom.add.release", "atom.add.acq_rel", "release + nanosleep"};
  for (int v = 0; v < 4; ++v) printf("%-28s %8.0f\n", names[v], r[v] / (double)iters);
  printf("%-28s %8.0f\n", "red.release, local parity", r[4] / (double)iters);
  printf("%-28s %8.0f\n", "cg::grid.sync", r[7] / (double)iters);
}
