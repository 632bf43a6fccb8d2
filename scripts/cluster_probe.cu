// Feasibility probe (developer tool): a cooperative launch with thread-block
// clusters of 2 at one CTA per SM and ~227 KB of dynamic smem — how many
// clusters are co-resident, does grid.sync() work inside a cluster launch,
// does a DSMEM store into the peer CTA's smem land.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

// grid barrier without a cooperative launch (the cooperative-groups
// algorithm: block 0 adds 2^31 - (n - 1), the others 1, so the top bit of
// the counter flips once per barrier); needs all CTAs co-resident
__device__ __forceinline__ void grid_bar(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned n = gridDim.x;
    const unsigned add = blockIdx.x == 0 ? 0x80000000u - (n - 1) : 1u;
    __threadfence();
    const unsigned old = atomicAdd(bar, add);
    unsigned cur;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
    } while (((old ^ cur) & 0x80000000u) == 0);
  }
  __syncthreads();
}

__global__ void probe(int* out, int iters, unsigned* gbar, int coop) {
  extern __shared__ int sm[];
  cg::grid_group grid = cg::this_grid();
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  for (int it = 0; it < iters; ++it) {
    sm[threadIdx.x] = -1;
    cl.sync();
    int* peer = cl.map_shared_rank(sm, rank ^ 1);
    peer[threadIdx.x] = (int)(blockIdx.x * 1000 + threadIdx.x + it);
    cl.sync();
    const int expect = (int)((blockIdx.x ^ 1) * 1000 + threadIdx.x + it);
    if (sm[threadIdx.x] != expect) atomicAdd(out, 1);
    if (coop) grid.sync(); else grid_bar(gbar);
  }
  if (threadIdx.x == 0) atomicAdd(out + 1, 1);
}

int main(int argc, char** argv) {
  const int force_ctas = argc > 1 ? atoi(argv[1]) : 0;   // cap the cooperative grid (e.g. under a profiler)
  int coop = argc > 2 ? atoi(argv[2]) : 1;                  // 0: no cooperative attribute, hand-rolled grid barrier
  int dev = 0, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = 227 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int csz : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csz; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(csz * 64);
    int ncl = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, probe, &cfg);
    printf("cluster %d: max active clusters %d (%s) -> %d CTAs of %d SMs\n", csz, ncl, cudaGetErrorString(e),
           ncl * csz, nsm);
    if (ncl <= 0) continue;
    int* out;
    cudaMalloc(&out, 16);
    cudaMemset(out, 0, 16);
    unsigned* gbar = reinterpret_cast<unsigned*>(out + 2);
    if (force_ctas > 0 && force_ctas / csz < ncl) ncl = force_ctas / csz;
    cfg.gridDim = dim3(ncl * csz);
    cfg.numAttrs = coop ? 2 : 1;
    int iters = 100;
    void* args[] = {&out, &iters, &gbar, &coop};
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    e = cudaLaunchKernelExC(&cfg, (const void*)probe, args);
    cudaEventRecord(b);
    cudaError_t e2 = cudaDeviceSynchronize();
    int h[2] = {0, 0};
    cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("  coop+cluster launch of %d CTAs: %s / %s; mismatches %d, CTAs done %d; %.2f us per iter\n", ncl * csz,
           cudaGetErrorString(e), cudaGetErrorString(e2), h[0], h[1], ms * 1e3 / iters);
    cudaFree(out);
  }
  return 0;
}
