// Feasibility probe (developer tool): a cooperative launch with thread-block
// clusters of 2 at one CTA per SM and ~227 KB of dynamic smem — how many
// clusters are co-resident, does grid.sync() work inside a cluster launch,
// does a DSMEM store into the peer CTA's smem land.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void probe(int* out, int iters) {
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
    grid.sync();
  }
  if (threadIdx.x == 0) atomicAdd(out + 1, 1);
}

int main() {
  int dev = 0, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = 227 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int csz : {2, 4, 8}) {
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
    cudaMalloc(&out, 8);
    cudaMemset(out, 0, 8);
    cfg.gridDim = dim3(ncl * csz);
    cfg.numAttrs = 2;
    int iters = 100;
    void* args[] = {&out, &iters};
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
