// Feasibility probe (developer tool) for the forward split-K reduction through
// distributed shared memory: (1) how many clusters of 4 / 8 / 16 CTAs are
// co-resident at one CTA per SM with ~225 KB of dynamic smem and 256 threads;
// (2) the time of the all-to-all inside a cluster of 8 that the reduction
// needs: every CTA's 4 epilogue warps push 2 x 32 rows x 64 fp32 (8 KB per
// destination, 64 KB per CTA, 7/8 of it remote) with st.shared::cluster.v4,
// then one cluster barrier.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(256, 1) a2a(unsigned long long* out, int iters) {
  extern __shared__ float sm[];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* recv = sm;   // [8 sources][16 n4][32 rows][4]
  unsigned long long t0 = 0, t1 = 0;
  for (int it = 0; it < iters; ++it) {
    cl.sync();
    if (it == iters - 1 && threadIdx.x == 0) t0 = clock64();
    if (warp >= 4) {
      const int ew = warp - 4;
      for (int mt = 0; mt < 2; ++mt) {
        const unsigned dst = 4 * mt + ew;
        float* rb = cl.map_shared_rank(recv, dst) + (size_t)rank * (16 * 32 * 4);
        uint32_t base;
        asm volatile("{ .reg .u64 a; cvta.to.shared.u64 a, %1; cvt.u32.u64 %0, a; }" : "=r"(base) : "l"(recv));
        (void)base;
#pragma unroll 4
        for (int n4 = 0; n4 < 16; ++n4) {
          float4 v = make_float4(rank + n4, lane, mt, it);
          *reinterpret_cast<float4*>(rb + (n4 * 32 + lane) * 4) = v;
        }
      }
    }
    cl.sync();
    if (it == iters - 1 && threadIdx.x == 0) t1 = clock64();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

__global__ void dummy() {}

int main() {
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int smem = 225 * 1024;
  cudaFuncSetAttribute(a2a, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(a2a, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {2, 4, 8, 16}) {
    cudaLaunchConfig_t oc = {};
    oc.gridDim = dim3(cs * 32);
    oc.blockDim = dim3(256);
    oc.dynamicSmemBytes = smem;
    cudaLaunchAttribute ca;
    ca.id = cudaLaunchAttributeClusterDimension;
    ca.val.clusterDim.x = cs; ca.val.clusterDim.y = 1; ca.val.clusterDim.z = 1;
    oc.attrs = &ca;
    oc.numAttrs = 1;
    int ncl = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, (void*)a2a, &oc);
    printf("cluster %2d: max active clusters %3d (%3d CTAs of %d SMs) %s\n", cs, ncl, ncl * cs, nsm,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
    cudaGetLastError();
  }
  unsigned long long* d;
  cudaMalloc(&d, 256 * sizeof(unsigned long long));
  for (int ncl : {1, 16}) {
    cudaLaunchConfig_t c = {};
    c.gridDim = dim3(8 * ncl);
    c.blockDim = dim3(256);
    c.dynamicSmemBytes = smem;
    cudaLaunchAttribute ca;
    ca.id = cudaLaunchAttributeClusterDimension;
    ca.val.clusterDim.x = 8; ca.val.clusterDim.y = 1; ca.val.clusterDim.z = 1;
    c.attrs = &ca;
    c.numAttrs = 1;
    for (int rep = 0; rep < 3; ++rep) {
      cudaError_t e = cudaLaunchKernelEx(&c, a2a, d, 20);
      cudaError_t e2 = cudaDeviceSynchronize();
      unsigned long long h[256];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      unsigned long long mx = 0, sum = 0;
      for (int i = 0; i < 8 * ncl; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
      printf("a2a cluster 8 x %2d: 64 KB per CTA (56 KB remote) + 2 cluster barriers: mean %llu max %llu cycles %s %s\n",
             ncl, sum / (8 * ncl), mx, cudaGetErrorString(e), cudaGetErrorString(e2));
    }
  }
  return 0;
}
