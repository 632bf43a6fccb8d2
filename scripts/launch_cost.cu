// launch_cost.cu — developer microbenchmark: per-launch cost of an (almost)
// empty persistent kernel, 1 CTA/SM with a large dynamic smem request,
// regular vs cooperative launch, with/without grid syncs, stream vs graph.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_cost scripts/launch_cost.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_plain(int* p) { if (threadIdx.x == 0 && p[blockIdx.x] == 12345) p[0] = 1; }
__global__ void k_sync(int* p, int nsync) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < nsync; ++i) g.sync();
  if (threadIdx.x == 0 && p[blockIdx.x] == 12345) p[0] = 1;
}
__global__ void k_tmem(int* p, int nsync) {
  __shared__ unsigned slot;
  cg::grid_group g = cg::this_grid();
  if ((threadIdx.x >> 5) == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"((unsigned)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  for (int i = 0; i < nsync; ++i) g.sync();
  if ((threadIdx.x >> 5) == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(slot));
  if (threadIdx.x == 0 && p[blockIdx.x] == 12345) p[0] = 1;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int* p; cudaMalloc(&p, 4096 * 4); cudaMemset(p, 0, 4096 * 4);
  cudaStream_t st; cudaStreamCreate(&st);
  const size_t smem = 227 * 1024;
  cudaFuncSetAttribute(k_plain, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_sync, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem - 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int N = 2000;
  auto timeit = [&](const char* name, auto fn) {
    for (int i = 0; i < 50; ++i) fn();
    cudaStreamSynchronize(st);
    cudaEventRecord(e0, st);
    for (int i = 0; i < N; ++i) fn();
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-48s %7.2f us/launch  (%s)\n", name, ms * 1e3 / N, cudaGetErrorString(cudaGetLastError()));
  };
  for (size_t sm : {(size_t)0, smem - 1024}) {
    printf("dynamic smem %zu\n", sm);
    timeit("plain <<<nsm,256>>>", [&] { k_plain<<<nsm, 256, sm, st>>>(p); });
    for (int ns : {0, 1, 3, 5}) {
      char nm[96]; snprintf(nm, sizeof nm, "cooperative, %d grid.sync", ns);
      timeit(nm, [&] { void* a[] = {&p, &ns}; cudaLaunchCooperativeKernel((void*)k_sync, nsm, 256, a, sm, st); });
    }
    int ns = 5;
    timeit("cooperative + TMEM alloc, 5 grid.sync", [&] { void* a[] = {&p, &ns}; cudaLaunchCooperativeKernel((void*)k_tmem, nsm, 256, a, sm, st); });
    // graph of 20 cooperative launches
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 20; ++i) { void* a[] = {&p, &ns}; cudaLaunchCooperativeKernel((void*)k_sync, nsm, 256, a, sm, st); }
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int i = 0; i < 5; ++i) cudaGraphLaunch(ge, st);
    cudaStreamSynchronize(st);
    cudaEventRecord(e0, st);
    for (int i = 0; i < 100; ++i) cudaGraphLaunch(ge, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-48s %7.2f us/launch  (%s)\n", "graph of cooperative, 5 grid.sync", ms * 1e3 / 2000, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
