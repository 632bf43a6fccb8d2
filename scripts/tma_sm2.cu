// tma_sm2.cu — developer microbenchmark: per-SM TMA streaming rate vs box
// height (128 / 256 rows of 128 B), boxes per stage, stage count and the
// number of producer threads per CTA (independent pipelines), for a grid of
// G CTAs each streaming a disjoint row strip of a 512 MiB bf16 matrix.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_sm2 scripts/tma_sm2.cu -lcuda
#include <cstdio>
#include "../paper_2206_04993_b200/csrc/tc_gemm.cuh"

using namespace geig::tc;

__global__ void __launch_bounds__(128) sm_stream2(const __grid_constant__ CUtensorMap map, int BH, int rows_per_cta,
                                                  int NB, int S, int NP, unsigned long long* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const uint32_t BOX = 128u * BH;
  const uint32_t STAGE = BOX * NB;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NP * S * STAGE);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NP * S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int pr = threadIdx.x / 32;            // producer pr = lane 0 of warp pr
  if ((threadIdx.x & 31) != 0 || pr >= NP) return;
  uint8_t* sm = smem + pr * S * STAGE;
  uint64_t* fb = full + pr * S;
  const int r0 = blockIdx.x * rows_per_cta;
  const int nk = 8192 / 64;
  const int rows_pp = rows_per_cta / NP;      // each producer: its own rows
  const int nsteps = (rows_pp / (BH * NB)) * nk;
  unsigned long long acc = 0;
  for (int it = 0; it < nsteps + S; ++it) {
    if (it >= S) {
      const int j = it - S;
      mbar_wait(&fb[j % S], (j / S) & 1);
      acc += sm[(j % S) * STAGE + 5];
    }
    if (it < nsteps) {
      const int st = it % S;
      mbar_expect_tx(&fb[st], STAGE);
      const int kb = it % nk, rb = it / nk;
      for (int q = 0; q < NB; ++q)
        tma_load_2d(sm + st * STAGE + q * BOX, &map, &fb[st], kb * 64, r0 + pr * rows_pp + (rb * NB + q) * BH);
    }
  }
  if (acc == 12345) sink[0] = acc;
}

int main() {
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  const int R = 32768, C = 8192;
  void* X;
  cudaMalloc(&X, (size_t)R * C * 2);
  cudaMemset(X, 1, (size_t)R * C * 2);
  CUtensorMap m128, m256;
  make_map(&m128, X, 2, C, R, C, 64, 128);
  make_map(&m256, X, 2, C, R, C, 64, 256);
  cudaFuncSetAttribute(sm_stream2, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  struct Cfg { int BH, NB, S, NP; };
  const Cfg cfgs[] = {{128, 2, 4, 1}, {256, 1, 4, 1}, {256, 2, 3, 1}, {128, 4, 3, 1}, {256, 3, 2, 1},
                      {128, 1, 4, 2}, {128, 2, 3, 2}, {256, 1, 3, 2}, {128, 1, 3, 4}, {128, 2, 2, 4}, {64, 4, 4, 2}};
  for (const Cfg& c : cfgs) {
    const size_t stage = 128u * c.BH * c.NB;
    const size_t sm = 1024 + (size_t)c.NP * c.S * stage + 512;
    if (sm > 227 * 1024) continue;
    CUtensorMap* mp = c.BH == 256 ? &m256 : &m128;
    if (c.BH == 64) { static CUtensorMap m64; make_map(&m64, X, 2, C, R, C, 64, 64); mp = &m64; }
    for (int G : {32, 64, 96, 128}) {
      const int unit = c.BH * c.NB * c.NP;
      const int rpc = (R / G) / unit * unit;
      if (rpc == 0) continue;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      for (int w = 0; w < 2; ++w) sm_stream2<<<G, 128, sm>>>(*mp, c.BH, rpc, c.NB, c.S, c.NP, sink);
      cudaEventRecord(e0);
      const int reps = 5;
      for (int w = 0; w < reps; ++w) sm_stream2<<<G, 128, sm>>>(*mp, c.BH, rpc, c.NB, c.S, c.NP, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = (double)G * rpc * C * 2;
      printf("box 64x%3d NB %d S %d producers %d (%3zu KB in flight) grid %3d : %7.1f GB/s  per-SM %6.1f GB/s\n", c.BH, c.NB,
             c.S, c.NP, c.NP * c.S * stage / 1024, G, bytes / (ms / reps * 1e-3) / 1e9,
             bytes / G / (ms / reps * 1e-3) / 1e9);
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  return 0;
}
