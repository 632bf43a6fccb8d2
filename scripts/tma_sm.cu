// tma_sm.cu — developer microbenchmark: aggregate DRAM streaming bandwidth of
// TMA tile loads vs the number of streaming CTAs (one per SM), i.e. how many
// SMs one GEMM phase needs to saturate HBM.  Each CTA streams a disjoint
// column strip of a row-major bf16 matrix in 128 x 64 boxes (16 KB), NB boxes
// per stage, S stages, plus an optional re-read 16 KB "operand" tile per
// stage from a small L2-resident buffer (like the V / Z tiles).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_sm scripts/tma_sm.cu -lcuda
#include <cstdio>
#include <vector>
#include "../paper_2206_04993_b200/csrc/tc_gemm.cuh"

using namespace geig::tc;

__global__ void __launch_bounds__(128) sm_stream(const __grid_constant__ CUtensorMap map,
                                                 const __grid_constant__ CUtensorMap mapb, int rows_per_cta,
                                                 int NB, int S, int opnd, unsigned long long* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const uint32_t STAGE = 16384u * NB + (opnd ? 16384u : 0u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * STAGE);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  // CTA b: rows [b*rows_per_cta, ...), all 8192 columns (128 K blocks of 64)
  const int r0 = blockIdx.x * rows_per_cta;
  const int nk = 8192 / 64;
  const int nsteps = (rows_per_cta / (128 * NB)) * nk;
  unsigned long long acc = 0;
  for (int it = 0; it < nsteps + S; ++it) {
    if (it >= S) {
      const int j = it - S;
      mbar_wait(&full[j % S], (j / S) & 1);
      acc += smem[(j % S) * STAGE + 5];
    }
    if (it < nsteps) {
      const int st = it % S;
      mbar_expect_tx(&full[st], STAGE);
      const int kb = it % nk, rb = it / nk;
      for (int q = 0; q < NB; ++q)
        tma_load_2d(smem + st * STAGE + q * 16384, &map, &full[st], kb * 64, r0 + (rb * NB + q) * 128);
      if (opnd) tma_load_2d(smem + st * STAGE + NB * 16384, &mapb, &full[st], kb * 64, 0);
    }
  }
  if (acc == 12345) sink[0] = acc;
}

int main() {
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  const int R = 32768, C = 8192;   // 512 MiB
  void *X, *B;
  cudaMalloc(&X, (size_t)R * C * 2);
  cudaMemset(X, 1, (size_t)R * C * 2);
  cudaMalloc(&B, (size_t)128 * C * 2);
  cudaMemset(B, 1, (size_t)128 * C * 2);
  CUtensorMap map, mapb;
  make_map(&map, X, 2, C, R, C, 64, 128);
  make_map(&mapb, B, 2, C, 128, C, 64, 128);
  cudaFuncSetAttribute(sm_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (int opnd = 0; opnd < 2; ++opnd)
    for (int NB : {1, 2})
      for (int S : {3, 4, 6}) {
        const size_t stage = 16384u * NB + (opnd ? 16384u : 0u);
        const size_t sm = 1024 + S * stage + 256;
        if (sm > 227 * 1024) continue;
        for (int G : {32, 48, 64, 96, 128, 148}) {
          // rows per CTA: a multiple of 128 * NB covering ~R / G rows... use fixed bytes per CTA
          int rpc = (R / G) / (128 * NB) * (128 * NB);
          if (rpc == 0) continue;
          cudaEvent_t e0, e1;
          cudaEventCreate(&e0); cudaEventCreate(&e1);
          for (int w = 0; w < 2; ++w) sm_stream<<<G, 128, sm>>>(map, mapb, rpc, NB, S, opnd, sink);
          cudaEventRecord(e0);
          const int reps = 5;
          for (int w = 0; w < reps; ++w) sm_stream<<<G, 128, sm>>>(map, mapb, rpc, NB, S, opnd, sink);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e1);
          const double bytes = (double)G * rpc * C * 2;
          const double opb = opnd ? (double)G * (rpc / (128 * NB)) * 128 * 16384 : 0;
          printf("opnd %d NB %d S %d grid %3d : X %7.1f GB/s  (+operand %6.1f GB/s) per-SM %5.1f GB/s\n", opnd, NB, S, G,
                 bytes / (ms / reps * 1e-3) / 1e9, opb / (ms / reps * 1e-3) / 1e9,
                 (bytes + opb) / G / (ms / reps * 1e-3) / 1e9);
        }
      }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  return 0;
}
