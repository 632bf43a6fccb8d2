// tma_bw.cu — developer microbenchmark: DRAM streaming bandwidth of TMA
// tile loads of a row-major bf16 matrix [R x C] for different box shapes,
// stage counts and traversal orders (no math).  Guides the product kernels'
// tiling.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -o tma_bw scripts/tma_bw.cu
#include <cstdio>
#include <vector>
#include "../paper_2206_04993_b200/csrc/tc_gemm.cuh"

using namespace geig::tc;

// each CTA: rows [r0, r0 + RB) x all columns in boxes of (64 cols x BH rows);
// per stage NB boxes adjacent along columns.  ORDER 0: CTA walks columns of
// its row strip (like the forward GEMM); ORDER 1: CTA walks rows of a column strip.
template <int BH, int NB, int S, int ORDER, int SPLIT, int BROWS = 0>
__global__ void __launch_bounds__(128) stream_kernel(const __grid_constant__ CUtensorMap map,
                                                    const __grid_constant__ CUtensorMap mapb, int R, int C,
                                                    int strips, unsigned long long* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  constexpr uint32_t BOX = 128 * BH;
  constexpr uint32_t STAGE = BOX * NB + 128 * BROWS * NB;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * STAGE);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int nsteps, r_fix = 0, c_fix = 0, off = 0;
  const int sp = blockIdx.x % SPLIT, bx = blockIdx.x / SPLIT;
  if (ORDER == 0) { r_fix = bx * BH; nsteps = C / (64 * NB) / SPLIT; off = sp * nsteps; }
  else { c_fix = bx * 64 * NB; nsteps = R / BH / SPLIT; off = sp * nsteps; }
  unsigned long long acc = 0;
  for (int it = 0; it < nsteps + S; ++it) {
    if (it >= S) {
      const int j = it - S;
      mbar_wait(&full[j % S], (j / S) & 1);
      acc += smem[(j % S) * STAGE + (threadIdx.x & 63)];
    }
    if (it < nsteps) {
      const int st = it % S;
      mbar_expect_tx(&full[st], STAGE);
      for (int q = 0; q < NB; ++q) {
        int c, r;
        if (ORDER == 0) { c = ((it + off) * NB + q) * 64; r = r_fix; }
        else { c = c_fix + q * 64; r = (it + off) * BH; }
        tma_load_2d(smem + st * STAGE + q * BOX, &map, &full[st], c, r);
        if (BROWS) tma_load_2d(smem + st * STAGE + NB * BOX + q * 128 * BROWS, &mapb, &full[st], c, 0);
      }
    }
  }
  if (acc == 12345) sink[0] = acc;
}

template <int BH, int NB, int S, int ORDER, int SPLIT, int BROWS = 0>
void run(const void* X, int R, int C, unsigned long long* sink) {
  CUtensorMap map, mapb;
  if (!make_map(&map, X, 2, C, R, C, 64, BH)) { printf("map failed\n"); return; }
  if (!make_map(&mapb, X, 2, C, 64, C, 64, BROWS ? BROWS : 64)) { printf("map failed\n"); return; }
  size_t sm = 1024 + (size_t)S * (128 * BH * NB + 128 * BROWS * NB) + 256;
  if (getenv("ONE_CTA_PER_SM")) sm = 200 * 1024;
  cudaFuncSetAttribute(stream_kernel<BH, NB, S, ORDER, SPLIT, BROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const int grid = (ORDER == 0 ? R / BH : C / (64 * NB)) * SPLIT;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) stream_kernel<BH, NB, S, ORDER, SPLIT, BROWS><<<grid, 128, sm>>>(map, mapb, R, C, grid, sink);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int w = 0; w < reps; ++w) stream_kernel<BH, NB, S, ORDER, SPLIT, BROWS><<<grid, 128, sm>>>(map, mapb, R, C, grid, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)R * C * 2;
  printf("order %d split %d box 64x%-3d x%d stages %2d grid %4d smem %6zu : %7.1f GB/s (%.1f us)\n", ORDER, SPLIT, BH, NB, S,
         grid, sm, bytes / (ms / reps * 1e-3) / 1e9, ms / reps * 1e3);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
}

int main() {
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  for (int R : {8192, 4096, 2048}) {
    const int C = 8192;
    void* X;
    cudaMalloc(&X, (size_t)R * C * 2);
    cudaMemset(X, 1, (size_t)R * C * 2);
    printf("R=%d (%d MiB): back-to-back reps (L2 reuse when the matrix fits)\n", R, R * C * 2 >> 20);
    run<128, 2, 6, 0, 2>(X, R, C, sink);
    run<64, 1, 12, 1, 1>(X, R, C, sink);
    cudaFree(X);
  }
  return 0;
}
