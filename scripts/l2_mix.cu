// l2_mix.cu — developer microbenchmark: can a chunked schedule read the batch
// from DRAM once and re-read it from L2 (the backward pass) at a combined rate
// above one DRAM pass?  Each CTA walks chunks of CH rows; per tile it loads
// tile j of chunk c (first touch, DRAM) and tile j of chunk c-LAG (expected
// L2 hit).  No math.  Compared with one pass and two sequential passes over
// the same 128 MiB matrix (a ring of 4 matrices defeats L2 between reps).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda
//   -o l2_mix scripts/l2_mix.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2206_04993_b200/csrc/tc_gemm.cuh"

using namespace geig::tc;

constexpr int BH = 128, BOXB = 128 * BH;   // box 64 cols x 128 rows = 16 KB

// mode 0: one pass; 1: mixed (first touch + re-read of chunk c-LAG); 2: two sequential passes
template <int S>
__global__ void __launch_bounds__(128) mix_kernel(const __grid_constant__ CUtensorMap map, int R, int C, int CH,
                                                  int mode, int lag, unsigned long long* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * BOXB);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint64_t pol_first = l2_policy_evict_first(), pol_last = l2_policy_evict_last();
  const int tpr = C / 64;                       // tiles per 128-row strip
  const int tiles_per_chunk = (CH / BH) * tpr;
  const int nch = R / CH;
  // this CTA's tiles in a chunk: j = blockIdx.x, +gridDim.x, ...
  const int myn = (tiles_per_chunk - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  // load list: (chunk, j, policy)
  int total;
  if (mode == 0) total = nch * myn;
  else total = 2 * nch * myn + (mode == 1 ? 0 : 0);
  unsigned long long acc = 0;
  for (int it = 0; it < total + S; ++it) {
    if (it >= S) {
      const int j = it - S;
      mbar_wait(&full[j % S], (j / S) & 1);
      acc += smem[(j % S) * BOXB + (threadIdx.x & 63)];
    }
    if (it < total) {
      int ch, jj;
      uint64_t pol;
      if (mode == 0) { ch = it / myn; jj = it % myn; pol = pol_first; }
      else if (mode == 2) {
        const int pass = it / (nch * myn), r = it % (nch * myn);
        ch = r / myn; jj = r % myn; pol = pass == 0 ? pol_last : pol_first;
      } else {
        // chunk-major interleave: for step s in [0, nch + lag): first-touch loads of chunk s and
        // re-reads of chunk s - lag, alternating tile by tile
        const int per = 2 * myn;
        const int s = it / per, r = it % per;
        const int fr = r & 1;          // 0: first touch, 1: re-read
        jj = r >> 1;
        ch = fr ? s - lag : s;
        pol = fr ? pol_first : pol_last;
        if (ch < 0 || ch >= nch) { ch = -1; }
      }
      const int st = it % S;
      if (ch < 0) ch = it / (2 * myn);   // first lag steps: re-read the chunk just touched
      const int t = jj * gridDim.x + blockIdx.x;
      const int strip = t / tpr, col = t % tpr;
      mbar_expect_tx(&full[st], BOXB);
      tma_load_2d_hint(smem + st * BOXB, &map, &full[st], col * 64, ch * CH + strip * BH, pol);
    }
  }
  if (acc == 12345) sink[0] = acc;
}

template <int S>
void run(const std::vector<void*>& mats, int R, int C, int CH, int mode, int lag, int grid, unsigned long long* sink) {
  std::vector<CUtensorMap> maps(mats.size());
  for (size_t i = 0; i < mats.size(); ++i)
    if (!make_map(&maps[i], mats[i], 2, C, R, C, 64, BH)) { printf("map failed\n"); return; }
  size_t sm = 1024 + (size_t)S * BOXB + 256;
  cudaFuncSetAttribute(mix_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (mode == 1) {
    // mixed mode covers nch + lag chunk steps; the re-read tail past the end is padded
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 4; ++w) mix_kernel<S><<<grid, 128, sm>>>(maps[w % maps.size()], R, C, CH, mode, lag, sink);
  cudaEventRecord(e0);
  const int reps = 12;
  for (int w = 0; w < reps; ++w) mix_kernel<S><<<grid, 128, sm>>>(maps[w % maps.size()], R, C, CH, mode, lag, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = ms / reps * 1e3;
  const double bytes = (double)R * C * 2;
  const double moved = mode == 0 ? bytes : 2 * bytes;
  printf("mode %d CH %5d (%3d MiB) lag %d grid %3d S %2d : %7.2f us  matrix-rate %7.1f GB/s  moved-rate %7.1f GB/s\n", mode,
         CH, (int)((double)CH * C * 2 / (1 << 20)), lag, grid, S, us, bytes / us * 1e-3, moved / us * 1e-3);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
}


// F-phase pattern: each CTA owns a 128*TMX-row strip of the matrix and a
// K range (split sp of SPLIT); per stage TMX X boxes (16 KB each, rows m0 +
// 128 j) plus VB boxes of a small L2-resident "V" matrix (16 KB each) at the
// same column.  grid = (R / (128 TMX)) * SPLIT.
template <int S, int TMX, int VB>
__global__ void __launch_bounds__(128) fwd_kernel(const __grid_constant__ CUtensorMap map,
                                                  const __grid_constant__ CUtensorMap vmap, int R, int C, int split,
                                                  unsigned long long* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  constexpr uint32_t STAGE = (TMX + VB) * BOXB;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * STAGE);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint64_t pol_first = l2_policy_evict_first(), pol_last = l2_policy_evict_last();
  const int strip = blockIdx.x / split, sp = blockIdx.x % split;
  const int kb = C / 64, kb0 = kb * sp / split, kbn = kb * (sp + 1) / split - kb0;
  unsigned long long acc = 0;
  for (int it = 0; it < kbn + S; ++it) {
    if (it >= S) {
      const int j = it - S;
      mbar_wait(&full[j % S], (j / S) & 1);
      acc += smem[(j % S) * STAGE + (threadIdx.x & 63)];
    }
    if (it < kbn) {
      const int st = it % S;
      mbar_expect_tx(&full[st], STAGE);
      const int c = (kb0 + it) * 64;
      for (int t = 0; t < TMX; ++t)
        tma_load_2d_hint(smem + st * STAGE + t * BOXB, &map, &full[st], c, (strip * TMX + t) * BH, pol_first);
      for (int t = 0; t < VB; ++t)
        tma_load_2d_hint(smem + st * STAGE + (TMX + t) * BOXB, &vmap, &full[st], c, t * BH, pol_last);
    }
  }
  if (acc == 12345) sink[0] = acc;
}

template <int S, int TMX, int VB>
void run_fwd(const std::vector<void*>& mats, const void* vm, int R, int C, int split, unsigned long long* sink) {
  std::vector<CUtensorMap> maps(mats.size());
  for (size_t i = 0; i < mats.size(); ++i)
    if (!make_map(&maps[i], mats[i], 2, C, R, C, 64, BH)) { printf("map failed\n"); return; }
  CUtensorMap vmap;
  if (!make_map(&vmap, vm, 2, C, 256, C, 64, BH)) { printf("map failed\n"); return; }
  const size_t sm = 1024 + (size_t)S * (TMX + VB) * BOXB + 256;
  cudaFuncSetAttribute(fwd_kernel<S, TMX, VB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const int grid = R / (BH * TMX) * split;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 4; ++w) fwd_kernel<S, TMX, VB><<<grid, 128, sm>>>(maps[w % maps.size()], vmap, R, C, split, sink);
  cudaEventRecord(e0);
  const int reps = 12;
  for (int w = 0; w < reps; ++w) fwd_kernel<S, TMX, VB><<<grid, 128, sm>>>(maps[w % maps.size()], vmap, R, C, split, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = ms / reps * 1e3;
  const double bytes = (double)R * C * 2;
  printf("fwd S %d TMX %d VB %d split %d grid %3d : %7.2f us  X-rate %7.1f GB/s  (+V %.0f%%)\n", S, TMX, VB, split, grid, us,
         bytes / us * 1e-3, 100.0 * VB / TMX);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
}

int main() {
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  const int R = 8192, C = 8192;   // 128 MiB bf16, like one config-3 batch (2 views x 4096 x 8192)
  std::vector<void*> mats(4);
  for (auto& m : mats) { cudaMalloc(&m, (size_t)R * C * 2); cudaMemset(m, 1, (size_t)R * C * 2); }
  if (getenv("FWD_ONLY")) {
    void* vm;
    cudaMalloc(&vm, (size_t)256 * C * 2);
    cudaMemset(vm, 1, (size_t)256 * C * 2);
    // R = 8192 rows = one batch of both views stacked (4096 x 8192 each)
    run_fwd<6, 1, 0>(mats, vm, R, C, 2, sink);    // X only, 16 KB stages (F at TM 1 without V)
    run_fwd<6, 1, 1>(mats, vm, R, C, 2, sink);    // F at TM 1: 16 KB X + 16 KB V per stage
    run_fwd<12, 1, 0>(mats, vm, R, C, 2, sink);
    run_fwd<4, 2, 0>(mats, vm, R, C, 4, sink);    // X only, 32 KB stages
    run_fwd<4, 2, 1>(mats, vm, R, C, 4, sink);    // F at TM 2: 32 KB X + 16 KB V per stage
    run_fwd<6, 2, 0>(mats, vm, R, C, 4, sink);
    run_fwd<3, 4, 1>(mats, vm, R, C, 8, sink);    // TM 4: 64 KB X + 16 KB V
    return 0;
  }
  for (int grid : {128, 148}) {
    run<8>(mats, R, C, 1024, 0, 1, grid, sink);
    run<12>(mats, R, C, 1024, 0, 1, grid, sink);
    run<8>(mats, R, C, 1024, 2, 1, grid, sink);
    for (int CH : {256, 512, 1024, 2048})
      for (int lag : {1, 2}) {
        run<8>(mats, R, C, CH, 1, lag, grid, sink);
        run<12>(mats, R, C, CH, 1, lag, grid, sink);
      }
  }
  return 0;
}
