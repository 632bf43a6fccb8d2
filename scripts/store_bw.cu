// store_bw.cu — developer microbenchmark: how fast can 128-147 CTAs write
// their epilogue tiles (64 player rows x 128..256 columns fp32 per CTA,
// row-major k x ld array) — scalar coalesced STG.32 (the fused kernel's
// epilogue pattern), STG.128 after a warp transpose through smem, or a TMA
// bulk tensor store from smem.  Optionally while other CTAs stream reads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda
//   -o store_bw scripts/store_bw.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include "../paper_2206_04993_b200/csrc/tc_gemm.cuh"

using namespace geig::tc;

// each CTA: MT tiles of 128 columns x 64 rows; 128 threads = 4 warps, thread
// owns column m = warp*32 + lane of each tile (like the TMEM drain)
template <int MODE>
__global__ void __launch_bounds__(128) store_kernel(float* out, int64_t ld, int MT, const __grid_constant__ CUtensorMap map,
                                                    int reps) {
  extern __shared__ uint8_t raw[];
  float* tile = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = 0; r < reps; ++r) {
    for (int mt = 0; mt < MT; ++mt) {
      const int64_t m0 = ((int64_t)blockIdx.x * MT + mt) * 128;
      const int m = warp * 32 + lane;
      if (MODE == 0) {
        float* o = out + m0 + m;
#pragma unroll 16
        for (int n = 0; n < 64; ++n) o[(int64_t)n * ld] = (float)(n + m + r);
      } else {
        for (int n = 0; n < 64; ++n) tile[n * 128 + m] = (float)(n + m + r);
        __syncthreads();
        if (MODE == 1) {
          // float4 rows: thread t writes row n = t / 32 * ... (2 KB rows: 32 threads x 16 B)
          for (int e = threadIdx.x; e < 64 * 32; e += 128) {
            const int n = e >> 5, q = e & 31;
            *reinterpret_cast<float4*>(out + (int64_t)n * ld + m0 + 4 * q) = *reinterpret_cast<const float4*>(tile + n * 128 + 4 * q);
          }
        } else {
          if (threadIdx.x == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&map),
                         "r"((int)m0), "r"(0), "r"(smem_u32(tile))
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
        }
        __syncthreads();
      }
    }
  }
  if (MODE == 2 && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// per-CTA epilogue write of MT tiles (64 players x 128 columns fp32 each):
// mode 0: float4 STG from a staged smem tile; mode 1: TMA bulk tensor stores
// of all MT tiles, one wait at the end.  In-kernel %globaltimer per CTA.
template <int MODE>
__global__ void __launch_bounds__(128) epi_kernel(float* out, int64_t ld, int MT, const __grid_constant__ CUtensorMap map,
                                                  unsigned long long* tms) {
  extern __shared__ uint8_t raw[];
  float* tile = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int mt = 0; mt < MT; ++mt)
    for (int n = 0; n < 64; ++n) tile[mt * 64 * 128 + n * 128 + warp * 32 + lane] = (float)(n + lane + mt);
  __syncthreads();
  unsigned long long t0 = geig::tc::gtimer();
  if (MODE == 0) {
    for (int mt = 0; mt < MT; ++mt) {
      const int64_t m0 = ((int64_t)blockIdx.x * MT + mt) * 128;
      for (int e = threadIdx.x; e < 64 * 32; e += 128) {
        const int n = e >> 5, q = e & 31;
        __stcg(reinterpret_cast<float4*>(out + (int64_t)n * ld + m0 + 4 * q),
               *reinterpret_cast<const float4*>(tile + mt * 64 * 128 + n * 128 + 4 * q));
      }
    }
    __syncthreads();
  } else {
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (int mt = 0; mt < MT; ++mt) {
        const int m0 = (blockIdx.x * MT + mt) * 128;
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&map),
                     "r"(m0), "r"(0), "r"(smem_u32(tile + mt * 64 * 128))
                     : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    __syncthreads();
  }
  __threadfence();
  unsigned long long t1 = geig::tc::gtimer();
  if (threadIdx.x == 0) { tms[blockIdx.x * 2] = t0; tms[blockIdx.x * 2 + 1] = t1; }
}

template <int MODE>
void run_epi(float* out, int64_t ld, int grid, int MT, unsigned long long* tms) {
  CUtensorMap map;
  if (!make_map(&map, out, 4, ld, 64, ld, 128, 64, false)) { printf("map failed\n"); return; }
  const size_t sm = 1024 + (size_t)MT * 64 * 128 * 4;
  cudaFuncSetAttribute(epi_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  for (int w = 0; w < 5; ++w) epi_kernel<MODE><<<grid, 128, sm>>>(out, ld, MT, map, tms);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> h(2 * grid);
  cudaMemcpy(h.data(), tms, 16 * grid, cudaMemcpyDeviceToHost);
  unsigned long long mn = ~0ull, mx = 0;
  double sum = 0;
  for (int i = 0; i < grid; ++i) { mn = std::min(mn, h[2 * i]); mx = std::max(mx, h[2 * i + 1]); sum += h[2 * i + 1] - h[2 * i]; }
  printf("epi mode %d grid %d MT %d: span %.2f us, mean per-CTA %.2f us\n", MODE, grid, MT, (mx - mn) * 1e-3,
         sum / grid * 1e-3);
}

template <int MODE>
void run(float* out, int64_t ld, int grid, int MT, int reps) {
  CUtensorMap map;
  if (!make_map(&map, out, 4, ld, 64, ld, 128, 64, false)) { printf("map failed\n"); return; }
  const size_t sm = 1024 + 64 * 128 * 4;
  cudaFuncSetAttribute(store_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) store_kernel<MODE><<<grid, 128, sm>>>(out, ld, MT, map, reps);
  cudaEventRecord(e0);
  const int N = 20;
  for (int w = 0; w < N; ++w) store_kernel<MODE><<<grid, 128, sm>>>(out, ld, MT, map, reps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = ms / N * 1e3;
  const double bytes = (double)grid * MT * 128 * 64 * 4 * reps;
  printf("mode %d grid %3d MT %d reps %d: %8.2f us  %7.1f GB/s  (%.1f MB)\n", MODE, grid, MT, reps, us, bytes / us * 1e-3,
         bytes / 1e6);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
}

int main() {
  const int64_t ld = 2 * 16384 + 256;
  float* out;
  cudaMalloc(&out, (size_t)ld * 64 * 4);
  unsigned long long* tms;
  cudaMalloc(&tms, 16 * 256);
  for (int MT : {1, 2}) {
    run_epi<0>(out, ld, 128, MT, tms);
    run_epi<1>(out, ld, 128, MT, tms);
    run_epi<0>(out, ld, 147, MT, tms);
    run_epi<1>(out, ld, 147, MT, tms);
  }
  if (getenv("EPI_ONLY")) return 0;
  for (int grid : {128, 147})
    for (int MT : {1, 2})
      for (int reps : {1, 8}) {
        if (grid * MT * 128 > 16384 + 256) continue;
        run<0>(out, ld, grid, MT, reps);
        run<1>(out, ld, grid, MT, reps);
        run<2>(out, ld, grid, MT, reps);
      }
  return 0;
}
