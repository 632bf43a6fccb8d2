// common.cuh — small device helpers shared by the geig kernels.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <atomic>
#include <cstdlib>

#ifndef GEIG_DEV_KNOBS
#define GEIG_DEV_KNOBS 0
#endif

namespace geig {

constexpr int GEIG_MAX_PEERS = 8;   // ranks of the peer-memory exchange (one NVLink domain of the box)

// Developer A/B and timing knobs read from the environment exist only in a
// build with -DGEIG_DEV_KNOBS=1 (GEIG_NVCC_EXTRA); the default library reads
// no environment variable, so nothing outside the ABI changes its schedule
// or its numerics.
inline const char* dev_knob(const char* name) {
#if GEIG_DEV_KNOBS
  return std::getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// function attributes are per device context, so a solver created on a
// second device sets them again.  Thread-safe (setting twice is harmless).
inline cudaError_t set_smem_attr_once(std::atomic<uint64_t>& done, const void* fn, int bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T>
__device__ __forceinline__ T from_f32(float x);
template <>
__device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace geig
