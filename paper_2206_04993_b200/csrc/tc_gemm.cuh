// tc_gemm.cuh — tcgen05 / TMA tensor-core minibatch products for sm_100a.
//
// One warp-specialised kernel computes C[M x N] = sum_kk A(m,kk) B(n,kk) for
// up to two "segments" (K ranges with their own operands and their own TMEM
// accumulator), with
//   * A staged by TMA (SWIZZLE_128B) either K-major (row-major [M][K]: the
//     forward product X V^T, dense A V^T) or MN-major (row-major [K][M]: the
//     backward product X^T W, read straight from the sample-major X without a
//     transpose pass),
//   * B staged by TMA K-major ([N][K]: V (k x d) or W^T (k x rows)),
//   * tcgen05.mma (kind::f16 bf16 or kind::tf32) issued by ONE thread,
//     accumulators in TMEM (fp32), 4-stage mbarrier ring TMA <-> MMA,
//   * epilogue: tcgen05.ld 32x32b -> registers -> player-major output
//     out[n*ldo + m] = scale*acc (plain store or fp32 red.add for split-K).
// CTA = 128 threads: warp0 lane0 = TMA producer, warp1 lane0 = MMA issuer,
// warp2 = TMEM allocator; all four warps run the epilogue (warp w owns TMEM
// lanes 32w..32w+31 = output rows m0+32w..).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>
#include <type_traits>
#include <cstdlib>
#include "../../include/geig.h"
#include "common.cuh"

namespace geig { namespace tc {

constexpr int TC_THREADS = 128;
constexpr int TC_BM = 128;
constexpr int TC_MAX_STAGES = 8;
constexpr int TC_MAX_SPLITS = 8;

// ----------------------------------------------------------------------------
// PTX wrappers
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// one elected lane of a converged warp (elect.sync): unlike a threadIdx test,
// the compiler then treats the lane's operands of the uniform-datapath
// instructions (UTMALDG, UTCHMMA) as uniform instead of wrapping every issue
// in an elect / broadcast loop
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TC_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TC_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// TMA load with an L2 eviction-priority hint (policy from l2_policy_*)
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                 int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// Programmatic dependent launch: the prologue (barrier init, TMEM alloc,
// descriptor prefetch) of a kernel overlaps the tail of its predecessor;
// griddepcontrol.wait precedes the first read of predecessor outputs.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <int EB>
__device__ __forceinline__ void umma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  if constexpr (EB == 2) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
  }
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor, SWIZZLE_128B, sm_100 version bits = 1.
// tf32 with round-to-nearest (ties away), low 13 mantissa bits zero
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// layout: 2 = SWIZZLE_128B; 1 = SWIZZLE_128B_BASE32B (128-byte rows swizzled in
// 32-byte chunks, 4-row atoms): the MN-major layout of 32-bit (tf32) operands,
// written by TMA with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B.
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 2) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

// ----------------------------------------------------------------------------
// kernel
// ----------------------------------------------------------------------------
struct TcMaps {
  CUtensorMap a[4];   // index = group * 2 + segment
  CUtensorMap b[4];
  CUtensorMap blo[4]; // bf16x2: low halves of the B operands (bf16(x - bf16(x)))
};

struct TcParams {
  int M[2];            // valid rows per group (host-side arrays; the kernel
  int N;               //   selects with blockIdx.z-uniform ternaries, never
  int BN;              //   runtime-indexes the parameter block)
  int nseg;            // 1 or 2
  int kblocks[2][2];   // [group][segment] K blocks
  int splits;          // split-K factor (blockIdx.y)
  float* out[2][2];    // [group][segment] output base (player-major)
  int64_t ldo;
  float scale;
  int atomic;          // 1: red.add, 0: store
  int64_t split_stride;  // store mode with splits > 1: output offset per split (elements)
  uint32_t idesc;
  unsigned long long* dbg; // optional per-CTA %globaltimer stamps (4 per CTA), nullable
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// 3xTF32 (X3, EB = 4, with SPLIT): the A tile is split in shared memory by
// warps 2-3 into hi = tf32_rna(a) (in place) and lo = a - hi (next to it);
// the B operand arrives as hi / lo planes; each K step issues
// A_hi B_hi + A_hi B_lo + A_lo B_hi (the a_lo b_lo term is below fp32 ulp).
template <int EB, bool A_MN, int TC_STAGES, bool SPLIT, bool X3 = false>
__global__ void __launch_bounds__(TC_THREADS)
tc_gemm_kernel(const __grid_constant__ TcMaps maps, const TcParams p) {
  static_assert(!X3 || (EB == 4 && SPLIT), "3xTF32 needs tf32 operands with B hi/lo planes");
  constexpr int ATOM = 128 / EB;           // elements per 128B row
  constexpr int BK = ATOM;                 // K per stage
  constexpr int UK = 32 / EB;              // K per MMA (16 bf16 / 8 tf32)
  constexpr uint32_t A_BYTES = TC_BM * 128;
  const int g = blockIdx.z;
  const int m0 = blockIdx.x * TC_BM;
  const int Mg = g == 0 ? p.M[0] : p.M[1];
  pdl_trigger();
  if (m0 >= Mg) return;
  const int BN = p.BN;
  const uint32_t B_BYTES = (uint32_t)BN * 128;
  constexpr uint32_t A_TOT = A_BYTES * (X3 ? 2 : 1);   // X3: A hi, A lo
  const uint32_t STAGE_BYTES = A_TOT + B_BYTES * (SPLIT ? 2 : 1);

  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned view of the dynamic smem that stays in the shared
  // address space (integer pointer round-trips would turn every later smem
  // access into a generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + TC_STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + TC_STAGES;
  uint64_t* accum_bar = empty_bar + TC_STAGES;
  uint64_t* conv_bar = accum_bar + 1;                    // X3: A split done (2 arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(conv_bar + TC_STAGES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t cta_id = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  if (p.dbg && threadIdx.x == 0) p.dbg[cta_id * 4 + 0] = gtimer();
  // per-segment K-block ranges of this split
  int kb_beg[2], kb_cnt[2];
  int total = 0;
  for (int s = 0; s < 2; ++s) {
    const int kb = s >= p.nseg ? 0 : (g == 0 ? (s == 0 ? p.kblocks[0][0] : p.kblocks[0][1])
                                             : (s == 0 ? p.kblocks[1][0] : p.kblocks[1][1]));
    const int b0 = (int)((int64_t)kb * blockIdx.y / p.splits);
    const int b1 = (int)((int64_t)kb * (blockIdx.y + 1) / p.splits);
    kb_beg[s] = b0;
    kb_cnt[s] = b1 - b0;
    total += kb_cnt[s];
  }
  uint32_t ncols = 32;
  while (ncols < (uint32_t)(p.nseg * BN)) ncols <<= 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
      if (X3) mbar_init(&conv_bar[s], 2);
    }
    mbar_init(accum_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < p.nseg; ++s) {
      tma_prefetch_desc(&maps.a[g * 2 + s]);
      tma_prefetch_desc(&maps.b[g * 2 + s]);
    }
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();

  if (total > 0) {
    if (threadIdx.x == 0) {
      // ---------------- TMA producer ----------------
      int it = 0;
      for (int s = 0; s < p.nseg; ++s) {
        const CUtensorMap* ma = &maps.a[g * 2 + s];
        const CUtensorMap* mb = &maps.b[g * 2 + s];
        for (int j = 0; j < kb_cnt[s]; ++j, ++it) {
          const int st = it % TC_STAGES;
          if (it >= TC_STAGES) mbar_wait(&empty_bar[st], ((it / TC_STAGES) + 1) & 1);
          uint8_t* sa = smem + st * STAGE_BYTES;
          uint8_t* sb = sa + A_TOT;
          mbar_expect_tx(&full_bar[st], STAGE_BYTES - (A_TOT - A_BYTES));   // X3: A lo is written by warps 2-3
          const int k0 = (kb_beg[s] + j) * BK;
          if constexpr (A_MN) {
#pragma unroll
            for (int q = 0; q < TC_BM / ATOM; ++q) tma_load_2d(sa + q * (BK * 128), ma, &full_bar[st], m0 + q * ATOM, k0);
          } else {
            tma_load_2d(sa, ma, &full_bar[st], k0, m0);
          }
          tma_load_2d(sb, mb, &full_bar[st], k0, 0);
          if constexpr (SPLIT) tma_load_2d(sb + B_BYTES, &maps.blo[g * 2 + s], &full_bar[st], k0, 0);
        }
      }
    } else if ((threadIdx.x >> 5) == 1 && elect_one()) {
      // ---------------- MMA issuer (lane 0 of the converged warp 1) ----------------
      int it = 0;
      for (int s = 0; s < p.nseg; ++s) {
        const uint32_t d_tmem = tmem_base + (uint32_t)(s * BN);
        for (int j = 0; j < kb_cnt[s]; ++j, ++it) {
          const int st = it % TC_STAGES;
          mbar_wait(X3 ? &conv_bar[st] : &full_bar[st], (it / TC_STAGES) & 1);
          if (p.dbg && it == 0) p.dbg[cta_id * 4 + 1] = gtimer();
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + st * STAGE_BYTES);
          const uint32_t sb = sa + A_TOT;
#pragma unroll
          for (int kk = 0; kk < BK / UK; ++kk) {
            uint64_t ad, bd;
            if constexpr (A_MN) {
              // MN-major A: 16-bit types in 128B-swizzle atoms of 8 rows (SBO 1024 B);
              // tf32 in 128B / 32B-chunk atoms of 4 rows (SBO 512 B)
              ad = EB == 2 ? make_sdesc(sa + kk * UK * 128, BK * 128, 1024)
                           : make_sdesc(sa + kk * UK * 128, BK * 128, 512, 1);
            } else {
              ad = make_sdesc(sa + kk * 32, 16, 1024);
            }
            bd = make_sdesc(sb + kk * 32, 16, 1024);
            umma<EB>(d_tmem, ad, bd, p.idesc, (j > 0 || kk > 0) ? 1u : 0u);
            if constexpr (SPLIT) umma<EB>(d_tmem, ad, make_sdesc(sb + B_BYTES + kk * 32, 16, 1024), p.idesc, 1u);
            if constexpr (X3) umma<EB>(d_tmem, ad + (uint64_t)(A_BYTES >> 4), bd, p.idesc, 1u);   // A lo x B hi
          }
          umma_commit(&empty_bar[st]);
        }
      }
      umma_commit(accum_bar);
    } else if (X3 && warp >= 2) {
      // ---------------- A-tile split (warps 2-3) ----------------
      const int ct = threadIdx.x - 64;
      int it = 0;
      for (int s = 0; s < p.nseg; ++s) {
        for (int j = 0; j < kb_cnt[s]; ++j, ++it) {
          const int st = it % TC_STAGES;
          mbar_wait(&full_bar[st], (it / TC_STAGES) & 1);
          float4* a = reinterpret_cast<float4*>(smem + st * STAGE_BYTES);
          float4* al = a + A_BYTES / 16;
#pragma unroll 4
          for (int e = ct; e < (int)(A_BYTES / 16); e += 64) {
            float4 x = a[e], hi, lo;
            hi.x = tf32_rna(x.x); hi.y = tf32_rna(x.y); hi.z = tf32_rna(x.z); hi.w = tf32_rna(x.w);
            lo.x = x.x - hi.x; lo.y = x.y - hi.y; lo.z = x.z - hi.z; lo.w = x.w - hi.w;
            a[e] = hi;
            al[e] = lo;
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tcgen05.mma reads
          __syncwarp();
          if (lane == 0) mbar_arrive(&conv_bar[st]);
        }
      }
    }
    // ---------------- epilogue (all 4 warps) ----------------
    // TMEM -> registers -> smem tile[n][m] (the idle pipeline buffers) ->
    // coalesced 16-byte stores (or red.global.add.v4.f32 for split-K) of
    // whole 512-byte output rows out[n][m0 .. m0+127].
    mbar_wait(accum_bar, 0);
    if (p.dbg && threadIdx.x == 0) p.dbg[cta_id * 4 + 2] = gtimer();
    __syncwarp();
    tc_fence_after();
    float* tile = reinterpret_cast<float*>(smem);          // [BN][TC_BM]
    const float scale = p.scale;
    const int N = p.N;
    const int64_t ldo = p.ldo;
    const bool atomic = p.atomic != 0;
    const int64_t soff = atomic ? 0 : (int64_t)blockIdx.y * p.split_stride;
    for (int s = 0; s < p.nseg; ++s) {
      if (kb_cnt[s] == 0) continue;
      float* out = (g == 0 ? (s == 0 ? p.out[0][0] : p.out[0][1]) : (s == 0 ? p.out[1][0] : p.out[1][1])) + soff;
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(tmem_base + ((uint32_t)(warp * 32) << 16) + (uint32_t)(s * BN + c0), r);
#pragma unroll
        for (int j = 0; j < 16; ++j) tile[(c0 + j) * TC_BM + warp * 32 + lane] = __uint_as_float(r[j]);
      }
      __syncthreads();
      const int mm = m0 + 4 * lane;
      const bool vec = ((ldo & 3) == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
      for (int n = warp; n < N; n += 4) {
        float4 v = *reinterpret_cast<const float4*>(tile + n * TC_BM + 4 * lane);
        v.x *= scale; v.y *= scale; v.z *= scale; v.w *= scale;
        float* dst = out + (int64_t)n * ldo + mm;
        if (vec && mm + 3 < Mg) {
          if (atomic)
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(v.x), "f"(v.y), "f"(v.z),
                         "f"(v.w)
                         : "memory");
          else
            *reinterpret_cast<float4*>(dst) = v;
        } else {
          const float vs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (mm + q < Mg) {
              if (atomic) atomicAdd(dst + q, vs[q]); else dst[q] = vs[q];
            }
        }
      }
      __syncthreads();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (p.dbg && threadIdx.x == 0) p.dbg[cta_id * 4 + 3] = gtimer();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(ncols));
  }
}

// Forward-product reshuffle: the split-K partials Zp[split][view] (k x ldz
// fp32, rows 0..2h) summed in fixed split order (deterministic) into the four
// backward B operands Zb[view][half] (k x hpad, T) — reading R1:
//   X backward: half0 (A_t) uses Z_y rows [0,h), half1 (B_t) uses Z_x rows [h,2h)
//   Y backward: half0 uses Z_x rows [0,h), half1 uses Z_y rows [h,2h)
template <typename T>
__device__ __forceinline__ void store4(T* dst, float a, float b, float c, float d);
template <>
__device__ __forceinline__ void store4<float>(float* dst, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(dst) = make_float4(a, b, c, d);
}
template <>
__device__ __forceinline__ void store4<__nv_bfloat16>(__nv_bfloat16* dst, float a, float b, float c, float d) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
  uint2 pk;
  pk.x = *reinterpret_cast<uint32_t*>(&lo);
  pk.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(dst) = pk;
}

template <typename T>
__device__ __forceinline__ void store4_lo(T* dst, float a, float b, float c, float d);
template <>
__device__ __forceinline__ void store4_lo<float>(float* dst, float a, float b, float c, float d) {   // 3xTF32
  store4<float>(dst, a - tf32_rna(a), b - tf32_rna(b), c - tf32_rna(c), d - tf32_rna(d));
}
template <>
__device__ __forceinline__ void store4_lo<__nv_bfloat16>(__nv_bfloat16* dst, float a, float b, float c, float d) {
  const float ha = __bfloat162float(__float2bfloat16_rn(a)), hb = __bfloat162float(__float2bfloat16_rn(b));
  const float hc = __bfloat162float(__float2bfloat16_rn(c)), hd = __bfloat162float(__float2bfloat16_rn(d));
  store4<__nv_bfloat16>(dst, a - ha, b - hb, c - hc, d - hd);
}

template <typename T>
__global__ void zshuffle_kernel(const float* __restrict__ Zp, T* __restrict__ Zb, int k, int64_t ldz, int h,
                                int64_t hpad, int splits, int lo) {
  pdl_trigger();
  pdl_wait();
  const int64_t vstride = (int64_t)k * ldz;
  const int64_t plane = (int64_t)k * hpad;
  const bool vec = ((h & 3) == 0) && ((ldz & 3) == 0) && ((hpad & 3) == 0);
  if (vec) {
    const int hq = h / 4;
    const int64_t per = (int64_t)k * hq;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < per; e += (int64_t)gridDim.x * blockDim.x) {
      const int n = (int)(e / hq), r = 4 * (int)(e % hq);
      float4 x0 = make_float4(0.f, 0.f, 0.f, 0.f), x1 = x0, y0 = x0, y1 = x0;
      for (int sp = 0; sp < splits; ++sp) {
        const float* zx = Zp + (int64_t)(2 * sp) * vstride + (int64_t)n * ldz;
        const float* zy = zx + vstride;
        const float4 a = *reinterpret_cast<const float4*>(zx + r), b = *reinterpret_cast<const float4*>(zx + h + r);
        const float4 c = *reinterpret_cast<const float4*>(zy + r), d = *reinterpret_cast<const float4*>(zy + h + r);
        x0.x += a.x; x0.y += a.y; x0.z += a.z; x0.w += a.w;
        x1.x += b.x; x1.y += b.y; x1.z += b.z; x1.w += b.w;
        y0.x += c.x; y0.y += c.y; y0.z += c.z; y0.w += c.w;
        y1.x += d.x; y1.y += d.y; y1.z += d.z; y1.w += d.w;
      }
      const int64_t o = (int64_t)n * hpad + r;
      const bool x3 = std::is_same<T, float>::value && lo;     // 3xTF32: hi planes hold tf32_rna(z)
      auto hv = [&](float v) { return x3 ? tf32_rna(v) : v; };
      store4<T>(Zb + 0 * plane + o, hv(y0.x), hv(y0.y), hv(y0.z), hv(y0.w));   // view x, half 0
      store4<T>(Zb + 1 * plane + o, hv(x1.x), hv(x1.y), hv(x1.z), hv(x1.w));   // view x, half 1
      store4<T>(Zb + 2 * plane + o, hv(x0.x), hv(x0.y), hv(x0.z), hv(x0.w));   // view y, half 0
      store4<T>(Zb + 3 * plane + o, hv(y1.x), hv(y1.y), hv(y1.z), hv(y1.w));   // view y, half 1
      if (lo) {                                                 // bf16x2 low halves
        store4_lo<T>(Zb + 4 * plane + o, y0.x, y0.y, y0.z, y0.w);
        store4_lo<T>(Zb + 5 * plane + o, x1.x, x1.y, x1.z, x1.w);
        store4_lo<T>(Zb + 6 * plane + o, x0.x, x0.y, x0.z, x0.w);
        store4_lo<T>(Zb + 7 * plane + o, y1.x, y1.y, y1.z, y1.w);
      }
    }
    return;
  }
  const int64_t per = (int64_t)k * h;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < per; e += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(e / h), r = (int)(e % h);
    float x0 = 0.f, x1 = 0.f, y0 = 0.f, y1 = 0.f;
    for (int sp = 0; sp < splits; ++sp) {
      const float* zx = Zp + (int64_t)(2 * sp) * vstride + (int64_t)n * ldz;
      const float* zy = zx + vstride;
      x0 += zx[r]; x1 += zx[h + r]; y0 += zy[r]; y1 += zy[h + r];
    }
    const int64_t o = (int64_t)n * hpad + r;
    const float v4[4] = {y0, x1, x0, y1};
    const bool x3 = std::is_same<T, float>::value && lo;     // 3xTF32: hi = tf32_rna(z), lo = z - hi
    for (int q = 0; q < 4; ++q) {
      const float hi = x3 ? tf32_rna(v4[q]) : (float)(T)v4[q];
      Zb[q * plane + o] = x3 ? (T)hi : (T)v4[q];
      if (lo) Zb[(4 + q) * plane + o] = (T)(v4[q] - hi);
    }
  }
}

// ----------------------------------------------------------------------------
// host side
// ----------------------------------------------------------------------------
struct TcPlan {
  int ready = 0;
  int splitb = 0;          // bf16x2: B operands as hi + lo bf16 (V and Z), 2 MMAs per K step
  int problem = 0, math = 0, k = 0, BN = 0, device = 0, nsm = 148;
  int64_t dx = 0, dy = 0, d = 0, max_rows = 0, ldz = 0, hpad = 0;
  float* Zt = nullptr;     // TC_MAX_SPLITS x 2 x k x ldz fp32 (CCA forward split-K partials)
  void* Zb = nullptr;      // 2 x 2 x k x hpad (bf16 or fp32)
  CUtensorMap* xm_dev = nullptr;    // multi-step fused launch: per-step A-operand maps (device)
  CUtensorMap* xm_host = nullptr;   // pinned staging of the same
  int xm_cap = 0;                   // steps of capacity
  cudaEvent_t xm_ev = nullptr;      // last copy of the staging buffer
  int* dep = nullptr;               // fused step: Gram-reduction counter (monotonic, zeroed once)
  int x3 = 0;                       // 3xTF32 products (tf32 plan with hi/lo operands)
  int opt_m_tiles = 0;              // geig_set_option(GEIG_OPT_FUSED_M_TILES): 0 = auto, 1 or 2
  int opt_pairs = 1;                // geig_set_option(GEIG_OPT_FUSED_PAIRS): CTA pairs in the fused step
  cudaAccessPolicyWindow l2win{};   // persisting-L2 window over the solver's state arena (num_bytes 0: none)
  float* Vx3 = nullptr;             // 3xTF32: [hi plane | lo plane] of V (2 x k x d fp32)
};

inline unsigned long long*& dbg_ptr() {
  static unsigned long long* p = nullptr;
  return p;
}

inline std::string& err_str() {
  static thread_local std::string e;
  return e;
}
inline const char* last_error() { return err_str().c_str(); }
inline geig_status tc_fail(geig_status st, const std::string& m) {
  err_str() = m;
  return st;
}

inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D row-major tensor [outer][inner] with row stride `stride_el` elements.
inline bool make_map(CUtensorMap* m, const void* base, int eb, int64_t inner, int64_t outer, int64_t stride_el,
                     int box_inner, int box_outer, bool swizzle = true, bool atom32 = false) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(stride_el * eb)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, eb == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                  const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle ? (atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B)
                          : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 3D bf16 map with the 128-byte swizzle: dims {inner, rows, blocks}, row
// stride stride_el, block stride block_el (elements); box {box_inner,
// box_rows, 1} lands like the 2D box of make_map (the column-owned forward's
// V operand: the gathered shadow [rank][hi|lo][k][W]).
inline bool make_map3(CUtensorMap* m, const void* base, int64_t inner, int64_t rows, int64_t blocks, int64_t stride_el,
                      int64_t block_el, int box_inner, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)blocks};
  cuuint64_t strides[2] = {(cuuint64_t)(stride_el * 2), (cuuint64_t)(block_el * 2)};
  cuuint32_t box[3] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

inline uint32_t make_idesc(int eb, bool a_mn, int N, int M) {
  const uint32_t fmt = eb == 2 ? 1u : 2u;  // BF16 : TF32
  return (1u << 4) | (fmt << 7) | (fmt << 10) | ((a_mn ? 1u : 0u) << 15) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

inline size_t smem_bytes(int BN, int stages, bool split = false, bool x3 = false) {
  return 1024 + (size_t)stages * (TC_BM * 128 * (x3 ? 2 : 1) + (size_t)BN * 128 * (split ? 2 : 1)) + 256;
}

// Stage count: enough bytes in flight per SM to cover DRAM latency. One
// resident CTA per SM (grid <= #SM) gets the deep ring, denser grids 4 stages.
template <int EB, bool A_MN, int ST, bool SPLIT, bool X3 = false>
inline cudaError_t launch_one(const TcMaps& maps, const TcParams& p, dim3 grid, cudaStream_t st) {
  static std::atomic<uint64_t> attr_done{0};
  {
    const size_t mx = std::min<size_t>(227 * 1024, smem_bytes(128, ST, SPLIT, X3));
    cudaError_t e = set_smem_attr_once(attr_done, (const void*)tc_gemm_kernel<EB, A_MN, ST, SPLIT, X3>, (int)mx);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = smem_bytes(p.BN, ST, SPLIT, X3);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, tc_gemm_kernel<EB, A_MN, ST, SPLIT, X3>, maps, p);
  return e == cudaSuccess ? cudaGetLastError() : e;
}

template <int EB, bool A_MN>
inline geig_status launch(const TcMaps& maps, const TcParams& p, dim3 grid, cudaStream_t st, int nsm,
                          bool split = false, bool x3 = false) {
  const int ctas = grid.x * grid.y * grid.z;
  const_cast<TcParams&>(p).dbg = dbg_ptr();
  if (dbg_ptr()) dbg_ptr() += (size_t)4 * ctas;   // next launch stamps after this one
  const bool one_per_sm = ctas <= nsm;
  cudaError_t e;
  if constexpr (EB == 4) {
    if (x3) {
      // 3xTF32 stage = A hi + A lo + B hi + B lo
      if (one_per_sm && smem_bytes(p.BN, 4, true, true) <= 227 * 1024) e = launch_one<EB, A_MN, 4, true, true>(maps, p, grid, st);
      else e = launch_one<EB, A_MN, 2, true, true>(maps, p, grid, st);
      if (e != cudaSuccess) return tc_fail(GEIG_ERR_CUDA, std::string("tc_gemm launch: ") + cudaGetErrorString(e));
      return GEIG_OK;
    }
  }
  if (split) {
    // bf16x2 stage = A + 2 B: 6 stages fit one CTA per SM
    if (one_per_sm && smem_bytes(p.BN, 6, true) <= 227 * 1024) e = launch_one<EB, A_MN, 6, true>(maps, p, grid, st);
    else e = launch_one<EB, A_MN, 3, true>(maps, p, grid, st);
  } else {
    if (one_per_sm && smem_bytes(p.BN, 8) <= 227 * 1024) e = launch_one<EB, A_MN, 8, false>(maps, p, grid, st);
    else if (ctas <= 2 * nsm && smem_bytes(p.BN, 3) <= 113 * 1024)
      // up to two CTAs per SM: every CTA of the grid resident at once, so the
      // HBM stream is shared by all tiles to the end instead of a ragged
      // second wave (config 4: 256 tiles on 148 SMs); 3 stages per CTA keep
      // 192 KB in flight per SM
      e = launch_one<EB, A_MN, 3, false>(maps, p, grid, st);
    else e = launch_one<EB, A_MN, 4, false>(maps, p, grid, st);
  }
  if (e != cudaSuccess) return tc_fail(GEIG_ERR_CUDA, std::string("tc_gemm launch: ") + cudaGetErrorString(e));
  return GEIG_OK;
}

// largest power-of-two split keeping the grid within one CTA per SM
inline int choose_splits_deep(int ctas, int kblocks, int nsm) {
  int s = 1;
  while (ctas * (s * 2) <= nsm && s * 2 <= kblocks) s *= 2;
  return s;
}

inline int choose_splits(int ctas, int kblocks, int nsm) {
  int s = 1;
  while (ctas * (s * 2) <= 2 * nsm && s * 2 <= kblocks) s *= 2;
  return s;
}

inline geig_status plan_create(TcPlan& t, int problem, int64_t dx, int64_t dy, int k, int math, int64_t max_rows,
                               int device) {
  t.x3 = math == GEIG_MATH_3XTF32 ? 1 : 0;
  t.splitb = (math == GEIG_MATH_BF16X2 || t.x3) ? 1 : 0;
  if (math == GEIG_MATH_BF16X2) math = GEIG_MATH_BF16;
  if (t.x3) math = GEIG_MATH_TF32;
  const int eb = math == GEIG_MATH_BF16 ? 2 : 4;
  const int align = 16 / eb;
  if (dx % align || dy % align)
    return tc_fail(GEIG_ERR_UNSUPPORTED, "tensor-core path needs dx, dy multiples of " + std::to_string(align) +
                                             " (TMA 16-byte strides); use GEIG_MATH_F32");
  if (!encode_fn()) return tc_fail(GEIG_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  t.problem = problem; t.math = math; t.k = k; t.dx = dx; t.dy = dy; t.d = dx + dy; t.device = device;
  t.max_rows = max_rows;
  t.BN = ((k + 15) / 16) * 16;
  cudaDeviceGetAttribute(&t.nsm, cudaDevAttrMultiProcessorCount, device);
  if (problem == GEIG_CCA) {
    t.ldz = ((max_rows + 3) / 4) * 4;
    t.hpad = ((max_rows / 2 + 7) / 8) * 8;
    if (cudaMalloc((void**)&t.Zt, (size_t)TC_MAX_SPLITS * 2 * k * t.ldz * 4) != cudaSuccess ||
        cudaMalloc(&t.Zb, (size_t)8 * k * t.hpad * eb) != cudaSuccess)
      return tc_fail(GEIG_ERR_CUDA, "cudaMalloc tc scratch");
    cudaMemset(t.Zb, 0, (size_t)8 * k * t.hpad * eb);
  }
  if (t.x3 && cudaMalloc((void**)&t.Vx3, (size_t)2 * k * t.d * 4) != cudaSuccess)
    return tc_fail(GEIG_ERR_CUDA, "cudaMalloc 3xTF32 operand planes");
  t.ready = 1;
  return GEIG_OK;
}

inline void plan_destroy(TcPlan& t) {
  if (t.Zt) cudaFree(t.Zt);
  if (t.Zb) cudaFree(t.Zb);
  if (t.Vx3) cudaFree(t.Vx3);
  t.Vx3 = nullptr;
  if (t.xm_dev) cudaFree(t.xm_dev);
  if (t.xm_host) cudaFreeHost(t.xm_host);
  if (t.xm_ev) cudaEventDestroy(t.xm_ev);
  if (t.dep) cudaFree(t.dep);
  t.dep = nullptr;
  t.xm_dev = nullptr; t.xm_host = nullptr; t.xm_cap = 0; t.xm_ev = nullptr;
  t.Zt = nullptr; t.Zb = nullptr; t.ready = 0;
}

// 3xTF32 B operand: hi = tf32_rna(v), lo = v - hi (planes n apart).
__global__ void tf32_split_kernel(const float* __restrict__ v, float* __restrict__ hl, int64_t n) {
  pdl_trigger();
  pdl_wait();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const float x = v[e], hi = tf32_rna(x);
    hl[e] = hi;
    hl[n + e] = x - hi;
  }
}
inline geig_status split_v_x3(TcPlan& t, const float* V, cudaStream_t st, int64_t* nl) {
  const int64_t n = (int64_t)t.k * t.d;
  tf32_split_kernel<<<(unsigned)std::min<int64_t>(4 * t.nsm, (n + 255) / 256), 256, 0, st>>>(V, t.Vx3, n);
  if (cudaGetLastError() != cudaSuccess) return tc_fail(GEIG_ERR_CUDA, "tf32 split launch failed");
  ++*nl;
  return GEIG_OK;
}

// CCA products: forward (K-major X, V) -> Zt -> shuffle -> backward (MN-major X, Zb).
inline geig_status products_cca(TcPlan& t, const void* X, const void* Y, int64_t b, float scale,
                                const __nv_bfloat16* Vbf, const float* V, float* AV, float* BV, cudaStream_t st,
                                int64_t* nl) {
  *nl = 0;
  if (!t.ready) return tc_fail(GEIG_ERR_STATE, "tc plan not ready");
  const int eb = t.math == GEIG_MATH_BF16 ? 2 : 4;
  const int ATOM = 128 / eb;
  const int h = (int)(b / 2);
  const int rows = 2 * h;
  const int k = t.k;
  if (t.x3) {
    geig_status e = split_v_x3(t, V, st, nl);
    if (e) return e;
  }
  const void* Vop = eb == 2 ? (const void*)Vbf : (t.x3 ? (const void*)t.Vx3 : (const void*)V);
  const int64_t dv[2] = {t.dx, t.dy};
  const void* Xv[2] = {X, Y};
  // ---- forward: Z_v = X_v V_v^T, M = rows, K = d_v; split-K partials stored
  //      (no atomics) and summed by the reshuffle ----
  int fsplits = 1;
  {
    TcMaps maps;
    TcParams p{};
    for (int v = 0; v < 2; ++v) {
      const char* vb = (const char*)Vop + (v == 0 ? 0 : t.dx * eb);
      if (!make_map(&maps.a[v * 2], Xv[v], eb, dv[v], rows, dv[v], ATOM, TC_BM) ||
          !make_map(&maps.b[v * 2], vb, eb, dv[v], k, t.d, ATOM, t.BN))
        return tc_fail(GEIG_ERR_CUDA, "tensor map encode (forward) failed");
      if (t.splitb && !make_map(&maps.blo[v * 2], vb + (int64_t)k * t.d * eb, eb, dv[v], k, t.d, ATOM, t.BN))
        return tc_fail(GEIG_ERR_CUDA, "tensor map encode (forward lo) failed");
      maps.a[v * 2 + 1] = maps.a[v * 2];
      maps.b[v * 2 + 1] = maps.b[v * 2];
      maps.blo[v * 2 + 1] = maps.blo[v * 2];
      p.M[v] = rows;
      p.kblocks[v][0] = (int)((dv[v] + ATOM - 1) / ATOM);
      p.kblocks[v][1] = 0;
      p.out[v][0] = t.Zt + (int64_t)v * k * t.ldz;
      p.out[v][1] = nullptr;
    }
    p.N = k; p.BN = t.BN; p.nseg = 1; p.ldo = t.ldz; p.scale = 1.f; p.atomic = 0;
    p.split_stride = (int64_t)2 * k * t.ldz;
    p.idesc = make_idesc(eb, false, t.BN, TC_BM);
    const int mt = (rows + TC_BM - 1) / TC_BM;
    p.splits = std::min(TC_MAX_SPLITS, choose_splits_deep(2 * mt, std::min(p.kblocks[0][0], p.kblocks[1][0]), t.nsm));
    if (const char* e = dev_knob("GEIG_FWD_SPLITS")) p.splits = std::max(1, std::min(TC_MAX_SPLITS, atoi(e)));
    fsplits = p.splits;
    dim3 grid(mt, p.splits, 2);
    geig_status s = eb == 2 ? launch<2, false>(maps, p, grid, st, t.nsm, t.splitb)
                            : launch<4, false>(maps, p, grid, st, t.nsm, t.splitb, t.x3);
    if (s) return s;
    ++*nl;
  }
  // ---- reshuffle: sum split partials -> Zb halves ----
  {
    const int64_t per = (int64_t)k * h / 4 + 1;
    const int blocks = (int)std::min<int64_t>(4 * t.nsm, (per + 255) / 256);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t le;
    if (eb == 2)
      le = cudaLaunchKernelEx(&cfg, zshuffle_kernel<__nv_bfloat16>, (const float*)t.Zt, (__nv_bfloat16*)t.Zb, k, t.ldz,
                              h, t.hpad, fsplits, t.splitb);
    else
      le = cudaLaunchKernelEx(&cfg, zshuffle_kernel<float>, (const float*)t.Zt, (float*)t.Zb, k, t.ldz, h, t.hpad,
                              fsplits, t.x3);
    if (le != cudaSuccess) return tc_fail(GEIG_ERR_CUDA, "zshuffle launch failed");
    if (cudaGetLastError() != cudaSuccess) return tc_fail(GEIG_ERR_CUDA, "zshuffle launch failed");
    ++*nl;
  }
  // ---- backward: AV_v = X_v[0:h]^T Zb[v][0], BV_v = X_v[h:2h]^T Zb[v][1] ----
  {
    TcMaps maps;
    TcParams p{};
    const int64_t plane = (int64_t)k * t.hpad;
    for (int v = 0; v < 2; ++v) {
      for (int s = 0; s < 2; ++s) {
        const char* xb = (const char*)Xv[v] + (int64_t)s * h * dv[v] * eb;
        const char* zb = (const char*)t.Zb + (int64_t)(v * 2 + s) * plane * eb;
        if (!make_map(&maps.a[v * 2 + s], xb, eb, dv[v], h, dv[v], ATOM, ATOM, true, eb == 4) ||
            !make_map(&maps.b[v * 2 + s], zb, eb, h, k, t.hpad, ATOM, t.BN))
          return tc_fail(GEIG_ERR_CUDA, "tensor map encode (backward) failed");
        if (t.splitb && !make_map(&maps.blo[v * 2 + s], zb + 4 * plane * eb, eb, h, k, t.hpad, ATOM, t.BN))
          return tc_fail(GEIG_ERR_CUDA, "tensor map encode (backward lo) failed");
        p.kblocks[v][s] = (h + ATOM - 1) / ATOM;
      }
      p.M[v] = (int)dv[v];
      const int64_t off = v == 0 ? 0 : t.dx;
      p.out[v][0] = AV + off;
      p.out[v][1] = BV + off;
    }
    p.N = k; p.BN = t.BN; p.nseg = 2; p.ldo = t.d; p.scale = scale;
    p.idesc = make_idesc(eb, true, t.BN, TC_BM);
    const int mt = (int)((std::max(t.dx, t.dy) + TC_BM - 1) / TC_BM);
    const int mtot = (int)((t.dx + TC_BM - 1) / TC_BM + (t.dy + TC_BM - 1) / TC_BM);
    p.splits = (mtot * 3 >= t.nsm * 2) ? 1 : choose_splits(mtot, p.kblocks[0][0], t.nsm);
    p.atomic = p.splits > 1;
    p.split_stride = 0;
    if (p.atomic) {
      if (cudaMemsetAsync(AV, 0, (size_t)k * t.d * 4, st) != cudaSuccess ||
          cudaMemsetAsync(BV, 0, (size_t)k * t.d * 4, st) != cudaSuccess)
        return tc_fail(GEIG_ERR_CUDA, "memset AV/BV failed");
    }
    dim3 grid(mt, p.splits, 2);
    geig_status s = eb == 2 ? launch<2, true>(maps, p, grid, st, t.nsm, t.splitb)
                            : launch<4, true>(maps, p, grid, st, t.nsm, t.splitb, t.x3);
    if (s) return s;
    ++*nl;
  }
  return GEIG_OK;
}

// Dense products: AV[:, r0:r1] = A[r0:r1] V^T, BV likewise (K-major A rows, tf32 or bf16).
inline geig_status products_dense(TcPlan& t, const void* A, const void* B, int64_t r0, int64_t r1,
                                  const __nv_bfloat16* Vbf, const float* V, float* AV, float* BV, cudaStream_t st,
                                  int64_t* nl) {
  *nl = 0;
  if (!t.ready) return tc_fail(GEIG_ERR_STATE, "tc plan not ready");
  const int eb = t.math == GEIG_MATH_BF16 ? 2 : 4;
  const int ATOM = 128 / eb;
  const int k = t.k;
  const int M = (int)(r1 - r0);
  if (t.x3) {
    geig_status e = split_v_x3(t, V, st, nl);
    if (e) return e;
  }
  const void* Vop = eb == 2 ? (const void*)Vbf : (t.x3 ? (const void*)t.Vx3 : (const void*)V);
  TcMaps maps;
  TcParams p{};
  const void* mats[2] = {A, B};
  float* outs[2] = {AV + r0, BV + r0};
  for (int g = 0; g < 2; ++g) {
    if (!make_map(&maps.a[g * 2], mats[g], eb, t.d, M, t.d, ATOM, TC_BM) ||
        !make_map(&maps.b[g * 2], Vop, eb, t.d, k, t.d, ATOM, t.BN))
      return tc_fail(GEIG_ERR_CUDA, "tensor map encode (dense) failed");
    if (t.x3 && !make_map(&maps.blo[g * 2], (const char*)Vop + (int64_t)k * t.d * eb, eb, t.d, k, t.d, ATOM, t.BN))
      return tc_fail(GEIG_ERR_CUDA, "tensor map encode (dense lo) failed");
    maps.a[g * 2 + 1] = maps.a[g * 2];
    maps.b[g * 2 + 1] = maps.b[g * 2];
    maps.blo[g * 2 + 1] = maps.blo[g * 2];
    p.M[g] = M;
    p.kblocks[g][0] = (int)((t.d + ATOM - 1) / ATOM);
    p.out[g][0] = outs[g];
  }
  p.N = k; p.BN = t.BN; p.nseg = 1; p.ldo = t.d; p.scale = 1.f;
  p.idesc = make_idesc(eb, false, t.BN, TC_BM);
  const int mt = (M + TC_BM - 1) / TC_BM;
  if (2 * mt * 3 >= t.nsm * 2) {
    // many M tiles (one CTA per SM, non-persistent grid).  3xTF32 is bound
    // by the SMs (the in-smem A split), so K is split when that fills the
    // last wave: config 4 (2 x 128 tiles on 148 SMs) runs 2 waves at 86%
    // occupancy unsplit and 7 waves at 99% with 4 splits (atomic epilogue
    // into the zeroed AV / BV rows): 1169 -> 1069 us.  tf32 / bf16 stream
    // A and B at the HBM rate with the 108-CTA second wave already, and
    // the split (atomics, more waves) measured slower: 403 -> 424 us.
    auto eff = [&](int s) {
      const long items = 2L * mt * s, waves = (items + t.nsm - 1) / t.nsm;
      return (double)items / (double)(waves * t.nsm);
    };
    int best = 1;
    for (int s = 2; t.x3 && s <= 8 && s <= p.kblocks[0][0]; ++s)
      if (eff(s) > eff(best) + 0.05) best = s;
    p.splits = best;
    if (const char* e = dev_knob("GEIG_DENSE_SPLITS")) p.splits = std::max(1, atoi(e));   // developer A/B
  } else {
    p.splits = choose_splits(2 * mt, p.kblocks[0][0], t.nsm);
  }
  p.atomic = p.splits > 1;
  p.split_stride = 0;
  if (p.atomic) {
    for (int g = 0; g < 2; ++g)
      if (cudaMemset2DAsync(outs[g], (size_t)t.d * 4, 0, (size_t)M * 4, k, st) != cudaSuccess)
        return tc_fail(GEIG_ERR_CUDA, "memset AV/BV rows failed");
  }
  dim3 grid(mt, p.splits, 2);
  geig_status s = eb == 2 ? launch<2, false>(maps, p, grid, st, t.nsm)
                          : launch<4, false>(maps, p, grid, st, t.nsm, t.x3 != 0, t.x3 != 0);
  if (s) return s;
  ++*nl;
  return GEIG_OK;
}

// Gram tables of the streamed (k > 64) update on the tensor cores (tf32 /
// 3xTF32 plans): per split s of the d columns (one split per update CTA,
// `splits` = the update grid), the partial rows
//   partial[s][i KP + j]          = sum_{c in split s} V''[i][c] AV''[j][c]   (G'^A)
//   partial[s][KP^2 + i KP + j]   = sum_{c in split s} V''[i][c] AUX[j][c]    (G'^C)
// as two groups of one launch: A operand = AV (group 0) / AUX (group 1), k
// rows, K-major over d (the split's K blocks); B operand = V'' (tf32, or its
// hi / lo planes with the in-smem A split for 3xTF32); store mode at
// split_stride = pstride (deterministic: the update's phase 2 sums the rows
// in fixed order).  The update's phase 1 then forms only the diagonals.
// Needs d / 32 >= splits (no empty split).
inline geig_status gram_dense_tc(TcPlan& t, const float* V, const float* AV, const float* AUX, float* partial,
                                 int64_t pstride, int KP, int splits, cudaStream_t st, int64_t* nl) {
  if (!t.ready || (t.math != GEIG_MATH_TF32 && t.math != GEIG_MATH_3XTF32))
    return tc_fail(GEIG_ERR_STATE, "tensor-core Gram needs a tf32 / 3xTF32 plan");
  const int eb = 4, ATOM = 32;
  const int k = t.k;
  const int kb = (int)((t.d + ATOM - 1) / ATOM);
  if (k > TC_BM || splits < 1 || kb < splits) return tc_fail(GEIG_ERR_UNSUPPORTED, "tensor-core Gram: shape");
  if (t.x3) {   // V's hi / lo planes (V may have changed since the products' split)
    geig_status e = split_v_x3(t, V, st, nl);
    if (e) return e;
  }
  const void* Vop = t.x3 ? (const void*)t.Vx3 : (const void*)V;
  TcMaps maps;
  TcParams p{};
  // one group, two segments (AV, then AUX against the same V): one CTA per
  // split (one wave), two TMEM accumulators
  const float* mats[2] = {AV, AUX};
  for (int sg = 0; sg < 2; ++sg) {
    if (!make_map(&maps.a[sg], mats[sg], eb, t.d, k, t.d, ATOM, TC_BM) ||
        !make_map(&maps.b[sg], Vop, eb, t.d, k, t.d, ATOM, t.BN))
      return tc_fail(GEIG_ERR_CUDA, "tensor map encode (Gram) failed");
    if (t.x3 && !make_map(&maps.blo[sg], (const char*)Vop + (int64_t)k * t.d * eb, eb, t.d, k, t.d, ATOM, t.BN))
      return tc_fail(GEIG_ERR_CUDA, "tensor map encode (Gram lo) failed");
    p.kblocks[0][sg] = kb;
    p.out[0][sg] = partial + (int64_t)sg * KP * KP;
    maps.a[2 + sg] = maps.a[sg];
    maps.b[2 + sg] = maps.b[sg];
    maps.blo[2 + sg] = maps.blo[sg];
  }
  p.M[0] = p.M[1] = k;
  p.N = k; p.BN = t.BN; p.nseg = 2; p.ldo = KP; p.scale = 1.f;
  p.idesc = make_idesc(eb, false, t.BN, TC_BM);
  p.splits = splits;
  p.atomic = 0;
  p.split_stride = pstride;
  dim3 grid(1, splits, 1);
  geig_status s = launch<4, false>(maps, p, grid, st, t.nsm, t.x3 != 0, t.x3 != 0);
  if (s) return s;
  ++*nl;
  return GEIG_OK;
}

}}  // namespace geig::tc
