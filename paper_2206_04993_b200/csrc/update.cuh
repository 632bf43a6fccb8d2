// update.cuh — stages a2-a4 of the hot path in ONE cooperative kernel:
// Gram tables, penalty coefficients, fused ascent/retraction/aux update.
//
// PAPER.md:1013-1025 (Alg. 2 lines 8-19).  With the products AV_j = A_t v_j,
// BV_j = B_t v_j and G^A_ij = <v_i, AV_j>, G^C_ij = <v_i, [Bv]_j>,
// G^B_ii = <v_i, BV_i>, s_j^2 = max(G^C_jj, rho) (line 8), player i's
// direction (lines 10-12) expands to
//   grad_i = G^B_ii AV_i - (G^A_ii - c_i) BV_i - sum_{j<i} L_ij [Bv]_j,
//   L_ij = G^B_ii G^A_ij / s_j^2,   c_i = sum_{j<i} G^A_ij G^C_ij / s_j^2,
// because (v_i^T A y_j) = G^A_ij / s_j, [By]_j = [Bv]_j / s_j and
// <v_i, [By]_j> = G^C_ij / s_j.  Then v_i' = v_i + eta grad_i,
// v_i <- v_i'/||v_i'|| (lines 16-17), [Bv]_i += gamma (BV_i - [Bv]_i) (19).
//
// Retraction folded forward: the state holds v'' = v + eta grad (line 16)
// and the division by ||v''|| (line 17) is applied when the next update
// reads it — products are linear in v, so A_t v = (A_t v'')/||v''||, and
// ||v''||^2 is one more diagonal of the Gram phase.  This removes a global
// reduction + grid barrier and a pass over V per step (geig_get returns
// the retracted v).
//
// One CTA (256 threads) per SM owns a contiguous column range of d; the
// four k x range tiles (V'', AV'', [Bv], BV'') stream through shared memory
// in 32-column sub-chunks with double-buffered cp.async (16-byte, zero-fill
// past the range).  Phases (grid.sync between them):
//  1  per-CTA Gram partials: G^A, G^C as 4x4 register micro-tiles per
//     thread (rows t, t+16, t+32, t+48 of each 64-row block: conflict-free
//     LDS.128 with a 36-float row stride), lower 64-blocks only; diagonals
//     <v''_i, BV''_i> and ||v''_i||^2.
//  2  deterministic reduction of the per-CTA partials (fixed order).
//  3  every CTA: normalisation factors, coefficients L (transposed in
//     smem), D1, D2; then stream the tiles again: L [Bv] micro-tiles,
//     grad, v'' (in place, + bf16 copy for the GEMMs), [Bv]' (in place).
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"
#include "tc_gemm.cuh"

namespace geig {

namespace cg = cooperative_groups;

constexpr int UPD_THREADS = 256;
constexpr int UPD_XC = 32;             // columns per sub-chunk
constexpr int UPD_S = UPD_XC + 4;      // smem row stride (36 == 4 mod 32)

struct UpdateArgs {
  float* V;              // k x d (in/out)
  float* AUX;            // k x d (in/out)
  const float* AV;       // k x d
  const float* BV;       // k x d
  __nv_bfloat16* Vbf;    // 2 x k x d bf16 shadow of the new V: hi plane, then lo = bf16(v - hi) (nullable)
  float* partial;        // gridDim x (2*KP*KP + 2*KP) scratch
  float* raw;            // 2*KP*KP + 2*KP reduced un-normalised tables
  float* raw_a;          // nullable: the first half of the resident raw row (tri(G^A) | diag G^B)
                         // lives here instead of raw (multi-GPU: summed over ranks with AV, BV)
  float* gram;           // 3 x k x k out: normalised GA, GB, GC of the step
  // Column-owned multi-GPU step (geig_set_partition): 0 = off.
  //  ld: row stride of V, AUX (and the Adam moments) when the update covers
  //      a column block [c0, c0 + d) of a wider state (V, AUX pre-offset);
  //  vbf_ld / vbf_lo: row stride / lo-plane offset of the bf16 shadow written
  //      by the update (the rank's block of the gathered shadow);
  //  own0, own1: the rank's columns — G^C and ||v''||^2 partials are formed
  //      over them only (the rest of the replicated state is stale);
  //  tout, tN, tstride: the reduced table row is written into tN chunks of
  //      tstride floats (one per rank, for the reduce-scatter)
  int64_t ld, vbf_ld, vbf_lo, own0, own1, tstride;
  float* tout;
  int tN;
  // Peer exchange of the column-owned step (geig_set_peers; nullptr = off):
  //  tpeer[r]: owner r's receive buffer (peer-mapped); the table row goes to
  //      tpeer[r] + tpeer_off (this rank's slot) instead of tout + r tstride;
  //  vpeer[0 .. vpeer_n): the other ranks' gathered shadows (peer-mapped):
  //      the update writes its shadow block into every peer's copy too
  float* tpeer[GEIG_MAX_PEERS];
  int64_t tpeer_off;
  __nv_bfloat16* vpeer[GEIG_MAX_PEERS];
  int vpeer_n;
  int k;
  int64_t d;
  int64_t segw;          // columns per CTA (multiple of 4)
  float eta, gamma, rho;
  unsigned long long* ts;  // 6 %globaltimer stamps of CTA 0 (phase boundaries), nullable
  unsigned long long* dbg; // developer: 64 stamps per CTA (%globaltimer, then clock64) (fused step), nullable
  int dbg_mode;            // developer timing knobs (results wrong when set)
  int ga_done;             // fused step: phase S wrote tri(G^A), diag(G^B) of the partial rows
  int pre_reduced;         // fused step: partial rows written and reduced into raw during F/S/B
  // Alg. 3 (smooth gamma-EigenGame): s_j^2 = exp(log rho +
  // (log nu - log rho) sigmoid(z_j)); z double-buffered: step t of a launch
  // reads zbuf[(zpar + t) & 1] and writes zbuf[(zpar + t + 1) & 1] (64 each)
  int smooth;
  float* zbuf;
  int zpar;
  float lnrho, lnnu;
  // Adam ascent on v_i (Appendix H): moments am, as (k x d);
  // step t of a launch uses bias corrections of the global count adam_t0 + t + 1
  int pair_tiles;          // fused CTA pairs: AV, BV tiles already in smem, V'' / [Bv] staged on the tile barrier
  int gram_tc;             // streamed update (k > 64): G'^A, G'^C partial rows written by the tensor-core Gram
                           // launch (tc::gram_dense_tc); phase 1 forms only the diagonals
  int adam;
  float* am;
  float* as;
  float b1, b2, eps;
  long long adam_t0;
};

// developer timeline stamp: slot `slot` of this CTA (thread 0 only)
__device__ __forceinline__ void dstamp(const UpdateArgs& p, int slot) {
  if (p.dbg && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) :: "memory");
    p.dbg[(size_t)blockIdx.x * 64 + slot] = t;
    p.dbg[(size_t)blockIdx.x * 64 + 32 + slot] = clock64();
  }
}

// developer timeline stamp by the calling thread (role threads of the fused kernel)
__device__ __forceinline__ void tstamp(const UpdateArgs& p, int slot) {
  if (p.dbg) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) :: "memory");
    p.dbg[(size_t)blockIdx.x * 64 + slot] = t;
    p.dbg[(size_t)blockIdx.x * 64 + 32 + slot] = clock64();
  }
}

// bf16 "x2" shadow of v: hi = bf16(v), lo = bf16(v - hi); the products may
// use hi alone (bf16) or hi + lo (bf16x2, ~fp32-accurate operand).
__device__ __forceinline__ void store_vbf4(__nv_bfloat16* hi, int64_t lo_off, size_t o, float4 v) {
  const __nv_bfloat162 h0 = __floats2bfloat162_rn(v.x, v.y), h1 = __floats2bfloat162_rn(v.z, v.w);
  const float2 f0 = __bfloat1622float2(h0), f1 = __bfloat1622float2(h1);
  const __nv_bfloat162 l0 = __floats2bfloat162_rn(v.x - f0.x, v.y - f0.y), l1 = __floats2bfloat162_rn(v.z - f1.x, v.w - f1.y);
  uint2 ph, pl;
  ph.x = *reinterpret_cast<const uint32_t*>(&h0); ph.y = *reinterpret_cast<const uint32_t*>(&h1);
  pl.x = *reinterpret_cast<const uint32_t*>(&l0); pl.y = *reinterpret_cast<const uint32_t*>(&l1);
  *reinterpret_cast<uint2*>(hi + o) = ph;
  *reinterpret_cast<uint2*>(hi + lo_off + o) = pl;
}
__device__ __forceinline__ void store_vbf1(__nv_bfloat16* hi, int64_t lo_off, size_t o, float v) {
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  hi[o] = h;
  hi[lo_off + o] = __float2bfloat16_rn(v - __bfloat162float(h));
}

__device__ __forceinline__ void stamp(const UpdateArgs& p, int slot) {
  if (p.ts && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) :: "memory");
    p.ts[slot] = t;
  }
}

__host__ __device__ constexpr size_t upd_smem_floats(int NB) {
  // double buffer of 4 tiles + phase-3 Lt (row stride KP + 4) + n, s^2, D1, D2
  return (size_t)2 * 4 * (NB * 64) * UPD_S + (size_t)(NB * 64) * (NB * 64 + 4) + 4 * (NB * 64);
}
__host__ __device__ constexpr size_t upd_partial_floats(int NB) { return 2 * (NB * 64) * (NB * 64) + 2 * (NB * 64); }

__device__ __forceinline__ void cp_async16(float* dst, const float* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async4(float* dst, const float* src, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Stage rows [0, KP) x columns [x0, x0+32) of the four k x d arrays into
// tiles[4][KP][UPD_S]; rows >= k and columns >= xend are zero-filled.
template <int KP, bool VEC>
__device__ __forceinline__ void stage_tiles(float* tiles, const float* s0, const float* s1, const float* s2,
                                            const float* s3, int k, int64_t d, int64_t x0, int64_t xend) {
  if (VEC) {
    constexpr int Q = UPD_XC / 4;                 // float4 per row
    for (int e = threadIdx.x; e < 4 * KP * Q; e += UPD_THREADS) {
      const int a = e / (KP * Q), rem = e % (KP * Q), r = rem / Q, q = rem % Q;
      const int64_t gx = x0 + 4 * q;
      const bool ok = r < k && gx < xend;
      // (four pointer arguments: a runtime-indexed pointer array lived in
      // local memory — ncu: 7% of the k > 64 update's stall samples)
      const float* base = a == 0 ? s0 : a == 1 ? s1 : a == 2 ? s2 : s3;
      const float* s = ok ? base + (int64_t)r * d + gx : base;
      cp_async16(tiles + ((size_t)a * KP + r) * UPD_S + 4 * q, s, ok ? 16 : 0);
    }
  } else {
    for (int e = threadIdx.x; e < 4 * KP * UPD_XC; e += UPD_THREADS) {
      const int a = e / (KP * UPD_XC), rem = e % (KP * UPD_XC), r = rem / UPD_XC, x = rem % UPD_XC;
      const int64_t gx = x0 + x;
      const bool ok = r < k && gx < xend;
      const float* base = a == 0 ? s0 : a == 1 ? s1 : a == 2 ? s2 : s3;
      const float* s = ok ? base + (int64_t)r * d + gx : base;
      cp_async4(tiles + ((size_t)a * KP + r) * UPD_S + x, s, ok ? 4 : 0);
    }
  }
}

template <int NB, bool VEC>
__global__ void __launch_bounds__(UPD_THREADS, 1)
update_kernel(UpdateArgs p) {
  constexpr int KP = NB * 64;
  constexpr int TILE = KP * UPD_S;               // floats per array tile
  constexpr int NPAIR = NB * (NB + 1) / 2;       // lower 64-block pairs
  constexpr int PSTRIDE = 2 * KP * KP + 2 * KP;  // per-CTA partial: GA', GC', diag GB', diag V'V'
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) float smem[];
  float* buf0 = smem;                            // [4][KP][UPD_S]
  float* buf1 = smem + 4 * TILE;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int k = p.k;
  const int64_t d = p.d;
  const int64_t c0 = (int64_t)blockIdx.x * p.segw;
  const int64_t c1 = min(d, c0 + p.segw);
  const int nsub = c1 > c0 ? (int)((c1 - c0 + UPD_XC - 1) / UPD_XC) : 0;
  // tile order (stage_tiles): 0 V', 1 AV', 2 AUX, 3 BV'
  stamp(p, 0);

  // ---------------- phase 1: Gram partial sums of this CTA's columns ----------------
  if (p.gram_tc) {
    // G'^A, G'^C of this CTA's partial row came from the tensor cores: the
    // diagonals <v''_i, BV''_i> and ||v''_i||^2 of its columns (warp per row)
    // (thread pair per row, each half of the column quads, every load of a
    // thread independent of the others: one L2 round trip, not one per row)
    float* out = p.partial + (size_t)blockIdx.x * PSTRIDE;
    static_assert(2 * KP <= UPD_THREADS || KP > 64, "thread pairs cover the rows");
    for (int i0 = 0; i0 < KP; i0 += UPD_THREADS / 2) {
      const int i = i0 + (tid >> 1), h = tid & 1;
      float gb = 0.f, nn = 0.f;
      if (i < k) {
        const float* vr = p.V + (int64_t)i * d;
        const float* br = p.BV + (int64_t)i * d;
        if (VEC) {
#pragma unroll 8
          for (int64_t x = c0 + 4 * h; x < c1; x += 8) {
            const float4 v = *reinterpret_cast<const float4*>(vr + x);
            const float4 bb = *reinterpret_cast<const float4*>(br + x);
            gb = fmaf(v.x, bb.x, fmaf(v.y, bb.y, fmaf(v.z, bb.z, fmaf(v.w, bb.w, gb))));
            nn = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, nn))));
          }
        } else {
          for (int64_t x = c0 + h; x < c1; x += 2) {
            gb = fmaf(vr[x], br[x], gb);
            nn = fmaf(vr[x], vr[x], nn);
          }
        }
      }
      gb += __shfl_xor_sync(0xffffffffu, gb, 1);
      nn += __shfl_xor_sync(0xffffffffu, nn, 1);
      if (h == 0 && i < KP) {
        out[2 * KP * KP + i] = gb;
        out[2 * KP * KP + KP + i] = nn;
      }
    }
  } else {
    const int ti = tid & 15, tj = tid >> 4;
    float accA[NPAIR][4][4], accC[NPAIR][4][4];
#pragma unroll
    for (int pr = 0; pr < NPAIR; ++pr)
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) accA[pr][a][b] = accC[pr][a][b] = 0.f;
    float gb[KP / 8], nn[KP / 8];
#pragma unroll
    for (int q = 0; q < KP / 8; ++q) gb[q] = nn[q] = 0.f;

    if (nsub > 0) stage_tiles<KP, VEC>(buf0, p.V, p.AV, p.AUX, p.BV, k, d, c0, c1);
    cp_async_commit();
    for (int sc = 0; sc < nsub; ++sc) {
      float* cur = (sc & 1) ? buf1 : buf0;
      float* nxt = (sc & 1) ? buf0 : buf1;
      if (sc + 1 < nsub) stage_tiles<KP, VEC>(nxt, p.V, p.AV, p.AUX, p.BV, k, d, c0 + (int64_t)(sc + 1) * UPD_XC, c1);
      cp_async_commit();
      cp_async_wait<1>();
      __syncthreads();
      const float* Vt = cur;
      const float* At = cur + TILE;
      const float* Ct = cur + 2 * TILE;
      const float* Bt = cur + 3 * TILE;
#pragma unroll 2
      for (int xq = 0; xq < UPD_XC / 4; ++xq) {
        int pr = 0;
#pragma unroll
        for (int bi = 0; bi < NB; ++bi) {
          float4 va[4];
#pragma unroll
          for (int a = 0; a < 4; ++a)
            va[a] = *reinterpret_cast<const float4*>(Vt + (bi * 64 + ti + 16 * a) * UPD_S + 4 * xq);
#pragma unroll
          for (int bj = 0; bj <= bi; ++bj, ++pr) {
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const int j = bj * 64 + tj + 16 * b;
              const float4 pa = *reinterpret_cast<const float4*>(At + j * UPD_S + 4 * xq);
              const float4 pc = *reinterpret_cast<const float4*>(Ct + j * UPD_S + 4 * xq);
#pragma unroll
              for (int a = 0; a < 4; ++a) {
                accA[pr][a][b] = fmaf(va[a].x, pa.x, fmaf(va[a].y, pa.y, fmaf(va[a].z, pa.z, fmaf(va[a].w, pa.w, accA[pr][a][b]))));
                accC[pr][a][b] = fmaf(va[a].x, pc.x, fmaf(va[a].y, pc.y, fmaf(va[a].z, pc.z, fmaf(va[a].w, pc.w, accC[pr][a][b]))));
              }
            }
          }
        }
      }
      // diagonals <v'_i, BV'_i> and <v'_i, v'_i>: warp w owns rows w + 8q
#pragma unroll
      for (int q = 0; q < KP / 8; ++q) {
        const int i = warp + 8 * q;
        const float v = Vt[i * UPD_S + lane];
        gb[q] = fmaf(v, Bt[i * UPD_S + lane], gb[q]);
        nn[q] = fmaf(v, v, nn[q]);
      }
      __syncthreads();
    }
    cp_async_wait<0>();
    float* out = p.partial + (size_t)blockIdx.x * PSTRIDE;
    {
      // the micro-tiles go through the idle tile buffers (row stride KP + 4:
      // the 16 ti lanes of a store hit distinct banks) and leave as coalesced
      // float4 rows of the lower 64-blocks — the direct lane-per-row stores
      // were uncoalesced (ncu: lg_throttle, 8% of the stall samples)
      constexpr int KPS = KP + 4;
      static_assert(2 * KP * KPS <= 8 * TILE, "Gram partials exceed the idle tile buffers");
      float* sA = smem;
      float* sC = smem + KP * KPS;
      int pr = 0;
#pragma unroll
      for (int bi = 0; bi < NB; ++bi)
#pragma unroll
        for (int bj = 0; bj <= bi; ++bj, ++pr)
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const int i = bi * 64 + ti + 16 * a, j = bj * 64 + tj + 16 * b;
              sA[i * KPS + j] = accA[pr][a][b];
              sC[i * KPS + j] = accC[pr][a][b];
            }
      __syncthreads();
      // row i of 64-block bi: columns [0, 64 (bi + 1)) (the blocks bj <= bi)
      for (int e = tid; e < KP * KP / 4; e += UPD_THREADS) {
        const int i = e / (KP / 4), c4 = e - i * (KP / 4);
        if (4 * c4 < 64 * (i / 64 + 1)) {
          const float4 va = *reinterpret_cast<const float4*>(sA + i * KPS + 4 * c4);
          const float4 vc = *reinterpret_cast<const float4*>(sC + i * KPS + 4 * c4);
          __stcg(reinterpret_cast<float4*>(out + i * KP + 4 * c4), va);
          __stcg(reinterpret_cast<float4*>(out + KP * KP + i * KP + 4 * c4), vc);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < KP / 8; ++q) {
      const float s1 = warp_sum(gb[q]);
      const float s2 = warp_sum(nn[q]);
      if (lane == 0) {
        out[2 * KP * KP + warp + 8 * q] = s1;
        out[2 * KP * KP + KP + warp + 8 * q] = s2;
      }
    }
  }   // (gram_tc else)
  grid.sync();
  stamp(p, 1);

  // ---------------- phase 2: reduce the per-CTA partials -> raw tables ----------------
  // Warp w of CTA c reduces the 32-entry groups c + G w, c + G (w + 8), ...:
  // each lane sums one entry over all G partial rows in a fixed order (8
  // interleaved accumulators, 32 loads in flight per lane), so a CTA's groups
  // proceed in parallel instead of one group per pair of CTA barriers (ncu:
  // the group-at-a-time loop was a chain of L2 round trips, ~10 us).
  {
    const int ngroups = (PSTRIDE + 31) / 32;
    const int G = gridDim.x;
    for (int grp = blockIdx.x + G * warp; grp < ngroups; grp += G * (UPD_THREADS / 32)) {
      const int e = grp * 32 + lane;
      bool ok = e < PSTRIDE;
      if (ok && e < 2 * KP * KP) {
        const int q = e % (KP * KP), i = q / KP, j = q % KP;
        ok = i < k && j < k && i >= j;
      } else if (ok) {
        ok = (e - 2 * KP * KP) % KP < k;
      }
      if (ok) {
        const float* srcp = p.partial + e;
        float s[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) s[u] = 0.f;
        int b = 0;
#pragma unroll 4
        for (; b + 8 <= G; b += 8)
#pragma unroll
          for (int u = 0; u < 8; ++u) s[u] += __ldcg(srcp + (size_t)(b + u) * PSTRIDE);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (b + u < G) s[u] += __ldcg(srcp + (size_t)(b + u) * PSTRIDE);
        p.raw[e] = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
      }
    }
  }
  dstamp(p, 11);
  grid.sync();
  stamp(p, 2);
  dstamp(p, 12);

  // ---------------- phase 3a: coefficients (every CTA, from the raw tables) ----------------
  // Normalisation folded in (retraction of the previous step, Alg. 2 line 17):
  // n_i = 1/||v'_i||, v_i = n_i v'_i, AV_i = n_i AV'_i, BV_i = n_i BV'_i, so
  // G^A_ij = n_i n_j G'^A_ij, G^C_ij = n_i G'^C_ij, G^B_ii = n_i^2 G'^B_ii.
  // Lt[j][i] = L_ij, row stride KP + 4: the coefficient loop stores it with
  // lanes over j (stride KP was a 32-way bank conflict, ncu: 32x the ideal
  // wavefronts), the penalty loop reads float4 rows of 4 consecutive i
  constexpr int LTS = KP + 4;
  float* Lt = smem + 8 * TILE;                   // [KP][LTS]
  float* Ns = Lt + KP * LTS;                      // n_i
  float* S2 = Ns + KP;                           // s_j^2 = max(G^C_jj, rho)
  float* D1s = S2 + KP;                          // G^B_ii
  float* D2s = D1s + KP;                         // G^A_ii - c_i
  {
    // The lower triangles of the raw G^A, G^C tables (written by phase 2 of
    // all CTAs, L2-resident) are staged into the idle tile buffers first:
    // every thread issues its float4 loads back to back, instead of the
    // coefficient loop below waiting one L2 round trip per (row, 32 j)
    // step (ncu: 11% of the kernel's stall samples on those loads).
    const float* rA = p.raw;
    const float* rC = p.raw + KP * KP;
    const float* rB = p.raw + 2 * KP * KP;
    const float* rN = rB + KP;
    float* sA = smem;                            // [KP][KP] (lower triangle, rows < k), in buf0/buf1
    float* sC = smem + KP * KP;
    static_assert(2 * KP * KP <= 8 * TILE, "raw tables exceed the idle tile buffers");
#pragma unroll 4
    for (int e = tid; e < KP * KP / 4; e += UPD_THREADS) {
      const int r = e / (KP / 4), c4 = e - r * (KP / 4);
      if (r < k && 4 * c4 <= r) {
        *reinterpret_cast<float4*>(sA + 4 * e) = __ldcg(reinterpret_cast<const float4*>(rA) + e);
        *reinterpret_cast<float4*>(sC + 4 * e) = __ldcg(reinterpret_cast<const float4*>(rC) + e);
      }
    }
    __syncthreads();
    for (int i = tid; i < KP; i += UPD_THREADS) {
      float n = 0.f, s2 = 1.f, gb = 0.f;
      if (i < k) {
        n = rsqrtf(rN[i]);
        gb = n * n * rB[i];
        s2 = fmaxf(n * sC[i * KP + i], p.rho);
      }
      Ns[i] = n; S2[i] = s2; D1s[i] = gb;
    }
    __syncthreads();
    // 1 / s_j^2 once per j (the loop below divided k^2 times per CTA)
    float rs2[KP / 32];
#pragma unroll
    for (int m = 0; m < KP / 32; ++m) rs2[m] = 1.f / S2[lane + 32 * m];
    for (int i = warp; i < KP; i += UPD_THREADS / 32) {
      const float ni = Ns[i];
      float c = 0.f;
#pragma unroll
      for (int m = 0; m < KP / 32; ++m) {
        const int j = lane + 32 * m;
        float l = 0.f;
        if (i < k && j < i) {
          const float ga = ni * Ns[j] * sA[i * KP + j];
          const float gc = ni * sC[i * KP + j];
          l = D1s[i] * ga * rs2[m];
          c = fmaf(ga, gc * rs2[m], c);
        }
        Lt[j * LTS + i] = l;
      }
      c = warp_sum(c);
      if (lane == 0) D2s[i] = i < k ? ni * ni * sA[i * KP + i] - c : 0.f;
    }
    {
      // diagnostics: normalised tables of the iteration-start state (slices over the CTAs)
      const int kk = k * k, per = (kk + (int)gridDim.x - 1) / (int)gridDim.x;
      const int e1 = min(kk, (int)(blockIdx.x + 1) * per);
      for (int e = blockIdx.x * per + tid; e < e1; e += UPD_THREADS) {
        const int i = e / k, j = e % k;
        const bool low = j <= i;
        p.gram[e] = low ? rsqrtf(rN[i]) * rsqrtf(rN[j]) * rA[i * KP + j] : 0.f;
        p.gram[(size_t)k * k + e] = (i == j) ? rB[i] / rN[i] : 0.f;
        p.gram[2 * (size_t)k * k + e] = low ? rsqrtf(rN[i]) * rC[i * KP + j] : 0.f;
      }
    }
    __syncthreads();
  }

  // ---------------- phase 3b: grad, v'' and [Bv]' for this CTA's columns ----------------
  {
    const int tx = tid & 7;            // columns 4tx..4tx+3 of the sub-chunk
    // Penalty sums sum_{j<i} L_ij [Bv]_j: row i needs i terms, so a fixed
    // row-group-per-thread mapping leaves the last rows' threads with twice
    // the average work.  NB == 2 (k > 64): thread pair (h = 0, 1; lanes l,
    // l ^ 8) owns row groups g1 = q and g2 = 31 - q (4 rows each), splits
    // their j range by alternating 4-blocks (h takes j0 = 4h, 4h + 8, ...)
    // and exchanges the partial sums by one shuffle, so every thread does
    // (g1 + g2 + 2) / 2 = 16.5 4-blocks; thread h writes back group g1 (h = 0)
    // or g2 (h = 1).  NB == 1: one row group per thread (tr = tid >> 3).
    const int hh = (tid >> 3) & 1;
    const int q = tid >> 4;
    const int i0 = NB == 2 ? 4 * (hh ? 31 - q : q) : 4 * (tid >> 3);
    if (nsub > 0) stage_tiles<KP, VEC>(buf0, p.V, p.AV, p.AUX, p.BV, k, d, c0, c1);
    cp_async_commit();
    for (int sc = 0; sc < nsub; ++sc) {
      float* cur = (sc & 1) ? buf1 : buf0;
      float* nxt = (sc & 1) ? buf0 : buf1;
      if (sc + 1 < nsub) stage_tiles<KP, VEC>(nxt, p.V, p.AV, p.AUX, p.BV, k, d, c0 + (int64_t)(sc + 1) * UPD_XC, c1);
      cp_async_commit();
      cp_async_wait<1>();
      __syncthreads();
      const float* Vt = cur;
      const float* At = cur + TILE;
      const float* Ct = cur + 2 * TILE;
      const float* Bt = cur + 3 * TILE;
      float acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
      if constexpr (NB == 2) {
        // j bounds rounded up to multiples of 4 (L_ij = 0 for j >= i, rows
        // of the staged tiles past k are zero)
        const int kr = (k + 3) & ~3;
        const int r1 = 4 * q, r2 = 4 * (31 - q);
        const int jm1 = min(r1 + 4, kr), jm2 = min(r2 + 4, kr);
        float a1[4][4], a2[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) a1[a][b] = a2[a][b] = 0.f;
        int j0 = 4 * hh;
#pragma unroll 1
        for (; j0 < jm1; j0 += 8) {      // both groups
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float4 l1 = *reinterpret_cast<const float4*>(Lt + (j0 + u) * LTS + r1);
            const float4 l2 = *reinterpret_cast<const float4*>(Lt + (j0 + u) * LTS + r2);
            const float4 x = *reinterpret_cast<const float4*>(Ct + (j0 + u) * UPD_S + 4 * tx);
            const float lv1[4] = {l1.x, l1.y, l1.z, l1.w}, lv2[4] = {l2.x, l2.y, l2.z, l2.w};
            const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int b = 0; b < 4; ++b) {
                a1[a][b] = fmaf(lv1[a], xv[b], a1[a][b]);
                a2[a][b] = fmaf(lv2[a], xv[b], a2[a][b]);
              }
          }
        }
#pragma unroll 1
        for (; j0 < jm2; j0 += 8) {      // group g2 only
          float4 l[4], x[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            l[u] = *reinterpret_cast<const float4*>(Lt + (j0 + u) * LTS + r2);
            x[u] = *reinterpret_cast<const float4*>(Ct + (j0 + u) * UPD_S + 4 * tx);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float lv[4] = {l[u].x, l[u].y, l[u].z, l[u].w}, xv[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int b = 0; b < 4; ++b) a2[a][b] = fmaf(lv[a], xv[b], a2[a][b]);
          }
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const float other = __shfl_xor_sync(0xffffffffu, hh ? a1[a][b] : a2[a][b], 8);
            acc[a][b] = (hh ? a2[a][b] : a1[a][b]) + other;
          }
      } else if (i0 < KP) {
        // j bound rounded up to a multiple of 4 (L_ij = 0 for j >= i, rows of
        // the staged tiles past k are zero): 4 j per branch-free iteration
        const int jmax = min(i0 + 4, (k + 3) & ~3);
#pragma unroll 1
        for (int j0 = 0; j0 < jmax; j0 += 4) {
          float4 l[4], x[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            l[u] = *reinterpret_cast<const float4*>(Lt + (j0 + u) * LTS + i0);
            x[u] = *reinterpret_cast<const float4*>(Ct + (j0 + u) * UPD_S + 4 * tx);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float lv[4] = {l[u].x, l[u].y, l[u].z, l[u].w}, xv[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(lv[a], xv[b], acc[a][b]);
          }
        }
      }
      const int64_t gx = c0 + (int64_t)sc * UPD_XC + 4 * tx;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int i = i0 + a;
        if (i < k && gx < c1) {
          const float4 av = *reinterpret_cast<const float4*>(At + i * UPD_S + 4 * tx);
          const float4 bv = *reinterpret_cast<const float4*>(Bt + i * UPD_S + 4 * tx);
          const float4 vv = *reinterpret_cast<const float4*>(Vt + i * UPD_S + 4 * tx);
          const float4 xa = *reinterpret_cast<const float4*>(Ct + i * UPD_S + 4 * tx);
          const float ni = Ns[i];
          const float d1 = D1s[i] * ni, d2 = D2s[i] * ni;
          float4 vn, an;
          vn.x = ni * vv.x + p.eta * (d1 * av.x - d2 * bv.x - acc[a][0]);
          vn.y = ni * vv.y + p.eta * (d1 * av.y - d2 * bv.y - acc[a][1]);
          vn.z = ni * vv.z + p.eta * (d1 * av.z - d2 * bv.z - acc[a][2]);
          vn.w = ni * vv.w + p.eta * (d1 * av.w - d2 * bv.w - acc[a][3]);
          an.x = xa.x + p.gamma * (ni * bv.x - xa.x);
          an.y = xa.y + p.gamma * (ni * bv.y - xa.y);
          an.z = xa.z + p.gamma * (ni * bv.z - xa.z);
          an.w = xa.w + p.gamma * (ni * bv.w - xa.w);
          const size_t o = (size_t)i * d + gx;
          if (VEC && gx + 3 < c1) {
            *reinterpret_cast<float4*>(p.V + o) = vn;
            *reinterpret_cast<float4*>(p.AUX + o) = an;
            if (p.Vbf) store_vbf4(p.Vbf, (int64_t)k * d, o, vn);
          } else {
            const float vs[4] = {vn.x, vn.y, vn.z, vn.w}, as[4] = {an.x, an.y, an.z, an.w};
            for (int t = 0; t < 4; ++t)
              if (gx + t < c1) {
                p.V[o + t] = vs[t];
                p.AUX[o + t] = as[t];
                if (p.Vbf) store_vbf1(p.Vbf, (int64_t)k * d, o + t, vs[t]);
              }
          }
        }
      }
      __syncthreads();
    }
    cp_async_wait<0>();
  }
  stamp(p, 3);
}

// ============================================================================
// Resident variant (k <= 64): every CTA loads its four k x W tiles ONCE
// (one cp.async burst, maximal memory-level parallelism), computes the Gram
// partials and, after the two grid barriers, the update from the same
// shared-memory tiles.  Compact lower-triangular reduction: raw layout
// [tri(A) | tri(C) | diag B | diag V'V'] with tri(i,j) = i(i+1)/2 + j.
// ============================================================================
constexpr int UPD_RES_WMAX = 168;   // max columns per CTA (smem: 4 x 64 x 172 x 4 B + tables)
constexpr int UPD_GT = 72;          // 8x4 lower-triangle Gram tiles of a 64 x 64 table
constexpr int UPD_GS = 3;           // column slices of the Gram phase (UPD_GT * UPD_GS <= UPD_THREADS)
// developer timing knobs (GEIG_DBG_MODE / GEIG_DBG_NOSTORE: skip work, wrong
// results) are compiled in only with -DGEIG_DEV_KNOBS=1 (GEIG_NVCC_EXTRA)
constexpr bool kDevKnobs = GEIG_DEV_KNOBS;
constexpr int UPD_LTS = 72;         // Lt row stride (padded)
constexpr int UPD_AUXF = 64 * UPD_LTS + 4 * 64 + 8 * 32 + 64 * 65 + 128;   // Lt | N, 1/s^2, D1, D2 | red | raw
constexpr int UPD_GREDF = (UPD_GS - 1) * UPD_GT * 64;                // Gram slice partials (aliases the above)

__host__ __device__ constexpr size_t upd_res_smem_floats(int W) {
  // 4 tiles + max(tables, Gram slice buffer) + TMA mbarrier (16 B)
  return (size_t)4 * 64 * (W + 4) + (UPD_AUXF > UPD_GREDF ? UPD_AUXF : UPD_GREDF) + 4;
}
__host__ __device__ constexpr int upd_raw_floats_res(int k) { return 2 * ((k * (k + 1) / 2 + k + 3) & ~3); }   // 2 padded halves

__device__ __forceinline__ int tri_index(int i, int j) { return i * (i + 1) / 2 + j; }

// ---------------------------------------------------------------------------
// Fused step side work for the otherwise idle warps 2-3 (64 threads, no smem
// beyond a 64-float scratch) of the GEMM phases:
//   during phase F: this CTA's partial G^C_ij = <v''_i, [Bv]_j> (j <= i) and
//     ||v''_i||^2 over its W columns, from global memory (the state is fixed
//     for the whole step), into the second half of its Gram partial row;
//   during phase B: this CTA's slice of the deterministic reduction of all
//     Gram partial rows (complete after phase S) into the raw tables.
// The update phase then starts at the coefficients (UpdateArgs::pre_reduced).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void gram_c_side(const UpdateArgs& p, int t) {
  const int k = p.k;
  const int64_t d = p.d;
  const int W = (int)p.segw;
  int64_t c0 = (int64_t)blockIdx.x * W;
  int64_t c1 = min(d, c0 + W);
  if (p.own1 > p.own0) { c0 = max(c0, p.own0); c1 = min(c1, p.own1); }   // column-owned: own columns only
  const int ntri = k * (k + 1) / 2, hA = (ntri + k + 3) & ~3;
  float* out = p.partial + (size_t)blockIdx.x * (2 * hA) + hA;
  const int nq = c1 > c0 ? (int)((c1 - c0) / 4) : 0;      // d % 4 == 0 on the fused path
  const int I = t & 7, J = t >> 3;                          // rows i = I + 8a, j = J + 8b
  auto ld = [&](const float* base, int r, int q) -> float4 {
    return r < k ? *reinterpret_cast<const float4*>(base + (int64_t)r * d + c0 + 4 * q)
                 : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  float acc[36];
#pragma unroll
  for (int e = 0; e < 36; ++e) acc[e] = 0.f;
#pragma unroll 1
  for (int q = 0; q < nq; ++q) {
    float4 va[8], pc[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      va[a] = ld(p.V, I + 8 * a, q);
      pc[a] = ld(p.AUX, J + 8 * a, q);
    }
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b <= a; ++b) {
        float& c = acc[a * (a + 1) / 2 + b];
        c = fmaf(va[a].x, pc[b].x, c);
        c = fmaf(va[a].y, pc[b].y, c);
        c = fmaf(va[a].z, pc[b].z, c);
        c = fmaf(va[a].w, pc[b].w, c);
      }
  }
  float nn = 0.f;
  if (t < k)
    for (int q = 0; q < nq; ++q) {
      const float4 v = ld(p.V, t, q);
      nn = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, nn))));
    }
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b <= a; ++b) {
      const int i = I + 8 * a, j = J + 8 * b;
      if (i < k && j <= i) out[tri_index(i, j)] = acc[a * (a + 1) / 2 + b];
    }
  if (t < k) out[ntri + t] = nn;
  for (int e = ntri + k + t; e < hA; e += 64) out[e] = 0.f;
}

// Warps 2-3 (named barrier 1, 64 threads): this CTA's slice [e0, e1) of the
// reduction of all Gram partial rows into the raw tables (fixed order).
__device__ __forceinline__ void reduce_side(const UpdateArgs& p, int t, float* scratch) {
  const int k = p.k;
  const int ntri = k * (k + 1) / 2, hA = (ntri + k + 3) & ~3, pstride = 2 * hA;
  const int G = gridDim.x;
  const int per = (pstride + G - 1) / G;
  const int e0 = blockIdx.x * per, e1 = min(pstride, e0 + per);
  const int lane = t & 31, half = t >> 5;
  for (int eb = e0; eb < e1; eb += 32) {
    const int e = eb + lane;
    float s = 0.f;
    if (e < e1) {
      int b = half;
      for (; b + 2 * 15 < G; b += 2 * 16) {      // 16 independent loads in flight
        float v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = p.partial[(size_t)(b + 2 * u) * pstride + e];
#pragma unroll
        for (int u = 0; u < 16; ++u) s += v[u];
      }
      for (; b < G; b += 2) s += p.partial[(size_t)b * pstride + e];
    }
    scratch[t] = s;
    asm volatile("bar.sync 1, 64;" ::: "memory");
    if (half == 0 && e < e1) {
      const float v = s + scratch[t + 32];
      if (p.tN > 0) {
        for (int r = 0; r < p.tN; ++r) {   // every rank's chunk (peer exchange: this rank's slot at owner r)
          if (p.tpeer[0]) p.tpeer[r][p.tpeer_off + e] = v;
          else p.tout[(int64_t)r * p.tstride + e] = v;
        }
      } else if (p.raw_a && e < hA) {
        p.raw_a[e] = v;
      } else {
        p.raw[e] = v;
      }
    }
    asm volatile("bar.sync 1, 64;" ::: "memory");
  }
}

// fp32 k x d state arrays as TMA tensors (box = one CTA's W+4 columns x 64
// rows, no swizzle; rows >= k and columns >= d are zero-filled by the TMA
// unit).  Order: V'', AV, [Bv], BV — the smem tile order.
struct UpdMaps {
  CUtensorMap t[4];
};

// The resident update as a device function over an explicit shared-memory
// arena, so the fused step kernel (fused_step.cuh) can run it after its GEMM
// phases inside the same cooperative launch.  `um` (param-space tensor maps)
// selects TMA staging of the tiles; nullptr stages them with cp.async.
// Coefficients of the update (Alg. 2 lines 8-11, the phase-3a algebra
// below) formed by warps 2-3 of the fused kernel during the backward phase,
// as soon as every CTA's slice of the Gram reduction is in p.raw (64 threads,
// named barrier 1; thread i owns player i).  `cf` (shared memory outside the
// GEMM ring): Lt [64][UPD_LTS] (Lt[j][i] = L_ij) | N | 1/s^2 | D1 | D2.  The
// raw rows are read from global memory (L2): row i of tri(G^A) and tri(G^C)
// is contiguous.  Also writes this CTA's slice of the normalised tables
// (geig_get_gram) and, in CTA 0, the Alg. 3 z ascent.
__device__ __forceinline__ void coef_early(const UpdateArgs& p, float* cf, int step, int t) {
  const int k = p.k;
  const int ntri = k * (k + 1) / 2, hA = (ntri + k + 3) & ~3;
  const float* rA = p.raw_a ? p.raw_a : p.raw;                 // [tri(G^A) | diag(G^B)]
  const float* rB = rA + ntri;
  const float* rC = p.raw + hA;                                 // [tri(G^C) | diag ||v''||^2]
  const float* rN = rC + ntri;
  float* Lt = cf;
  float* Ns = Lt + 64 * UPD_LTS;
  float* IS2 = Ns + 64;
  float* D1s = IS2 + 64;
  float* D2s = D1s + 64;
  const int i = t;
  {
    float n = 0.f, is2 = 0.f, gb = 0.f;
    if (i < k) {
      n = rsqrtf(__ldcg(rN + i));
      gb = n * n * __ldcg(rB + i);
      const float gcii = n * __ldcg(rC + tri_index(i, i));      // <v_i, [Bv]_i>
      if (p.smooth) {
        // Alg. 3 l.7: [<v,Bv>]_i = exp(log rho + (log nu - log rho) sigma(z_i))
        const float* zr = p.zbuf + ((p.zpar + step) & 1) * 64;
        const float z = zr[i];
        const float sg = 1.f / (1.f + expf(-z));
        const float br = expf(p.lnrho + (p.lnnu - p.lnrho) * sg);
        is2 = 1.f / br;
        if (blockIdx.x == 0) {   // l.14 / l.21: z_i += gamma (<v_i,[Bv]_i> - br) br (log nu - log rho) sigma (1 - sigma)
          float* zw = p.zbuf + ((p.zpar + step + 1) & 1) * 64;
          zw[i] = z + p.gamma * (gcii - br) * br * (p.lnnu - p.lnrho) * sg * (1.f - sg);
        }
      } else {
        is2 = 1.f / fmaxf(gcii, p.rho);                        // Alg. 2 l.8
      }
    }
    Ns[i] = n; IS2[i] = is2; D1s[i] = gb;
  }
  asm volatile("bar.sync 1, 64;" ::: "memory");
  // row i: L_ij = G^B_ii G^A_ij / s_j^2 (j < i) into Lt[j][i]; c_i = sum_{j<i} G^A_ij G^C_ij / s_j^2
  {
    const float ni = Ns[i], d1 = D1s[i];
    const int base = i * (i + 1) / 2;
    float c = 0.f;
#pragma unroll 8
    for (int j = 0; j < 64; ++j) {
      float l = 0.f;
      if (i < k && j < i) {
        const float aij = ni * Ns[j] * __ldcg(rA + base + j);
        l = d1 * aij * IS2[j];
        c = fmaf(aij, ni * __ldcg(rC + base + j) * IS2[j], c);
      }
      Lt[j * UPD_LTS + i] = l;
    }
    D2s[i] = i < k ? ni * ni * __ldcg(rA + base + i) - c : 0.f;
  }
  // the step's normalised tables (geig_get_gram), written by all CTAs in slices
  {
    const int G = gridDim.x, kk = k * k;
    const int per = (kk + G - 1) / G;
    const int e1 = min(kk, (int)(blockIdx.x + 1) * per);
    for (int e = blockIdx.x * per + t; e < e1; e += 64) {
      const int ii = e / k, j = e - (e / k) * k;
      const bool low = j <= ii;
      const int tij = tri_index(ii, low ? j : 0);
      p.gram[e] = low ? Ns[ii] * Ns[j] * __ldcg(rA + tij) : 0.f;
      p.gram[(size_t)kk + e] = (ii == j) ? D1s[ii] : 0.f;
      p.gram[2 * (size_t)kk + e] = low ? Ns[ii] * __ldcg(rC + tij) : 0.f;
    }
  }
  asm volatile("bar.sync 1, 64;" ::: "memory");
}

// PRE: -1 runtime p.pre_reduced, 0 / 1 compile-time (fused kernel: 1).
// ADAM: the Appendix-H branch of the write-back is compiled in (runtime
// p.adam); the fused kernel's plain instance leaves it out (its untaken
// per-element branch measured ~1 us of the update phase).
template <bool VEC, int PRE = -1, bool ADAM = true>
__device__ __forceinline__ void update_res_phases(const UpdateArgs& p, float* smem, cg::grid_group& grid,
                                                  const UpdMaps* um = nullptr, int step = 0,
                                                  float* coef = nullptr, uint64_t* tbar_ext = nullptr,
                                                  bool tbar_ready = false) {
  // tbar_ready: the caller initialised tbar_ext (with the init and shared-memory
  // proxy fences) earlier, off this critical path (fused kernel: end of phase F)
  // coef: coefficients already formed (coef_early, fused kernel) — no table
  // staging, phase 3a skipped
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int k = p.k;
  const int64_t d = p.d;                         // columns covered (the block's width when column-owned)
  const int64_t lds = p.ld ? p.ld : d;           // row stride of V, AUX, Adam moments
  const int64_t bld = p.vbf_ld ? p.vbf_ld : lds; // row stride of the bf16 shadow
  const int64_t blo = p.vbf_lo ? p.vbf_lo : (int64_t)k * bld;   // its lo-plane offset
  const int W = (int)p.segw;                     // multiple of 8
  const int S = W + 4;                           // S/4 odd: conflict-free LDS.128 below
  const int64_t c0 = (int64_t)blockIdx.x * W;
  const int64_t c1 = min(d, c0 + W);
  float* Vt = smem;
  float* At = Vt + 64 * S;
  float* Ct = At + 64 * S;
  float* Bt = Ct + 64 * S;
  float* Lt = coef ? coef : Bt + 64 * S;         // [64][UPD_LTS] Lt[j][i]
  float* Ns = Lt + 64 * UPD_LTS;
  float* IS2 = Ns + 64;                          // 1 / s_j^2
  float* D1s = IS2 + 64;
  float* D2s = D1s + 64;
  float* red = D2s + 64;                         // [8][32]
  float* rs = red + 8 * 32;                      // staged raw tables
  float* gred = Lt;                              // phase 1 only: Gram slice partials
  // the tile barrier: outside the arena when the caller provides one (the
  // fused kernel: its barrier region, never a TMA destination)
  uint64_t* tbar = tbar_ext ? tbar_ext
                            : reinterpret_cast<uint64_t*>(Bt + 64 * S + (UPD_AUXF > UPD_GREDF ? UPD_AUXF : UPD_GREDF));
  const int ntri = k * (k + 1) / 2;
  const int hA = (ntri + k + 3) & ~3;            // half row: [tri | diag | pad]
  const int pstride = 2 * hA;                    // per-CTA partial row (16-byte multiple)
  stamp(p, 0);

  // ---------------- stage the four tiles once ----------------
  const bool early_raw = um && !coef && (PRE == 1 || (PRE < 0 && p.pre_reduced));
  if (early_raw) {
    // pre-reduced tables: stage them first (the coefficients need them
    // before the tiles; the tiles' TMA then streams behind them)
    for (int e = 4 * tid; e < pstride; e += 4 * UPD_THREADS)
      cp_async16(rs + e, (p.raw_a && e < hA) ? p.raw_a + e : p.raw + e, 16);
    cp_async_commit();
  }
  if (um) {
    if (p.pair_tiles) {
      // fused CTA pairs: AV, BV tiles written by pair_exchange, V'' and [Bv]
      // in flight on the tile barrier (waited below)
    } else {
    if (warp == 0 && tc::elect_one()) {   // (elected lane: no elect / broadcast loop around the TMA issues)
      asm volatile("fence.proxy.async.global;" ::: "memory");   // state / products written by generic stores
      if (!tbar_ready) {
        tc::mbar_init(tbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // smem last written through the async proxy (GEMM ring) or generic
        // stores of a previous use: order them before the TMA writes below
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
      tc::mbar_expect_tx(tbar, (uint32_t)(4 * 64 * S * 4));
      float* dst[4] = {Vt, At, Ct, Bt};
#pragma unroll
      for (int a = 0; a < 4; ++a) tc::tma_load_2d(dst[a], &um->t[a], tbar, (int)c0, 0);
    }
    __syncthreads();
    // pre-reduced tables (fused step): the coefficients do not read the
    // tiles, so their staging overlaps the coefficient phase (wait below)
    if (!(PRE == 1 || (PRE < 0 && p.pre_reduced))) tc::mbar_wait(tbar, 0);
    }
  } else {
    auto stage = [&](float* dst, const float* src) {
      if (VEC) {
        const int Q = W / 4;
        for (int e = tid; e < 64 * Q; e += UPD_THREADS) {
          const int r = e / Q, q = e - r * Q;
          const int64_t gx = c0 + 4 * q;
          const bool ok = r < k && gx < c1;
          cp_async16(dst + r * S + 4 * q, ok ? src + (int64_t)r * d + gx : src, ok ? 16 : 0);
        }
      } else {
        for (int e = tid; e < 64 * W; e += UPD_THREADS) {
          const int r = e / W, x = e - r * W;
          const int64_t gx = c0 + x;
          const bool ok = r < k && gx < c1;
          cp_async4(dst + r * S + x, ok ? src + (int64_t)r * d + gx : src, ok ? 4 : 0);
        }
      }
    };
    stage(Vt, p.V);
    stage(At, p.AV);
    stage(Ct, p.AUX);
    stage(Bt, p.BV);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
  }
  dstamp(p, 8);

  const bool pre = PRE < 0 ? p.pre_reduced != 0 : PRE != 0;
  if (pre) { stamp(p, 1); stamp(p, 2); }   // phases 1-2 ran as side work of the GEMM phases
  if constexpr (PRE != 1) if (!pre) {
  // ---------------- phase 1: Gram partials ----------------
  // Partial row layout (pstride = 2 hA floats):
  //   [tri(G^A) | diag(G^B) | pad][tri(G^C) | diag ||v''||^2 | pad].
  // With p.ga_done the fused step's phase S has already written the first
  // half from the forward products z (reading R3); only G^C and ||v''||^2
  // are formed here.
  {
    float* out = p.partial + (size_t)blockIdx.x * pstride;
    float* pst = gred;                              // compact partial row, written after the slice reduction
    const int nq = W / 4;
    if (p.ga_done) {
      // G^C_ij = <v''_i, [Bv]_j>, j <= i: 64 tiles (I, J) = (t & 7, t >> 3)
      // of rows i = I + 8a, j = J + 8b (a, b < 8, pairs b <= a: 36 sums),
      // 4 column slices (sl = tid >> 6).  Quarter-warps read 8 consecutive
      // V rows (conflict-free) and one broadcast [Bv] row.
      const int sl = tid >> 6, t = tid & 63;
      const int I = t & 7, J = t >> 3;
      float acc[36];
#pragma unroll
      for (int e = 0; e < 36; ++e) acc[e] = 0.f;
      const int q0 = sl * nq / 4, q1 = (kDevKnobs && (p.dbg_mode & 128)) ? q0 : (sl + 1) * nq / 4;
#pragma unroll 1
      for (int q = q0; q < q1; ++q) {
        float4 va[8], pc[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          va[a] = *reinterpret_cast<const float4*>(Vt + (I + 8 * a) * S + 4 * q);
          pc[a] = *reinterpret_cast<const float4*>(Ct + (J + 8 * a) * S + 4 * q);
        }
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
          for (int b = 0; b <= a; ++b) {
            float& c = acc[a * (a + 1) / 2 + b];
            c = fmaf(va[a].x, pc[b].x, c);
            c = fmaf(va[a].y, pc[b].y, c);
            c = fmaf(va[a].z, pc[b].z, c);
            c = fmaf(va[a].w, pc[b].w, c);
          }
      }
      // ||v''_i||^2: 4 threads per row
      float nn = 0.f;
      {
        const int i = tid >> 2, part = tid & 3;
        for (int q = part; q < nq; q += 4) {
          const float4 v = *reinterpret_cast<const float4*>(Vt + i * S + 4 * q);
          nn = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, nn))));
        }
        nn += __shfl_xor_sync(0xffffffffu, nn, 1);
        nn += __shfl_xor_sync(0xffffffffu, nn, 2);
      }
      if (p.dbg) { __syncthreads(); dstamp(p, 27); }
      if (sl > 0) {
#pragma unroll
        for (int e = 0; e < 36; ++e) gred[(size_t)(sl - 1) * 36 * 64 + e * 64 + t] = acc[e];
      }
      __syncthreads();
      if (sl == 0) {
#pragma unroll
        for (int e = 0; e < 36; ++e)
#pragma unroll
          for (int s2 = 0; s2 < 3; ++s2) acc[e] += gred[(size_t)s2 * 36 * 64 + e * 64 + t];
      }
      __syncthreads();
      if (sl == 0) {
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
          for (int b = 0; b <= a; ++b) {
            const int i = I + 8 * a, j = J + 8 * b;
            if (i < k && j <= i) pst[hA + tri_index(i, j)] = acc[a * (a + 1) / 2 + b];
          }
      }
      if ((tid & 3) == 0 && (tid >> 2) < k) pst[hA + ntri + (tid >> 2)] = nn;
      for (int e = hA + ntri + k + tid; e < pstride; e += UPD_THREADS) pst[e] = 0.f;
      __syncthreads();
      dstamp(p, 28);
      for (int e = hA + 4 * tid; e < pstride; e += 4 * UPD_THREADS)
        *reinterpret_cast<float4*>(out + e) = *reinterpret_cast<const float4*>(pst + e);
    } else {
      // G^A and G^C together: 72 register tiles of 8 rows (i) x 4 rows (j)
      // over the lower triangle, 3 column slices (threads 0..215); threads
      // 216..255 form the diagonals <v''_i, BV''_i> and ||v''_i||^2.
      const bool gt = tid < UPD_GT * UPD_GS;     // warp 6 straddles the two roles: no barrier inside them
      const int sl = gt ? tid / UPD_GT : 0, t = gt ? tid - sl * UPD_GT : 0;
      int I = 0;
      while ((I + 1) * (I + 2) <= t) ++I;          // t = I(I+1) + J, J < 2I+2
      const int J = t - I * (I + 1);
      float accA[8][4], accC[8][4];
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) accA[a][b] = accC[a][b] = 0.f;
      if (gt) {
        const int q0 = sl * nq / UPD_GS, q1 = (sl + 1) * nq / UPD_GS;
        const float* vb = Vt + (8 * I) * S;
        const float* ab = At + (4 * J) * S;
        const float* cb = Ct + (4 * J) * S;
        for (int q = q0; q < q1; ++q) {
          float4 va[8], pa[4], pc[4];
#pragma unroll
          for (int a = 0; a < 8; ++a) va[a] = *reinterpret_cast<const float4*>(vb + a * S + 4 * q);
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            pa[b] = *reinterpret_cast<const float4*>(ab + b * S + 4 * q);
            pc[b] = *reinterpret_cast<const float4*>(cb + b * S + 4 * q);
          }
#pragma unroll
          for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              accA[a][b] = fmaf(va[a].x, pa[b].x, fmaf(va[a].y, pa[b].y, fmaf(va[a].z, pa[b].z, fmaf(va[a].w, pa[b].w, accA[a][b]))));
              accC[a][b] = fmaf(va[a].x, pc[b].x, fmaf(va[a].y, pc[b].y, fmaf(va[a].z, pc[b].z, fmaf(va[a].w, pc[b].w, accC[a][b]))));
            }
        }
        if (sl > 0) {
          float* g = gred + (size_t)(sl - 1) * UPD_GT * 64 + t;
#pragma unroll
          for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              g[(a * 4 + b) * UPD_GT] = accA[a][b];
              g[(32 + a * 4 + b) * UPD_GT] = accC[a][b];
            }
        }
      } else {
        for (int r = 0; r < 2; ++r) {
          const int i = tid - UPD_GT * UPD_GS + r * (UPD_THREADS - UPD_GT * UPD_GS);
          if (i >= k) break;
          float gb = 0.f, nn = 0.f;
          for (int q = 0; q < nq; ++q) {
            const float4 v = *reinterpret_cast<const float4*>(Vt + i * S + 4 * q);
            const float4 bb = *reinterpret_cast<const float4*>(Bt + i * S + 4 * q);
            gb = fmaf(v.x, bb.x, fmaf(v.y, bb.y, fmaf(v.z, bb.z, fmaf(v.w, bb.w, gb))));
            nn = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, nn))));
          }
          accA[0][r] = gb;
          accC[0][r] = nn;
        }
      }
      __syncthreads();
      if (gt && sl == 0) {
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int s2 = 0; s2 < UPD_GS - 1; ++s2) {
              accA[a][b] += gred[(size_t)s2 * UPD_GT * 64 + (a * 4 + b) * UPD_GT + t];
              accC[a][b] += gred[(size_t)s2 * UPD_GT * 64 + (32 + a * 4 + b) * UPD_GT + t];
            }
      }
      __syncthreads();
      if (gt && sl == 0) {
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int i = 8 * I + a, j = 4 * J + b;
            if (i < k && j <= i) {
              pst[tri_index(i, j)] = accA[a][b];
              pst[hA + tri_index(i, j)] = accC[a][b];
            }
          }
      } else if (!gt) {
        for (int r = 0; r < 2; ++r) {
          const int i = tid - UPD_GT * UPD_GS + r * (UPD_THREADS - UPD_GT * UPD_GS);
          if (i < k) {
            pst[ntri + i] = accA[0][r];
            pst[hA + ntri + i] = accC[0][r];
          }
        }
      }
      for (int e = ntri + k + tid; e < hA; e += UPD_THREADS) pst[e] = 0.f;
      for (int e = hA + ntri + k + tid; e < pstride; e += UPD_THREADS) pst[e] = 0.f;
      __syncthreads();
      for (int e = 4 * tid; e < pstride; e += 4 * UPD_THREADS)
        *reinterpret_cast<float4*>(out + e) = *reinterpret_cast<const float4*>(pst + e);
    }
  }
  dstamp(p, 9);
  grid.sync();
  stamp(p, 1);
  dstamp(p, 10);

  // ---------------- phase 2: reduce partials (compact entries) ----------------
  // a CTA owns a contiguous entry range; lanes over entries, warps over the
  // partial index; all loads of a thread issued before the adds.
  {
    const int G = gridDim.x;
    const int per = (pstride + G - 1) / G;
    const int e0 = blockIdx.x * per, e1 = min(pstride, e0 + per);
    for (int eb = e0; eb < e1; eb += 32) {
      const int e = eb + lane;
      float vals[24];
#pragma unroll
      for (int t = 0; t < 24; ++t) {
        const int b = warp + 8 * t;
        vals[t] = (e < e1 && b < G) ? p.partial[(size_t)b * pstride + e] : 0.f;
      }
      float s = 0.f;
#pragma unroll
      for (int t = 0; t < 24; ++t) s += vals[t];
      for (int b = warp + 8 * 24; b < G; b += 8) s += (e < e1) ? p.partial[(size_t)b * pstride + e] : 0.f;
      red[warp * 32 + lane] = s;
      __syncthreads();
      if (warp == 0 && e < e1) {
        float t = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) t += red[w * 32 + lane];
        p.raw[e] = t;
      }
      __syncthreads();
    }
  }
  dstamp(p, 11);
  grid.sync();
  stamp(p, 2);
  dstamp(p, 12);
  }  // !pre_reduced

  if (!coef) {
  // ---------------- phase 3a: coefficients ----------------
  // the reduced raw tables are staged into shared memory with one burst of
  // independent 16-byte async copies, then the coefficients are formed from smem.
  {
    if (!early_raw) {
      for (int e = 4 * tid; e < pstride; e += 4 * UPD_THREADS)
        cp_async16(rs + e, (p.raw_a && e < hA) ? p.raw_a + e : p.raw + e, 16);
      cp_async_commit();
    }
    cp_async_wait<0>();
    __syncthreads();
    dstamp(p, 19);
    const float* rA = rs;
    const float* rB = rs + ntri;
    const float* rC = rs + hA;
    const float* rN = rC + ntri;
    if (tid < 64) {
      const int i = tid;
      float n = 0.f, is2 = 0.f, gb = 0.f;
      if (i < k) {
        n = rsqrtf(rN[i]);
        gb = n * n * rB[i];
        const float gcii = n * rC[tri_index(i, i)];            // <v_i, [Bv]_i>
        if (p.smooth) {
          // Alg. 3 l.7: [<v,Bv>]_i = exp(log rho + (log nu - log rho) sigma(z_i))
          const float* zr = p.zbuf + ((p.zpar + step) & 1) * 64;
          const float z = zr[i];
          const float sg = 1.f / (1.f + expf(-z));
          const float br = expf(p.lnrho + (p.lnnu - p.lnrho) * sg);
          is2 = 1.f / br;
          if (blockIdx.x == 0) {   // l.14 / l.21: z_i += gamma (<v_i,[Bv]_i> - br) br (log nu - log rho) sigma (1 - sigma)
            float* zw = p.zbuf + ((p.zpar + step + 1) & 1) * 64;
            zw[i] = z + p.gamma * (gcii - br) * br * (p.lnnu - p.lnrho) * sg * (1.f - sg);
          }
        } else {
          is2 = 1.f / fmaxf(gcii, p.rho);                      // Alg. 2 l.8
        }
      }
      Ns[i] = n; IS2[i] = is2; D1s[i] = gb;
    }
    __syncthreads();
    dstamp(p, 20);
    // L_ij = G^B_ii G^A_ij / s_j^2 (j < i), transposed: Lt[j][i]; lanes over i
    for (int e = tid; e < 64 * 64; e += UPD_THREADS) {
      const int j = e >> 6, i = e & 63;
      float l = 0.f;
      if (i < k && j < i) l = D1s[i] * (Ns[i] * Ns[j] * rA[tri_index(i, j)]) * IS2[j];
      Lt[j * UPD_LTS + i] = l;
    }
    // c_i = sum_{j<i} G^A_ij G^C_ij / s_j^2 (4 threads per i), D2_i = G^A_ii - c_i
    {
      const int i = tid >> 2, q = tid & 3;
      float c = 0.f;
      if (i < k) {
        const float ni = Ns[i];
        for (int j = q; j < i; j += 4)
          c = fmaf(ni * Ns[j] * rA[tri_index(i, j)], ni * rC[tri_index(i, j)] * IS2[j], c);
      }
      c += __shfl_xor_sync(0xffffffffu, c, 1);
      c += __shfl_xor_sync(0xffffffffu, c, 2);
      if (q == 0) D2s[i] = i < k ? Ns[i] * Ns[i] * rA[tri_index(i, i)] - c : 0.f;
    }
    // the step's normalised tables (geig_get_gram), written by all CTAs in slices
    {
      const int G = gridDim.x, kk = k * k;
      const int per = (kk + G - 1) / G;
      const int e1 = min(kk, (int)(blockIdx.x + 1) * per);
      for (int e = blockIdx.x * per + tid; e < e1; e += UPD_THREADS) {
        const int i = e / k, j = e - (e / k) * k;
        const bool low = j <= i;
        const int tij = tri_index(i, low ? j : 0);
        p.gram[e] = low ? Ns[i] * Ns[j] * rA[tij] : 0.f;
        p.gram[(size_t)kk + e] = (i == j) ? D1s[i] : 0.f;
        p.gram[2 * (size_t)kk + e] = low ? Ns[i] * rC[tij] : 0.f;
      }
    }
    __syncthreads();
  }
  }  // !coef
  dstamp(p, 13);

  if (um && (PRE == 1 || (PRE < 0 && p.pre_reduced))) tc::mbar_wait(tbar, 0);   // tiles staged
  dstamp(p, 21);

  // ---------------- phase 3b: grad, v'' and [Bv]' from the resident tiles ----------------
  // 3b-1: the triangular penalty sums P_ix = sum_{j<i} L_ij [Bv]_jx (fp32
  // FMA).  Work item = (row-group pair, column quad): rows 4g..4g+3 and
  // 60-4g..63-4g (equal triangular cost per item), 4 columns; per j a float4
  // of [Bv] and two (near-broadcast) float4 of L feed 32 FMAs, j unrolled by
  // 4 so the shared loads of the next iterations overlap the FMAs.  The item
  // then forms the Alg. 2 direction
  //   grad_ix = D1_i AV_ix - D2_i BV_ix - P_ix
  // in place of the AV tile (each element owned by one thread).
  // 3b-2: v'' = n_i v + eta grad (or Adam), [Bv]' = [Bv] + gamma (n_i BV - [Bv]),
  // float4 over (row, column quad), coalesced stores.
  {
    const int nq4 = W / 4;
    for (int item = tid; item < 8 * nq4; item += UPD_THREADS) {
      const int pr = item / nq4, q = item - pr * nq4;
      const int iA = 4 * pr, iB = 60 - 4 * pr;
      // j bounds rounded up to multiples of 4 (L_ij = 0 for j >= i, the rows
      // of Ct past k are zero): 4 j per iteration with no remainder branches,
      // so the 12 shared loads of an iteration issue ahead of its 128 FMAs
      const int kr = (k + 3) & ~3;
      const int jA = min(iA + 4, kr), jB = min(iB + 4, kr);
      float accA[4][4], accB[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) accA[a][b] = accB[a][b] = 0.f;
      const float* cp = Ct + 4 * q;
      int j0 = (kDevKnobs && (p.dbg_mode & 512)) ? jB : 0;   // developer: skip the penalty sums (timing only)
#pragma unroll 1
      for (; j0 < jA; j0 += 4) {
        float4 x[4], la[4], lb[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          x[u] = *reinterpret_cast<const float4*>(cp + (j0 + u) * S);
          la[u] = *reinterpret_cast<const float4*>(Lt + (j0 + u) * UPD_LTS + iA);
          lb[u] = *reinterpret_cast<const float4*>(Lt + (j0 + u) * UPD_LTS + iB);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float xv[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
          const float lav[4] = {la[u].x, la[u].y, la[u].z, la[u].w}, lbv[4] = {lb[u].x, lb[u].y, lb[u].z, lb[u].w};
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              accA[a][b] = fmaf(lav[a], xv[b], accA[a][b]);
              accB[a][b] = fmaf(lbv[a], xv[b], accB[a][b]);
            }
        }
      }
#pragma unroll 1
      for (; j0 < jB; j0 += 4) {
        float4 x[4], lb[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          x[u] = *reinterpret_cast<const float4*>(cp + (j0 + u) * S);
          lb[u] = *reinterpret_cast<const float4*>(Lt + (j0 + u) * UPD_LTS + iB);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float xv[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
          const float lbv[4] = {lb[u].x, lb[u].y, lb[u].z, lb[u].w};
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) accB[a][b] = fmaf(lbv[a], xv[b], accB[a][b]);
        }
      }
      auto direction = [&](int i0, const float (&acc)[4][4]) {
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int i = i0 + a;
          if (i < k) {
            const float ni = Ns[i];
            const float d1 = D1s[i] * ni, d2 = D2s[i] * ni;
            float4* ap = reinterpret_cast<float4*>(At + i * S + 4 * q);
            const float4 av = *ap;
            const float4 bv = *reinterpret_cast<const float4*>(Bt + i * S + 4 * q);
            float4 gq;
            gq.x = d1 * av.x - d2 * bv.x - acc[a][0];
            gq.y = d1 * av.y - d2 * bv.y - acc[a][1];
            gq.z = d1 * av.z - d2 * bv.z - acc[a][2];
            gq.w = d1 * av.w - d2 * bv.w - acc[a][3];
            *ap = gq;
          }
        }
      };
      direction(iA, accA);
      direction(iB, accB);
    }
    __syncthreads();
    if (tid == 0) dstamp(p, 22);
    const int nq = W / 4;
    for (int e = tid; e < k * nq; e += UPD_THREADS) {
      const int i = e / nq, q = e - (e / nq) * nq;
      const int64_t gx = c0 + 4 * q;
      if (gx >= c1) continue;
      const float4 gr = *reinterpret_cast<const float4*>(At + i * S + 4 * q);   // grad (3b-1)
      const float4 bv = *reinterpret_cast<const float4*>(Bt + i * S + 4 * q);
      const float4 vv = *reinterpret_cast<const float4*>(Vt + i * S + 4 * q);
      const float4 xa = *reinterpret_cast<const float4*>(Ct + i * S + 4 * q);
      const float ni = Ns[i];
      float4 vn, an;
      if (ADAM && p.adam) {
        // Appendix H: Adam ascent on v_i with the Alg. 2 direction as the gradient
        const size_t o0 = (size_t)i * lds + gx;
        float4 m4 = *reinterpret_cast<const float4*>(p.am + o0);
        float4 s4 = *reinterpret_cast<const float4*>(p.as + o0);
        const float tt = (float)(p.adam_t0 + step + 1);
        const float cb1 = 1.f / (1.f - powf(p.b1, tt)), cb2 = 1.f / (1.f - powf(p.b2, tt));
        auto upd = [&](float gv, float& mv, float& sv, float v) {
          mv = p.b1 * mv + (1.f - p.b1) * gv;
          sv = p.b2 * sv + (1.f - p.b2) * gv * gv;
          return v + p.eta * (mv * cb1) / (sqrtf(sv * cb2) + p.eps);
        };
        vn.x = upd(gr.x, m4.x, s4.x, ni * vv.x);
        vn.y = upd(gr.y, m4.y, s4.y, ni * vv.y);
        vn.z = upd(gr.z, m4.z, s4.z, ni * vv.z);
        vn.w = upd(gr.w, m4.w, s4.w, ni * vv.w);
        if (VEC && gx + 3 < c1) {
          *reinterpret_cast<float4*>(p.am + o0) = m4;
          *reinterpret_cast<float4*>(p.as + o0) = s4;
        } else {
          const float ms[4] = {m4.x, m4.y, m4.z, m4.w}, ss[4] = {s4.x, s4.y, s4.z, s4.w};
          for (int tq = 0; tq < 4; ++tq)
            if (gx + tq < c1) { p.am[o0 + tq] = ms[tq]; p.as[o0 + tq] = ss[tq]; }
        }
      } else {
        vn.x = ni * vv.x + p.eta * gr.x;
        vn.y = ni * vv.y + p.eta * gr.y;
        vn.z = ni * vv.z + p.eta * gr.z;
        vn.w = ni * vv.w + p.eta * gr.w;
      }
      if (kDevKnobs && p.dbg && !isfinite(vn.x + vn.y + vn.z + vn.w))
        atomicCAS(&p.dbg[(size_t)gridDim.x * 64 + (size_t)blockIdx.x * 8 + 3], 0ull, (unsigned long long)(step + 1));
      if (kDevKnobs && p.dbg && !isfinite(gr.x + gr.y + gr.z + gr.w))
        atomicCAS(&p.dbg[(size_t)gridDim.x * 64 + (size_t)blockIdx.x * 8 + 4], 0ull, (unsigned long long)(step + 1));
      if (kDevKnobs && p.dbg && !isfinite(bv.x + bv.y + bv.z + bv.w + vv.x + vv.y + vv.z + vv.w))
        atomicCAS(&p.dbg[(size_t)gridDim.x * 64 + (size_t)blockIdx.x * 8 + 5], 0ull, (unsigned long long)(step + 1));
      an.x = xa.x + p.gamma * (ni * bv.x - xa.x);
      an.y = xa.y + p.gamma * (ni * bv.y - xa.y);
      an.z = xa.z + p.gamma * (ni * bv.z - xa.z);
      an.w = xa.w + p.gamma * (ni * bv.w - xa.w);
      const size_t o = (size_t)i * lds + gx;
      const size_t ob = (size_t)i * bld + gx;
      if (kDevKnobs && (p.dbg_mode & 256)) {   // developer: no state write-back (timing only)
        if (vn.x == 12345.f && an.x == 12345.f) p.V[o] = 0.f;
      } else if (VEC && gx + 3 < c1) {
        *reinterpret_cast<float4*>(p.V + o) = vn;
        *reinterpret_cast<float4*>(p.AUX + o) = an;
        if (p.Vbf) store_vbf4(p.Vbf, blo, ob, vn);
        for (int q = 0; q < p.vpeer_n; ++q)   // peer exchange: the block into every peer's gathered shadow
          store_vbf4(p.vpeer[q], blo, ob, vn);
      } else {
        const float vs[4] = {vn.x, vn.y, vn.z, vn.w}, as[4] = {an.x, an.y, an.z, an.w};
        for (int tq = 0; tq < 4; ++tq)
          if (gx + tq < c1) {
            p.V[o + tq] = vs[tq];
            p.AUX[o + tq] = as[tq];
            if (p.Vbf) store_vbf1(p.Vbf, blo, ob + tq, vs[tq]);
            for (int q = 0; q < p.vpeer_n; ++q) store_vbf1(p.vpeer[q], blo, ob + tq, vs[tq]);
          }
      }
    }
  }
  stamp(p, 3);
  dstamp(p, 14);
}

template <bool VEC>
__global__ void __launch_bounds__(UPD_THREADS, 1)
update_res_kernel(UpdateArgs p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) float smem[];
  update_res_phases<VEC>(p, smem, grid);
}

// geig_get: the stored state is v'' = v + eta grad (the retraction is folded
// into the next update); return the retracted v = v'' / ||v''|| (one CTA per row).
__global__ void __launch_bounds__(256)
normalize_rows_kernel(const float* __restrict__ Vin, float* __restrict__ Vout, int64_t d) {
  __shared__ float red[8];
  const int i = blockIdx.x;
  float s = 0.f;
  for (int64_t x = threadIdx.x; x < d; x += blockDim.x) {
    const float v = Vin[(int64_t)i * d + x];
    s = fmaf(v, v, s);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = rsqrtf(t);
  }
  __syncthreads();
  const float inv = red[0];
  for (int64_t x = threadIdx.x; x < d; x += blockDim.x) Vout[(int64_t)i * d + x] = Vin[(int64_t)i * d + x] * inv;
}

// Alg. 2 lines 2-3: v_i = g_i / ||g_i||, [Bv]_i = v_i.  One CTA per player.
__global__ void __launch_bounds__(256)
init_state_kernel(const float* __restrict__ G, float* V, float* AUX, __nv_bfloat16* Vbf, int64_t d) {
  __shared__ float red[8];
  const int i = blockIdx.x;
  float s = 0.f;
  for (int64_t x = threadIdx.x; x < d; x += blockDim.x) {
    const float g = G[(int64_t)i * d + x];
    s = fmaf(g, g, s);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = rsqrtf(t);
  }
  __syncthreads();
  const float inv = red[0];
  for (int64_t x = threadIdx.x; x < d; x += blockDim.x) {
    const float v = G[(int64_t)i * d + x] * inv;
    V[(int64_t)i * d + x] = v;
    AUX[(int64_t)i * d + x] = v;
    if (Vbf) store_vbf1(Vbf, (int64_t)gridDim.x * d, (size_t)i * d + x, v);
  }
}

// hi/lo bf16 shadow of an fp32 array (dst holds 2 x n: hi plane, lo plane)
__global__ void f32_to_bf16_kernel(const float* __restrict__ src, __nv_bfloat16* dst, int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    store_vbf1(dst, n, (size_t)e, src[e]);
}

}  // namespace geig
