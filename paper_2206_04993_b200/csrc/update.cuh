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
// One CTA (256 threads) per SM owns a contiguous column range of d; the
// four k x range tiles (V, AV, [Bv], BV) stream through shared memory in
// 32-column sub-chunks with double-buffered cp.async (16-byte, zero-fill
// past the range).  Phases (grid.sync between them):
//  1  per-CTA Gram partials: G^A, G^C as 4x4 register micro-tiles per
//     thread (rows t, t+16, t+32, t+48 of each 64-row block: conflict-free
//     LDS.128 with a 36-float row stride), lower 64-blocks only; diag G^B.
//  2a deterministic reduction of the per-CTA partials -> gram.
//  2b coefficients L (stored transposed), D1 = G^B_ii, D2 = G^A_ii - c_i.
//  3  stream the tiles again: L [Bv] micro-tiles, grad, v' (to scratch),
//     [Bv]' (to the state), per-CTA ||v'||^2 partials.
//  4  reduce the norms, V = v'/||v'|| (+ bf16 copy of V for the GEMMs).
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"

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
  float* Vtmp;           // k x d scratch (v')
  __nv_bfloat16* Vbf;    // k x d bf16 copy of the new V (nullable)
  float* partial;        // gridDim x (2*KP*KP + KP) scratch
  float* gram;           // 3 x k x k out: GA, GB, GC (zeroed by the host)
  float* coef;           // k x k (Lt, transposed L) + k (D1) + k (D2)
  float* norm_partial;   // gridDim x k
  int k;
  int64_t d;
  int64_t segw;          // columns per CTA (multiple of 4)
  float eta, gamma, rho;
  unsigned long long* ts;  // 6 %globaltimer stamps of CTA 0 (phase boundaries), nullable
};

__device__ __forceinline__ void stamp(const UpdateArgs& p, int slot) {
  if (p.ts && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.ts[slot] = t;
  }
}

__host__ __device__ constexpr size_t upd_smem_floats(int NB) {
  // phase 1/3 double buffer of 4 tiles + phase-3 Lt + D1 + D2 + Ns + red
  return (size_t)2 * 4 * (NB * 64) * UPD_S + (size_t)(NB * 64) * (NB * 64) + 3 * (NB * 64) + 256;
}

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
__device__ __forceinline__ void stage_tiles(float* tiles, const float* const* src, int k, int64_t d, int64_t x0,
                                            int64_t xend) {
  if (VEC) {
    constexpr int Q = UPD_XC / 4;                 // float4 per row
    for (int e = threadIdx.x; e < 4 * KP * Q; e += UPD_THREADS) {
      const int a = e / (KP * Q), rem = e % (KP * Q), r = rem / Q, q = rem % Q;
      const int64_t gx = x0 + 4 * q;
      const bool ok = r < k && gx < xend;
      const float* s = ok ? src[a] + (int64_t)r * d + gx : src[a];
      cp_async16(tiles + ((size_t)a * KP + r) * UPD_S + 4 * q, s, ok ? 16 : 0);
    }
  } else {
    for (int e = threadIdx.x; e < 4 * KP * UPD_XC; e += UPD_THREADS) {
      const int a = e / (KP * UPD_XC), rem = e % (KP * UPD_XC), r = rem / UPD_XC, x = rem % UPD_XC;
      const int64_t gx = x0 + x;
      const bool ok = r < k && gx < xend;
      const float* s = ok ? src[a] + (int64_t)r * d + gx : src[a];
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
  const float* src[4] = {p.V, p.AV, p.AUX, p.BV};   // tile order: 0 V, 1 AV, 2 AUX, 3 BV
  stamp(p, 0);

  // ---------------- phase 1: Gram partial sums of this CTA's columns ----------------
  {
    const int ti = tid & 15, tj = tid >> 4;
    float accA[NPAIR][4][4], accC[NPAIR][4][4];
#pragma unroll
    for (int pr = 0; pr < NPAIR; ++pr)
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) accA[pr][a][b] = accC[pr][a][b] = 0.f;
    float gb[KP / 8];
#pragma unroll
    for (int q = 0; q < KP / 8; ++q) gb[q] = 0.f;

    if (nsub > 0) { stage_tiles<KP, VEC>(buf0, src, k, d, c0, c1); }
    cp_async_commit();
    for (int sc = 0; sc < nsub; ++sc) {
      float* cur = (sc & 1) ? buf1 : buf0;
      float* nxt = (sc & 1) ? buf0 : buf1;
      if (sc + 1 < nsub) stage_tiles<KP, VEC>(nxt, src, k, d, c0 + (int64_t)(sc + 1) * UPD_XC, c1);
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
      // diagonal of G^B: warp w owns rows w + 8q, lanes over the 32 columns
#pragma unroll
      for (int q = 0; q < KP / 8; ++q) {
        const int i = warp + 8 * q;
        gb[q] = fmaf(Vt[i * UPD_S + lane], Bt[i * UPD_S + lane], gb[q]);
      }
      __syncthreads();
    }
    cp_async_wait<0>();
    // write this CTA's partials: [2][KP][KP] (A, C) + [KP] (GB diag)
    float* out = p.partial + (size_t)blockIdx.x * (2 * KP * KP + KP);
    {
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
              out[i * KP + j] = accA[pr][a][b];
              out[KP * KP + i * KP + j] = accC[pr][a][b];
            }
    }
#pragma unroll
    for (int q = 0; q < KP / 8; ++q) {
      const float s = warp_sum(gb[q]);
      if (lane == 0) out[2 * KP * KP + warp + 8 * q] = s;
    }
  }
  grid.sync();
  stamp(p, 1);

  // ---------------- phase 2a: reduce the per-CTA partials -> gram ----------------
  {
    float* red = smem;                            // [8][32]
    const int pstride = 2 * KP * KP + KP;
    const int total = pstride;
    const int ngroups = (total + 31) / 32;
    const int G = gridDim.x;
    for (int grp = blockIdx.x; grp < ngroups; grp += G) {
      const int e = grp * 32 + lane;
      int table = 0, i = 0, j = 0;
      bool ok = e < total;
      if (ok) {
        if (e < 2 * KP * KP) { table = e < KP * KP ? 0 : 2; const int q = e % (KP * KP); i = q / KP; j = q % KP; }
        else { table = 1; i = j = e - 2 * KP * KP; }
        ok = i < k && j < k && i >= j;
      }
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
      if (ok) {
        const float* srcp = p.partial + e;
        int b = warp;
        for (; b + 24 < G; b += 32) {
          s0 += srcp[(size_t)b * pstride];
          s1 += srcp[(size_t)(b + 8) * pstride];
          s2 += srcp[(size_t)(b + 16) * pstride];
          s3 += srcp[(size_t)(b + 24) * pstride];
        }
        for (; b < G; b += 8) s0 += srcp[(size_t)b * pstride];
      }
      red[warp * 32 + lane] = (s0 + s1) + (s2 + s3);
      __syncthreads();
      if (warp == 0 && ok) {
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) s += red[w * 32 + lane];
        p.gram[(size_t)table * k * k + (size_t)i * k + j] = s;
      }
      __syncthreads();
    }
  }
  grid.sync();
  stamp(p, 2);

  // ---------------- phase 2b: coefficients ----------------
  {
    const float* GA = p.gram;
    const float* GB = p.gram + (size_t)k * k;
    const float* GC = p.gram + 2 * (size_t)k * k;
    const int nwarps = gridDim.x * (UPD_THREADS / 32);
    for (int i = blockIdx.x * (UPD_THREADS / 32) + warp; i < k; i += nwarps) {
      const float gbii = GB[(size_t)i * k + i];
      float c = 0.f;
      for (int j = lane; j < k; j += 32) {
        float l = 0.f;
        if (j < i) {
          const float s2 = fmaxf(GC[(size_t)j * k + j], p.rho);
          const float ga = GA[(size_t)i * k + j];
          l = gbii * ga / s2;
          c = fmaf(ga, GC[(size_t)i * k + j] / s2, c);
        }
        p.coef[(size_t)j * k + i] = l;       // Lt[j][i]
      }
      c = warp_sum(c);
      if (lane == 0) {
        p.coef[(size_t)k * k + i] = gbii;                              // D1
        p.coef[(size_t)k * k + k + i] = GA[(size_t)i * k + i] - c;     // D2
      }
    }
  }
  grid.sync();
  stamp(p, 3);

  // ---------------- phase 3: grad, v', aux' ----------------
  float* Lt = smem + 8 * TILE;                   // [KP][KP]  Lt[j][i]
  float* D1s = Lt + KP * KP;
  float* D2s = D1s + KP;
  float* Ns = D2s + KP;
  float* red = Ns + KP;                          // [8][32]
  for (int e = tid; e < KP * KP; e += UPD_THREADS) {
    const int j = e / KP, i = e % KP;
    Lt[e] = (i < k && j < k) ? p.coef[(size_t)j * k + i] : 0.f;
  }
  for (int e = tid; e < KP; e += UPD_THREADS) {
    D1s[e] = e < k ? p.coef[(size_t)k * k + e] : 0.f;
    D2s[e] = e < k ? p.coef[(size_t)k * k + k + e] : 0.f;
    Ns[e] = 0.f;
  }
  __syncthreads();
  {
    const int tx = tid & 7;            // columns 4tx..4tx+3 of the sub-chunk
    const int tr = tid >> 3;           // rows 4tr..4tr+3
    const int i0 = 4 * tr;
    if (nsub > 0) stage_tiles<KP, VEC>(buf0, src, k, d, c0, c1);
    cp_async_commit();
    for (int sc = 0; sc < nsub; ++sc) {
      float* cur = (sc & 1) ? buf1 : buf0;
      float* nxt = (sc & 1) ? buf0 : buf1;
      if (sc + 1 < nsub) stage_tiles<KP, VEC>(nxt, src, k, d, c0 + (int64_t)(sc + 1) * UPD_XC, c1);
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
      if (i0 < KP) {
        const int jmax = min(i0 + 3, k);         // L_ij = 0 for j >= i
        for (int j = 0; j < jmax; ++j) {
          const float4 l = *reinterpret_cast<const float4*>(Lt + j * KP + i0);
          const float4 x = *reinterpret_cast<const float4*>(Ct + j * UPD_S + 4 * tx);
          const float lv[4] = {l.x, l.y, l.z, l.w}, xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(lv[a], xv[b], acc[a][b]);
        }
      }
      const int64_t gx = c0 + (int64_t)sc * UPD_XC + 4 * tx;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int i = i0 + a;
        float sq = 0.f;
        if (i < k && gx < c1) {
          const float4 av = *reinterpret_cast<const float4*>(At + i * UPD_S + 4 * tx);
          const float4 bv = *reinterpret_cast<const float4*>(Bt + i * UPD_S + 4 * tx);
          const float4 vv = *reinterpret_cast<const float4*>(Vt + i * UPD_S + 4 * tx);
          const float4 xa = *reinterpret_cast<const float4*>(Ct + i * UPD_S + 4 * tx);
          const float d1 = D1s[i], d2 = D2s[i];
          float4 vn, an;
          vn.x = vv.x + p.eta * (d1 * av.x - d2 * bv.x - acc[a][0]);
          vn.y = vv.y + p.eta * (d1 * av.y - d2 * bv.y - acc[a][1]);
          vn.z = vv.z + p.eta * (d1 * av.z - d2 * bv.z - acc[a][2]);
          vn.w = vv.w + p.eta * (d1 * av.w - d2 * bv.w - acc[a][3]);
          an.x = xa.x + p.gamma * (bv.x - xa.x);
          an.y = xa.y + p.gamma * (bv.y - xa.y);
          an.z = xa.z + p.gamma * (bv.z - xa.z);
          an.w = xa.w + p.gamma * (bv.w - xa.w);
          const size_t o = (size_t)i * d;
          if (VEC && gx + 3 < c1) {
            *reinterpret_cast<float4*>(p.Vtmp + o + gx) = vn;
            *reinterpret_cast<float4*>(p.AUX + o + gx) = an;
          } else {
            const float vs[4] = {vn.x, vn.y, vn.z, vn.w}, as[4] = {an.x, an.y, an.z, an.w};
            for (int t = 0; t < 4; ++t)
              if (gx + t < c1) { p.Vtmp[o + gx + t] = vs[t]; p.AUX[o + gx + t] = as[t]; }
          }
          // zero-filled columns past the range give vn = 0 automatically
          sq = vn.x * vn.x + vn.y * vn.y + vn.z * vn.z + vn.w * vn.w;
        }
        sq += __shfl_xor_sync(0xffffffffu, sq, 1);
        sq += __shfl_xor_sync(0xffffffffu, sq, 2);
        sq += __shfl_xor_sync(0xffffffffu, sq, 4);
        if (tx == 0 && i < k) Ns[i] += sq;
      }
      __syncthreads();
    }
    cp_async_wait<0>();
  }
  for (int e = tid; e < k; e += UPD_THREADS) p.norm_partial[(size_t)blockIdx.x * k + e] = Ns[e];
  grid.sync();
  stamp(p, 4);

  // ---------------- phase 4: retraction v <- v'/||v'|| ----------------
  for (int r0 = 0; r0 < k; r0 += 32) {
    const int i = r0 + lane;
    float s0 = 0.f, s1 = 0.f;
    if (i < k) {
      int b = warp;
      for (; b + 8 < (int)gridDim.x; b += 16) {
        s0 += p.norm_partial[(size_t)b * k + i];
        s1 += p.norm_partial[(size_t)(b + 8) * k + i];
      }
      if (b < (int)gridDim.x) s0 += p.norm_partial[(size_t)b * k + i];
    }
    red[warp * 32 + lane] = s0 + s1;
    __syncthreads();
    if (warp == 0 && i < k) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) s += red[w * 32 + lane];
      Ns[i] = rsqrtf(s);
    }
    __syncthreads();
  }
  if (c1 > c0) {
    const int64_t w = c1 - c0;
    if (VEC) {
      const int64_t nq = w / 4;
      for (int64_t e = tid; e < (int64_t)k * nq; e += UPD_THREADS) {
        const int r = (int)(e / nq);
        const int64_t gx = c0 + 4 * (e % nq);
        const size_t o = (size_t)r * d + gx;
        float4 v = *reinterpret_cast<const float4*>(p.Vtmp + o);
        const float sc = Ns[r];
        v.x *= sc; v.y *= sc; v.z *= sc; v.w *= sc;
        *reinterpret_cast<float4*>(p.V + o) = v;
        if (p.Vbf) {
          __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
          uint2 pk;
          pk.x = *reinterpret_cast<uint32_t*>(&lo);
          pk.y = *reinterpret_cast<uint32_t*>(&hi);
          *reinterpret_cast<uint2*>(p.Vbf + o) = pk;
        }
      }
    } else {
      for (int64_t e = tid; e < (int64_t)k * w; e += UPD_THREADS) {
        const int r = (int)(e / w);
        const size_t o = (size_t)r * d + c0 + (e % w);
        const float v = p.Vtmp[o] * Ns[r];
        p.V[o] = v;
        if (p.Vbf) p.Vbf[o] = __float2bfloat16_rn(v);
      }
    }
  }
  stamp(p, 5);
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
    if (Vbf) Vbf[(int64_t)i * d + x] = __float2bfloat16_rn(v);
  }
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ src, __nv_bfloat16* dst, int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = __float2bfloat16_rn(src[e]);
}

}  // namespace geig
