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
// Phases (grid.sync between them), 256 threads per CTA:
//  1  Gram partials over column segments: 64x64 (i,j) blocks of table A or C
//     (lower blocks only) as 4x4 register micro-tiles per thread fed by
//     float4 shared-memory loads; table B's diagonal as warp dot products.
//  2a deterministic reduction of the partials over segments -> gram.
//  2b coefficients L, D1 = G^B_ii, D2 = G^A_ii - c_i (one warp per row).
//  3  per 64-column chunk: L [Bv] as 4x4 micro-tiles, grad, v', [Bv]'
//     (in place), partial ||v'||^2.
//  4  reduce norms, V = v'/||v'|| (+ bf16 copy of V for the GEMMs).
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"

namespace geig {

namespace cg = cooperative_groups;

constexpr int UPD_THREADS = 256;
constexpr int UPD_CW = 64;       // columns per update chunk
constexpr int UPD_SUB = 32;      // columns per shared-memory sub-chunk of a Gram unit
constexpr int UPD_LD = 68;       // padded row (64 + 4) of the transposed tiles

struct UpdateArgs {
  float* V;              // k x d (in/out)
  float* AUX;            // k x d (in/out)
  const float* AV;       // k x d
  const float* BV;       // k x d
  float* Vtmp;           // k x d scratch (v')
  __nv_bfloat16* Vbf;    // k x d bf16 copy of the new V (nullable)
  float* partial;        // nseg x units x 4096 scratch
  float* gram;           // 3 x k x k out: GA, GB, GC
  float* coef;           // k x k (L) + k (D1) + k (D2)
  float* norm_partial;   // gridDim x k
  int k;
  int64_t d;
  int segw;              // columns per Gram segment (multiple of UPD_SUB)
  float eta, gamma, rho;
};

__host__ __device__ inline int upd_nb(int k) { return (k + 63) / 64; }
__host__ __device__ inline int upd_units_per_seg(int k) {
  const int nb = upd_nb(k);
  return nb * (nb + 1) + 1;   // 2 tables x lower block pairs + 1 GB-diagonal unit
}

// unit u of a segment -> (table 0=A / 2=C / 1=B-diag, block row bi, block col bj)
__device__ __forceinline__ void upd_decode(int u, int nb, int& table, int& bi, int& bj) {
  const int pairs = nb * (nb + 1) / 2;
  if (u == 2 * pairs) { table = 1; bi = bj = 0; return; }
  table = u < pairs ? 0 : 2;
  int r = u < pairs ? u : u - pairs;
  int i = 0;
  while (r >= i + 1) { r -= i + 1; ++i; }
  bi = i; bj = r;
}

template <bool VEC>
__device__ __forceinline__ float4 ld4(const float* p, int64_t x, int64_t d) {
  if (VEC && x + 3 < d) return *reinterpret_cast<const float4*>(p + x);
  float4 r;
  r.x = x < d ? p[x] : 0.f;
  r.y = x + 1 < d ? p[x + 1] : 0.f;
  r.z = x + 2 < d ? p[x + 2] : 0.f;
  r.w = x + 3 < d ? p[x + 3] : 0.f;
  return r;
}
template <bool VEC>
__device__ __forceinline__ void st4(float* p, int64_t x, int64_t d, float4 v) {
  if (VEC && x + 3 < d) { *reinterpret_cast<float4*>(p + x) = v; return; }
  if (x < d) p[x] = v.x;
  if (x + 1 < d) p[x + 1] = v.y;
  if (x + 2 < d) p[x + 2] = v.z;
  if (x + 3 < d) p[x + 3] = v.w;
}

template <bool VEC>
__global__ void __launch_bounds__(UPD_THREADS)
update_kernel(UpdateArgs p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) float smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int k = p.k;
  const int64_t d = p.d;
  const int nb = upd_nb(k);
  const int ups = upd_units_per_seg(k);
  const int nseg = (int)((d + p.segw - 1) / p.segw);

  // ---------------- phase 1: Gram partial sums ----------------
  {
    float* Vs = smem;                       // [UPD_SUB][UPD_LD]  (x-major: Vs[x][i])
    float* Ps = smem + UPD_SUB * UPD_LD;    // [UPD_SUB][UPD_LD]
    const int ti = tid & 15, tj = tid >> 4; // micro-tile rows 4ti.., cols 4tj..
    for (int w = blockIdx.x; w < ups * nseg; w += gridDim.x) {
      const int seg = w / ups, u = w % ups;
      int table, bi, bj;
      upd_decode(u, nb, table, bi, bj);
      const int64_t c0 = (int64_t)seg * p.segw;
      const int64_t c1 = min((int64_t)d, c0 + p.segw);
      float* out = p.partial + ((int64_t)seg * ups + u) * 4096;
      if (table == 1) {
        // diagonal of G^B: one warp per player row, lanes over columns
        for (int i = warp; i < k; i += UPD_THREADS / 32) {
          float s = 0.f;
          for (int64_t x = c0 + lane; x < c1; x += 32)
            s = fmaf(p.V[(int64_t)i * d + x], p.BV[(int64_t)i * d + x], s);
          s = warp_sum(s);
          if (lane == 0) out[i] = s;
        }
        continue;
      }
      const float* P = table == 0 ? p.AV : p.AUX;
      const int i0 = bi * 64, j0 = bj * 64;
      const bool active = !(bi == bj && ti < tj);   // micro-tile strictly above the diagonal
      float acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
      for (int64_t x0 = c0; x0 < c1; x0 += UPD_SUB) {
        for (int e = tid; e < 64 * UPD_SUB; e += UPD_THREADS) {
          const int r = e / UPD_SUB, x = e % UPD_SUB;
          const int64_t gx = x0 + x;
          const bool inx = gx < c1;
          Vs[x * UPD_LD + r] = (inx && i0 + r < k) ? p.V[(int64_t)(i0 + r) * d + gx] : 0.f;
          Ps[x * UPD_LD + r] = (inx && j0 + r < k) ? P[(int64_t)(j0 + r) * d + gx] : 0.f;
        }
        __syncthreads();
        if (active) {
#pragma unroll 8
          for (int x = 0; x < UPD_SUB; ++x) {
            const float4 a = *reinterpret_cast<const float4*>(Vs + x * UPD_LD + 4 * ti);
            const float4 b = *reinterpret_cast<const float4*>(Ps + x * UPD_LD + 4 * tj);
            const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int ii = 0; ii < 4; ++ii)
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) acc[ii][jj] = fmaf(av[ii], bv[jj], acc[ii][jj]);
          }
        }
        __syncthreads();
      }
#pragma unroll
      for (int ii = 0; ii < 4; ++ii)
        *reinterpret_cast<float4*>(out + (4 * ti + ii) * 64 + 4 * tj) =
            make_float4(acc[ii][0], acc[ii][1], acc[ii][2], acc[ii][3]);
    }
  }
  grid.sync();

  // ---------------- phase 2a: reduce partials -> gram ----------------
  // 32 consecutive entries per CTA iteration (lanes), the 8 warps split the
  // segments, fixed-order combine through shared memory (deterministic).
  {
    float* red = smem;                       // [8][32]
    const int pairs = nb * (nb + 1) / 2;
    const int64_t per_table = (int64_t)pairs * 4096;
    const int64_t total = 2 * per_table + k;
    const int64_t ngroups = (total + 31) / 32;
    for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
      const int64_t e = grp * 32 + lane;
      int u = 0, q = 0;
      const bool ok = e < total;
      if (ok) {
        if (e < 2 * per_table) { u = (int)(e / 4096); q = (int)(e % 4096); }
        else { u = 2 * pairs; q = (int)(e - 2 * per_table); }
      }
      float s0 = 0.f, s1 = 0.f;
      if (ok) {
        const float* src = p.partial + (int64_t)u * 4096 + q;
        const int64_t stride = (int64_t)ups * 4096;
        int sg = warp;
        for (; sg + 8 < nseg; sg += 16) {
          s0 += src[(int64_t)sg * stride];
          s1 += src[(int64_t)(sg + 8) * stride];
        }
        if (sg < nseg) s0 += src[(int64_t)sg * stride];
      }
      red[warp * 32 + lane] = s0 + s1;
      __syncthreads();
      if (warp == 0 && ok) {
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) s += red[w * 32 + lane];
        int table, bi, bj;
        upd_decode(u, nb, table, bi, bj);
        int i, j;
        if (table == 1) { i = j = q; }
        else { i = bi * 64 + q / 64; j = bj * 64 + q % 64; }
        if (i < k && j < k && (table == 1 || i >= j))
          p.gram[(int64_t)table * k * k + (int64_t)i * k + j] = s;
      }
      __syncthreads();
    }
  }
  grid.sync();

  // ---------------- phase 2b: coefficients ----------------
  {
    const float* GA = p.gram;
    const float* GB = p.gram + (int64_t)k * k;
    const float* GC = p.gram + 2 * (int64_t)k * k;
    const int nwarps = gridDim.x * (UPD_THREADS / 32);
    for (int i = blockIdx.x * (UPD_THREADS / 32) + warp; i < k; i += nwarps) {
      const float gbii = GB[(int64_t)i * k + i];
      float c = 0.f;
      for (int j = lane; j < k; j += 32) {
        float l = 0.f;
        if (j < i) {
          const float s2 = fmaxf(GC[(int64_t)j * k + j], p.rho);
          const float ga = GA[(int64_t)i * k + j];
          l = gbii * ga / s2;
          c = fmaf(ga, GC[(int64_t)i * k + j] / s2, c);
        }
        p.coef[(int64_t)j * k + i] = l;       // stored transposed: Lt[j][i]
      }
      c = warp_sum(c);
      if (lane == 0) {
        p.coef[(int64_t)k * k + i] = gbii;                              // D1
        p.coef[(int64_t)k * k + k + i] = GA[(int64_t)i * k + i] - c;    // D2
      }
    }
  }
  grid.sync();

  // ---------------- phase 3: grad, v', aux' ----------------
  const int kp = (k + 3) & ~3;                    // rows padded to a float4
  float* Ns = smem;                               // kp (norm partial)
  float* red4 = Ns + kp;                          // 256 (phase-4 reduction scratch)
  float* Lt = red4 + 256;                         // k x kp  (Lt[j][i])
  float* Xs = Lt + (size_t)k * kp;                // k x UPD_CW (AUX chunk)
  float* D1s = Xs + (size_t)k * UPD_CW;           // k
  float* D2s = D1s + kp;                          // k
  for (int e = tid; e < k * kp; e += UPD_THREADS) {
    const int j = e / kp, i = e % kp;
    Lt[e] = i < k ? p.coef[(int64_t)j * k + i] : 0.f;
  }
  for (int e = tid; e < k; e += UPD_THREADS) {
    D1s[e] = p.coef[(int64_t)k * k + e];
    D2s[e] = p.coef[(int64_t)k * k + k + e];
    Ns[e] = 0.f;
  }
  __syncthreads();
  const int nchunk = (int)((d + UPD_CW - 1) / UPD_CW);
  const int tx = tid & 15;          // 4 columns 4tx..4tx+3
  const int tr = tid >> 4;          // 4 rows per pass: 4(tr + 16 pass)..
  const int nrb = (k + 3) / 4;      // row blocks of 4
  for (int ch = blockIdx.x; ch < nchunk; ch += gridDim.x) {
    const int64_t cx = (int64_t)ch * UPD_CW;
    for (int e = tid; e < k * (UPD_CW / 4); e += UPD_THREADS) {
      const int r = e / (UPD_CW / 4), q = e % (UPD_CW / 4);
      const float4 v = ld4<VEC>(p.AUX + (int64_t)r * d, cx + 4 * q, d);
      *reinterpret_cast<float4*>(Xs + r * UPD_CW + 4 * q) = v;
    }
    __syncthreads();
    const int64_t gx = cx + 4 * tx;
    for (int rb0 = 0; rb0 < nrb; rb0 += 16) {
      const int rb = rb0 + tr;               // every lane iterates (full-warp shuffles below)
      const int i0 = 4 * rb;
      float acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
      const int jmax = rb < nrb ? min(i0 + 3, k) : 0;   // L_ij = 0 for j >= i
      for (int j = 0; j < jmax; ++j) {
        const float4 l = *reinterpret_cast<const float4*>(Lt + (size_t)j * kp + i0);
        const float4 x = *reinterpret_cast<const float4*>(Xs + j * UPD_CW + 4 * tx);
        const float lv[4] = {l.x, l.y, l.z, l.w}, xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(lv[a], xv[b], acc[a][b]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int i = i0 + a;
        float sq = 0.f;
        if (i < k && gx < d) {
          const int64_t o = (int64_t)i * d;
          const float4 av = ld4<VEC>(p.AV + o, gx, d);
          const float4 bv = ld4<VEC>(p.BV + o, gx, d);
          const float4 vv = ld4<VEC>(p.V + o, gx, d);
          const float4 xa = *reinterpret_cast<const float4*>(Xs + i * UPD_CW + 4 * tx);
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
          // zero the padding lanes of a ragged tail before squaring
          if (!(gx + 1 < d)) vn.y = 0.f;
          if (!(gx + 2 < d)) vn.z = 0.f;
          if (!(gx + 3 < d)) vn.w = 0.f;
          st4<VEC>(p.Vtmp + o, gx, d, vn);
          st4<VEC>(p.AUX + o, gx, d, an);
          sq = vn.x * vn.x + vn.y * vn.y + vn.z * vn.z + vn.w * vn.w;
        }
        // reduce over the 16 threads (tx) sharing row i (a half warp)
        sq += __shfl_xor_sync(0xffffffffu, sq, 1);
        sq += __shfl_xor_sync(0xffffffffu, sq, 2);
        sq += __shfl_xor_sync(0xffffffffu, sq, 4);
        sq += __shfl_xor_sync(0xffffffffu, sq, 8);
        if (tx == 0 && i < k) Ns[i] += sq;
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < k; e += UPD_THREADS) p.norm_partial[(int64_t)blockIdx.x * k + e] = Ns[e];
  grid.sync();

  // ---------------- phase 4: retraction v <- v'/||v'|| ----------------
  // every CTA reduces the per-CTA norm partials: lanes over rows i, warps
  // over the partial index, fixed-order combine (deterministic).
  {
    float* red = red4;                        // [8][32]
    for (int i0 = 0; i0 < k; i0 += 32) {
      const int i = i0 + lane;
      float s0 = 0.f, s1 = 0.f;
      if (i < k) {
        int b = warp;
        for (; b + 8 < (int)gridDim.x; b += 16) {
          s0 += p.norm_partial[(int64_t)b * k + i];
          s1 += p.norm_partial[(int64_t)(b + 8) * k + i];
        }
        if (b < (int)gridDim.x) s0 += p.norm_partial[(int64_t)b * k + i];
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
  }
  for (int ch = blockIdx.x; ch < nchunk; ch += gridDim.x) {
    const int64_t cx = (int64_t)ch * UPD_CW;
    for (int e = tid; e < k * (UPD_CW / 4); e += UPD_THREADS) {
      const int r = e / (UPD_CW / 4), q = e % (UPD_CW / 4);
      const int64_t gx = cx + 4 * q;
      if (gx >= d) continue;
      const int64_t o = (int64_t)r * d;
      float4 v = ld4<VEC>(p.Vtmp + o, gx, d);
      const float sc = Ns[r];
      v.x *= sc; v.y *= sc; v.z *= sc; v.w *= sc;
      st4<VEC>(p.V + o, gx, d, v);
      if (p.Vbf) {
        __nv_bfloat16* q2 = p.Vbf + o + gx;
        if (VEC && gx + 3 < d) {
          __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
          uint2 pk;
          pk.x = *reinterpret_cast<uint32_t*>(&lo);
          pk.y = *reinterpret_cast<uint32_t*>(&hi);
          *reinterpret_cast<uint2*>(q2) = pk;
        } else {
          const float vs[4] = {v.x, v.y, v.z, v.w};
          for (int t = 0; t < 4 && gx + t < d; ++t) q2[t] = __float2bfloat16_rn(vs[t]);
        }
      }
    }
  }
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
