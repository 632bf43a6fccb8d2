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
// Phases (grid.sync between them):
//  1  Gram partials: work units = (32x32 pair tile of table A/C [lower
//     tiles] or B [diagonal tiles]) x (segment of SEG columns of d).
//  2a deterministic reduction of the partials over segments -> gram.
//  2b coefficients L, D1 = G^B_ii, D2 = G^A_ii - c_i (one warp per row).
//  3  per column chunk: grad, v', [Bv]' (in place), partial ||v'||^2.
//  4  reduce norms, V = v'/||v'|| (+ optional bf16 copy of V for the GEMMs).
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"

namespace geig {

namespace cg = cooperative_groups;

constexpr int UPD_THREADS = 256;
constexpr int UPD_SEG = 256;     // columns per Gram work unit
constexpr int UPD_CW = 32;       // columns per update chunk

struct UpdateArgs {
  float* V;              // k x d (in/out)
  float* AUX;            // k x d (in/out)
  const float* AV;       // k x d
  const float* BV;       // k x d
  float* Vtmp;           // k x d scratch (v')
  __nv_bfloat16* Vbf;    // k x d bf16 copy of the new V (nullable)
  float* partial;        // nseg x units x 1024 scratch
  float* gram;           // 3 x k x k out: GA, GB, GC (zeroed by the host)
  float* coef;           // k x k (L) + k (D1) + k (D2)
  float* norm_partial;   // gridDim x k
  int k;
  int64_t d;
  float eta, gamma, rho;
};

__device__ __forceinline__ void unit_decode(int u, int T, int& table, int& ti, int& tj) {
  // units 0..nlt-1 : table A lower tiles; nlt..2nlt-1 : table C; then T diagonal B tiles
  const int nlt = T * (T + 1) / 2;
  if (u < 2 * nlt) {
    table = (u < nlt) ? 0 : 2;  // gram slots: 0 = GA, 1 = GB, 2 = GC
    int r = (u < nlt) ? u : u - nlt;
    int i = 0;
    while (r >= i + 1) { r -= i + 1; ++i; }
    ti = i; tj = r;
  } else {
    table = 1; ti = tj = u - 2 * nlt;
  }
}

__global__ void __launch_bounds__(UPD_THREADS)
update_kernel(UpdateArgs p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ float smem[];
  const int tid = threadIdx.x;
  const int k = p.k;
  const int64_t d = p.d;
  const int T = (k + 31) / 32;
  const int nlt = T * (T + 1) / 2;
  const int units = 2 * nlt + T;
  const int nseg = (int)((d + UPD_SEG - 1) / UPD_SEG);

  // ---------------- phase 1: Gram partial sums ----------------
  {
    float* Vs = smem;                 // [32][65]
    float* Ps = smem + 32 * 65;       // [32][65]
    const int li = tid >> 3;          // 0..31 : row i within tile
    const int lj = (tid & 7) * 4;     // 0..28 : 4 columns j within tile
    for (int w = blockIdx.x; w < units * nseg; w += gridDim.x) {
      const int seg = w / units, u = w % units;
      int table, ti, tj;
      unit_decode(u, T, table, ti, tj);
      const float* P = table == 0 ? p.AV : (table == 1 ? p.BV : p.AUX);
      const int i0 = ti * 32, j0 = tj * 32;
      const int64_t c0 = (int64_t)seg * UPD_SEG;
      const int64_t c1 = min((int64_t)d, c0 + UPD_SEG);
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      for (int64_t x0 = c0; x0 < c1; x0 += 64) {
        for (int e = tid; e < 32 * 64; e += UPD_THREADS) {
          const int r = e >> 6, x = e & 63;
          const int64_t gx = x0 + x;
          const bool inx = gx < c1;
          Vs[r * 65 + x] = (inx && i0 + r < k) ? p.V[(int64_t)(i0 + r) * d + gx] : 0.f;
          Ps[r * 65 + x] = (inx && j0 + r < k) ? P[(int64_t)(j0 + r) * d + gx] : 0.f;
        }
        __syncthreads();
#pragma unroll 8
        for (int x = 0; x < 64; ++x) {
          const float a = Vs[li * 65 + x];
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[c] = fmaf(a, Ps[(lj + c) * 65 + x], acc[c]);
        }
        __syncthreads();
      }
      float* out = p.partial + ((int64_t)seg * units + u) * 1024;
#pragma unroll
      for (int c = 0; c < 4; ++c) out[li * 32 + lj + c] = acc[c];
    }
  }
  grid.sync();

  // ---------------- phase 2a: reduce partials -> gram ----------------
  {
    const int64_t total = (int64_t)units * 1024;
    for (int64_t e = (int64_t)blockIdx.x * UPD_THREADS + tid; e < total;
         e += (int64_t)gridDim.x * UPD_THREADS) {
      const int u = (int)(e >> 10), q = (int)(e & 1023);
      int table, ti, tj;
      unit_decode(u, T, table, ti, tj);
      const int i = ti * 32 + (q >> 5), j = tj * 32 + (q & 31);
      if (i >= k || j >= k) continue;
      float s = 0.f;
      for (int sg = 0; sg < nseg; ++sg) s += p.partial[((int64_t)sg * units + u) * 1024 + q];
      const bool keep = (table == 1) ? (i == j) : (i >= j);
      p.gram[(int64_t)table * k * k + (int64_t)i * k + j] = keep ? s : 0.f;
    }
  }
  grid.sync();

  // ---------------- phase 2b: coefficients ----------------
  {
    const float* GA = p.gram;
    const float* GB = p.gram + (int64_t)k * k;
    const float* GC = p.gram + 2 * (int64_t)k * k;
    const int lane = tid & 31, warp = tid >> 5;
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
        p.coef[(int64_t)i * k + j] = l;
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
  float* Ls = smem;                                 // k x k
  float* D1s = Ls + (size_t)k * k;                  // k
  float* D2s = D1s + k;                             // k
  float* Xs = D2s + k;                              // k x UPD_CW  (AUX chunk)
  float* Ns = Xs + (size_t)k * UPD_CW;              // k (norm partial)
  for (int e = tid; e < k * k + 2 * k; e += UPD_THREADS) Ls[e] = p.coef[e];
  for (int e = tid; e < k; e += UPD_THREADS) Ns[e] = 0.f;
  __syncthreads();
  const int nchunk = (int)((d + UPD_CW - 1) / UPD_CW);
  const int lane = tid & 31, warp = tid >> 5;
  for (int ch = blockIdx.x; ch < nchunk; ch += gridDim.x) {
    const int64_t gx = (int64_t)ch * UPD_CW + lane;
    const bool in = gx < d;
    for (int i = warp; i < k; i += UPD_THREADS / 32)
      Xs[i * UPD_CW + lane] = in ? p.AUX[(int64_t)i * d + gx] : 0.f;
    __syncthreads();
    for (int i = warp; i < k; i += UPD_THREADS / 32) {
      float vn = 0.f;
      if (in) {
        const int64_t o = (int64_t)i * d + gx;
        float g = D1s[i] * p.AV[o] - D2s[i] * p.BV[o];
        const float* Li = Ls + (size_t)i * k;
        for (int j = 0; j < i; ++j) g = fmaf(-Li[j], Xs[j * UPD_CW + lane], g);
        vn = p.V[o] + p.eta * g;
        const float ax = Xs[i * UPD_CW + lane];
        p.AUX[o] = ax + p.gamma * (p.BV[o] - ax);
        p.Vtmp[o] = vn;
      }
      const float sq = warp_sum(vn * vn);
      if (lane == 0) Ns[i] += sq;
    }
    __syncthreads();
  }
  for (int e = tid; e < k; e += UPD_THREADS) p.norm_partial[(int64_t)blockIdx.x * k + e] = Ns[e];
  grid.sync();

  // ---------------- phase 4: retraction v <- v'/||v'|| ----------------
  for (int i = tid; i < k; i += UPD_THREADS) {
    float s = 0.f;
    for (int b = 0; b < (int)gridDim.x; ++b) s += p.norm_partial[(int64_t)b * k + i];
    Ns[i] = rsqrtf(s);
  }
  __syncthreads();
  for (int ch = blockIdx.x; ch < nchunk; ch += gridDim.x) {
    const int64_t gx = (int64_t)ch * UPD_CW + lane;
    if (gx >= d) continue;
    for (int i = warp; i < k; i += UPD_THREADS / 32) {
      const int64_t o = (int64_t)i * d + gx;
      const float v = p.Vtmp[o] * Ns[i];
      p.V[o] = v;
      if (p.Vbf) p.Vbf[o] = __float2bfloat16_rn(v);
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
