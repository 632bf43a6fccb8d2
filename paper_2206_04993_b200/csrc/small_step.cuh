// small_step.cuh — the whole step of Alg. 2 for SMALL problems in one CTA,
// T steps per launch (the fp32 FFMA variant for configs 0 and 1).
//
// PAPER.md:1005-1025 (Alg. 2 lines 4-19; Alg. 1, for the
// dense full-batch problem).  Config 1 (dx = dy = 64, k = 8, b = 256) is
// 128 KB of batch and ~0.5 M multiply-adds per step: a grid-wide schedule
// spends its time in launches and grid barriers (~4 launches, 77 us per
// step on the staged path), so here ONE CTA of 512 threads runs every stage
// with __syncthreads between them and keeps the state resident in shared
// memory across the steps of the launch:
//
//   state   V'' (k x d), [Bv] (k x d) in smem for the whole launch (the
//           retraction of Alg. 2 l.17 folded into the next step, as in
//           update.cuh: the products use v'' and the coefficients carry
//           n_i = 1/||v''_i||)
//   batch   row chunks of [X | Y] (rc rows, both views side by side) stream
//           through a double-buffered cp.async ring; the NEXT chunk (also
//           across a step boundary: batches do not depend on the state) is
//           in flight while the current one is used — each byte is read
//           from HBM once per step (z of a row needs only that row, so the
//           forward and the backward products of a chunk use the same
//           staged rows)
//   F       z = [X v''_x, Y v''_y] for the chunk's rows (4 rows x 2
//           players register tiles)
//   B       AV''_i = (1/h) [X1^T zy1 ; Y1^T zx1], BV''_i = (1/h) [X2^T zx2 ;
//           Y2^T zy2] (halves of reading R1) accumulated in registers over
//           all chunks: thread = (4 players x 4 columns tile, row group g),
//           the RG row groups of a tile are lanes of one warp and are summed
//           by shuffles in fixed order at the end of the step (deterministic)
//   G       raw tables G'^A_ij = <v''_i, AV''_j>, G'^C_ij = <v''_i, [Bv]_j>
//           (j <= i), G'^B_ii = <v''_i, BV''_i>, ||v''_i||^2: warp dot
//           products over d
//   C       coefficients (Alg. 2 l.8-11; Alg. 3 l.7, 14, 21 when smooth):
//           the algebra of update.cuh's phase 3a
//   U       v'' <- n v'' + eta (D1 n AV'' - D2 n BV'' - sum_{j<i} L_ij [Bv]_j),
//           [Bv] <- [Bv] + gamma (n BV'' - [Bv]) (l.12-19)
//
// Dense (Alg. 1 products A v, B v of full d x d matrices): A and B are staged
// into smem ONCE per launch and the products are the forward tile loop with
// the rows of A (B) in place of the batch rows.
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"
#include "tc_gemm.cuh"

namespace geig {

namespace cgs = cooperative_groups;
constexpr int SM_THREADS = 512;
constexpr int SM_SMEM_MAX = 227 * 1024;

struct SmallParams {
  int dense;                 // 1: dense problem (xs / x0, y0 are A, B, d x d)
  int k, KPr;                // players; padded player count (8 or 16)
  int dx, dy, d;             // view widths (dense: dx = d, dy = 0)
  int b, h;                  // batch rows, half (reading R1)
  int nsteps;
  const void* const* xs;     // nsteps x 2 device pointers (X_t, Y_t); nullptr: x0, y0 for every step
  const void* x0;
  const void* y0;
  float scale, eta, gamma, rho;
  float* V;                  // k x d v'' (in/out)
  float* AUX;                // k x d [Bv] (in/out)
  float* AV;                 // k x d out: AV'' of the last step (scaled)
  float* BV;                 // k x d out: BV'' of the last step
  __nv_bfloat16* Vbf;        // 2 x k x d bf16 shadow (hi, lo) of the final v'' (nullable)
  float* gram;               // 3 x k x k normalised tables of the last step
  int smooth;                // Alg. 3
  float* zbuf;
  int zpar;
  float lnrho, lnnu;
  int rc;                    // rows per chunk (multiple of 4)
  int dpad;                  // (unused: chunk rows are unpadded, [rc][dx] | [rc][dy])
  int RG;                    // row groups of the backward (1, 2 or 4)
  unsigned long long* ts;    // %globaltimer at start / end (nullable, CTA 0)
  unsigned long long* prof;  // developer: clock64 cycles per phase summed over the launch (8 slots), nullable
  int cl;                    // CTAs of the thread-block cluster running the step (1: one CTA): CTA r takes
                             // rows [r bq, (r + 1) bq) of every batch and owns columns [r dq, (r + 1) dq)
  int bq, dq;                // rows / columns per cluster rank (dq a multiple of 4)
};

// developer phase profile: thread 0 adds the cycles since the last mark to slot `ph`
struct SmProf {
  long long last = 0;
  long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  __device__ __forceinline__ void mark(bool on, int ph) {
    if (on) {
      const long long c = clock64();
      acc[ph] += c - last;
      last = c;
    }
  }
};

template <typename T>
__device__ __forceinline__ float4 ld4(const T* p);
template <>
__device__ __forceinline__ float4 ld4<float>(const float* p) { return *reinterpret_cast<const float4*>(p); }
template <>
__device__ __forceinline__ float4 ld4<__nv_bfloat16>(const __nv_bfloat16* p) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}

// One 1-D bulk copy (TMA engine, no tensor map) global -> shared, completing
// on the mbarrier (16-byte aligned addresses, size a multiple of 16).
__device__ __forceinline__ void sm_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}

// Thread 0 stages rows [r0, r0 + nr) of both views into buf: the rows of
// a view are one contiguous block in global memory, so a chunk is two bulk
// copies (X block [rc][dx], then the Y block [rc][dy] at buf + rc dx;
// 16-byte aligned: dx, dy multiples of 16 B).  Rows of the last quad past
// nr keep stale values: their z is computed and never read.
template <typename T>
__device__ __forceinline__ void sm_stage_rows(T* buf, const T* X, const T* Y, int dx, int dy, int rc, int r0, int nr,
                                              uint64_t* bar) {
  const uint32_t bx = (uint32_t)nr * (uint32_t)dx * (uint32_t)sizeof(T), by = (uint32_t)nr * (uint32_t)dy * (uint32_t)sizeof(T);
  tc::mbar_expect_tx(bar, bx + by);
  sm_bulk(buf, X + (int64_t)r0 * dx, bx, bar);
  if (by) sm_bulk(buf + (size_t)rc * dx, Y + (int64_t)r0 * dy, by, bar);
}

// out[r][i] (row stride ldo) = sum_{c < len} rows[r][c] * V[i][c] (row
// strides dr, ldv), rows [0, nr4) (multiple of 4), players [0, KP); 4 rows x
// 2 players per unit, players fastest across lanes (the 4 lanes of a row
// quad read the same X words: broadcast).  Accumulated over c ascending.
template <typename T>
__device__ __forceinline__ void sm_forward(const T* rows, int dr, const float* V, int ldv, int len, int nr4, int KP,
                                           float* out, int ldo, int u0, int ustride) {
  const int nip = KP / 2;
  const int nunits = (nr4 / 4) * nip;
  for (int u = u0; u < nunits; u += ustride) {
    const int ip = u % nip, r4 = u / nip;
    const T* xr = rows + (4 * r4) * dr;
    const float* v0 = V + (2 * ip) * ldv;
    const float* v1 = v0 + ldv;
    float acc[4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a) acc[a][0] = acc[a][1] = 0.f;
    // Two row quads share each 8-lane shared-memory phase and their rows are
    // whole multiples of 128 B apart in the unpadded chunk: odd row quads
    // take the column quads of a pair in swapped order (c + 4, then c), so
    // the phase's X and V words fall in disjoint banks.
    const int sw = ((r4 & 1) && (len & 7) == 0) ? 4 : 0;
    const int len8 = (len & 7) == 0 ? len : 0;
    for (int c = 0; c < len8; c += 8) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cc = c + (h == 0 ? sw : (sw ^ 4));
        const float4 w0 = *reinterpret_cast<const float4*>(v0 + cc);
        const float4 w1 = *reinterpret_cast<const float4*>(v1 + cc);
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const float4 x = ld4<T>(xr + a * dr + cc);
          acc[a][0] = fmaf(x.x, w0.x, fmaf(x.y, w0.y, fmaf(x.z, w0.z, fmaf(x.w, w0.w, acc[a][0]))));
          acc[a][1] = fmaf(x.x, w1.x, fmaf(x.y, w1.y, fmaf(x.z, w1.z, fmaf(x.w, w1.w, acc[a][1]))));
        }
      }
    }
    for (int c = len8; c < len; c += 4) {   // views whose width is not a multiple of 8
      const float4 w0 = *reinterpret_cast<const float4*>(v0 + c);
      const float4 w1 = *reinterpret_cast<const float4*>(v1 + c);
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const float4 x = ld4<T>(xr + a * dr + c);
        acc[a][0] = fmaf(x.x, w0.x, fmaf(x.y, w0.y, fmaf(x.z, w0.z, fmaf(x.w, w0.w, acc[a][0]))));
        acc[a][1] = fmaf(x.x, w1.x, fmaf(x.y, w1.y, fmaf(x.z, w1.z, fmaf(x.w, w1.w, acc[a][1]))));
      }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      out[(4 * r4 + a) * ldo + 2 * ip] = acc[a][0];
      out[(4 * r4 + a) * ldo + 2 * ip + 1] = acc[a][1];
    }
  }
}

__device__ __forceinline__ int sm_tri(int i, int j) { return i * (i + 1) / 2 + j; }
__device__ __forceinline__ void sm_untri(int e, int& i, int& j) {
  i = (int)((sqrtf(8.f * (float)e + 1.f) - 1.f) * 0.5f);
  while (sm_tri(i + 1, 0) <= e) ++i;
  while (sm_tri(i, 0) > e) --i;
  j = e - sm_tri(i, 0);
}

// acc[16] += z[a] * x[cc] over rows [rbeg, rend) with stride RG (4 players x 4 columns)
template <typename T>
__device__ __forceinline__ void sm_bwd_rows(float (&acc)[16], const T* col, int dr, const float* zs, int ldz,
                                            int zcol, int rbeg, int rend, int RG) {
#pragma unroll 2
  for (int r = rbeg; r < rend; r += RG) {
    const float4 x = ld4<T>(col + r * dr);
    const float4 z = *reinterpret_cast<const float4*>(zs + r * ldz + zcol);
    const float xv[4] = {x.x, x.y, x.z, x.w}, zv[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) acc[4 * a + cc] = fmaf(zv[a], xv[cc], acc[4 * a + cc]);
  }
}

template <typename T, int KP>
__global__ void __launch_bounds__(SM_THREADS, 1)
small_step_kernel(const SmallParams p) {
  extern __shared__ __align__(16) uint8_t sm_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = p.k, d = p.d, dx = p.dx;
  const int ldz = 2 * KP + 4;                       // z row stride (floats): float4 rows of 8 lanes conflict-free
  const int ldv = d + 4;                            // state row stride: rows 4 banks apart
  // ---- shared memory layout (small_smem_bytes) ----
  float* Vs = reinterpret_cast<float*>(sm_raw);     // [KP][ldv] v''
  float* Cs = Vs + KP * ldv;                        // [KP][ldv] [Bv] (swaps with Bs every step)
  float* As = Cs + KP * ldv;                        // [KP][ldv] AV''
  float* Bs = As + KP * ldv;                        // [KP][ldv] BV''
  float* zs = Bs + KP * ldv;                        // [rc][ldz] (dense: unused)
  float* tab = zs + (p.dense ? 0 : p.rc * ldz);     // tables
  const int ntri = k * (k + 1) / 2;
  float* rA = tab;                                  // tri(G'^A)
  float* rC = rA + ntri;                            // tri(G'^C)
  float* rB = rC + ntri;                            // diag G'^B
  float* rN = rB + KP;                              // ||v''||^2
  float* Ns = rN + KP;
  float* IS2 = Ns + KP;
  float* D1s = IS2 + KP;
  float* D2s = D1s + KP;
  float* Lt = D2s + KP;                             // [KP][KP] Lt[j][i] = L_ij
  float* pt = Lt + KP * KP;                         // cluster: this CTA's partial tables [tri A | tri C | B | N]
  const int npt = 2 * ntri + 2 * KP;
  uint64_t* full = reinterpret_cast<uint64_t*>(pt + npt + ((KP * KP + npt) & 1));   // 2 mbarriers (8-byte aligned)
  // chunk buffers, 16-byte aligned (the same offset as small_smem_bytes)
  const size_t ring_off = ((size_t)(reinterpret_cast<float*>(full + 2) - Vs) + 3) & ~(size_t)3;
  T* ring = reinterpret_cast<T*>(Vs + ring_off);
  T* const buf0 = ring;                             // dense: A (d rows)
  T* const buf1 = ring + (size_t)p.rc * d;         // dense: B (d rows); CCA: [rc][dx] | [rc][dy]

  if (p.ts && tid == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.ts[0] = t;
  }
  if (tid == 0) {
    tc::mbar_init(&full[0], 1);
    tc::mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // ---- state into smem (rows >= k zero) ----
  for (int e = tid; e < KP * d; e += SM_THREADS) {
    const int i = e / d, c = e - i * d;
    Vs[i * ldv + c] = i < k ? p.V[e] : 0.f;
    Cs[i * ldv + c] = i < k ? p.AUX[e] : 0.f;
  }
  __syncthreads();
  // cluster rank: rows [rlo, rhi) of every batch, own columns [clo, chi)
  cgs::cluster_group cluster = cgs::this_cluster();
  const int C = p.cl;
  const int rank = C > 1 ? (int)cluster.block_rank() : 0;
  const int rlo = p.dense ? 0 : min(p.b, rank * p.bq), rhi = p.dense ? 0 : min(p.b, rlo + p.bq);
  const int clo = C > 1 ? min(d, rank * p.dq) : 0, chi = C > 1 ? min(d, clo + p.dq) : d;
  const int nrows = rhi - rlo;
  const int nchunks = p.dense ? 1 : max(1, (nrows + p.rc - 1) / p.rc);
  auto batch = [&](int t, int v) -> const T* {
    return reinterpret_cast<const T*>(p.xs ? p.xs[2 * t + v] : (v == 0 ? p.x0 : p.y0));
  };
  if (tid == 0) {
    if (p.dense) {
      // A and B once for the launch (Alg. 1: the same full-batch matrices every step)
      sm_stage_rows<T>(buf0, batch(0, 0), batch(0, 0), d, 0, p.rc, 0, d, &full[0]);
      sm_stage_rows<T>(buf1, batch(0, 1), batch(0, 1), d, 0, p.rc, 0, d, &full[1]);
    } else {
      sm_stage_rows<T>(buf0, batch(0, 0), batch(0, 1), dx, p.dy, p.rc, rlo, min(p.rc, nrows), &full[0]);
    }
  }

  // backward unit of this thread: tile (4 players i4, 4 columns c4), row
  // group g.  Lane bits 0-2: 8 consecutive column quads (the 8 lanes of a
  // shared-memory phase read 128 contiguous bytes of one row; z broadcast),
  // bits 3..: the row group (RG <= 4), then the (i4, column-quad group).
  const int RG = p.RG;
  const int lgRG = RG >= 4 ? 2 : (RG >= 2 ? 1 : 0);
  const int g = (tid >> 3) & (RG - 1);
  const int rest = tid >> (3 + lgRG);
  const int ni4 = KP / 4;
  const int i4 = rest % ni4, c4 = (rest / ni4) * 8 + (tid & 7);
  const bool bwd = 4 * c4 < d;
  const int cb = 4 * c4;
  const bool colx = cb < dx;                        // view of the tile's columns (dx % 4 == 0)

  int q = 0;                                        // global chunk counter (ring parity)
  const bool prof = p.prof && tid == 0;
  SmProf pf;
  if (prof) pf.last = clock64();
  for (int t = 0; t < p.nsteps; ++t) {
    float acc[32];                                  // [0,16): AV'' tile, [16,32): BV'' tile ([a][cc])
#pragma unroll
    for (int e = 0; e < 32; ++e) acc[e] = 0.f;

    if (p.dense) {
      if (t == 0) { tc::mbar_wait(&full[0], 0); tc::mbar_wait(&full[1], 0); }   // A, B resident
    } else {
      for (int c = 0; c < nchunks; ++c, ++q) {
        const int r0 = rlo + c * p.rc, nr = min(p.rc, rhi - r0);
        // next chunk (of this step or of the next one) into the other buffer:
        // its previous contents were last read before the barrier that ended
        // the previous chunk
        if (tid == 0) {
          int tn = t, cn = c + 1;
          if (cn == nchunks) { tn = t + 1; cn = 0; }
          if (tn < p.nsteps)
            sm_stage_rows<T>(((q & 1) ? buf0 : buf1), batch(tn, 0), batch(tn, 1), dx, p.dy, p.rc, rlo + cn * p.rc,
                             min(p.rc, nrows - cn * p.rc), &full[(q + 1) & 1]);
        }
        tc::mbar_wait(&full[q & 1], (uint32_t)((q >> 1) & 1));
        pf.mark(prof, 0);
        const T* rows = ((q & 1) ? buf1 : buf0);
        const int nr4 = (nr + 3) & ~3;
        // ---- F: z[r][0:KP] = x_r . v''_x, z[r][KP:2KP] = y_r . v''_y ----
        sm_forward<T>(rows, dx, Vs, ldv, dx, nr4, KP, zs, ldz, tid, SM_THREADS);
        sm_forward<T>(rows + (size_t)p.rc * dx, p.dy, Vs + dx, ldv, p.dy, nr4, KP, zs + KP, ldz,
                      (tid + SM_THREADS / 2) % SM_THREADS, SM_THREADS);
        __syncthreads();
        pf.mark(prof, 1);
        // ---- B: the tile over the chunk's rows of group g: rows [0, ra) are
        // in the A half (AV_x uses zy, AV_y uses zx), rows [ra, rb) in the B
        // half (BV_x uses zx, BV_y uses zy), rows >= 2h unused (odd b) ----
        if (bwd) {
          const int ra = min(max(p.h - r0, 0), nr), rb = min(max(2 * p.h - r0, 0), nr);
          const T* col = colx ? rows + cb : rows + (size_t)p.rc * dx + (cb - dx);
          const int dr = colx ? dx : p.dy;
          sm_bwd_rows<T>(*reinterpret_cast<float(*)[16]>(acc), col, dr, zs, ldz, (colx ? KP : 0) + 4 * i4, g, ra, RG);
          const int rb0 = ra + ((g - ra) % RG + RG) % RG;   // first row >= ra of group g
          sm_bwd_rows<T>(*reinterpret_cast<float(*)[16]>(acc + 16), col, dr, zs, ldz, (colx ? 0 : KP) + 4 * i4, rb0,
                         rb, RG);
        }
        __syncthreads();   // the buffer is refilled by the next iteration's stage
        pf.mark(prof, 2);
      }
      // ---- combine the RG row groups (lanes 8 g + cq of one warp): a
      // reduce-scatter over the 32 accumulators in fixed order; the lane of
      // group g keeps 32 / RG sums ----
      int base = 0;
#pragma unroll
      for (int l = 0; l < 2; ++l) {
        const int o = RG >> (l + 1);
        if (o >= 1) {
          const int half = 16 >> l;
          const bool up = (g & o) != 0;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (j < half) {
              const float send = up ? acc[j] : acc[j + half];
              const float keep = up ? acc[j + half] : acc[j];
              acc[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8 * o);
            }
          }
          if (up) base += half;
        }
      }
      if (bwd) {
        const int n = 32 / RG;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (j < n) {
            const int f = base + j, m = f >> 4, a = (f >> 2) & 3, cc = f & 3;
            (m ? Bs : As)[(4 * i4 + a) * ldv + cb + cc] = p.scale * acc[j];
          }
        }
      }
    }
    if (p.dense) {
      // products of the resident A, B (Alg. 1): As[i][c] = (A v''_i)_c =
      // sum_r A[c][r] v''_i[r], Bs likewise; 4 rows of A x 2 players per unit
      const int d4 = (d + 3) & ~3;
      const int nip = KP / 2, nunits = (d4 / 4) * nip;
      for (int u = tid; u < 2 * nunits; u += SM_THREADS) {
        const int m = u / nunits, uu = u - m * nunits;
        const int ip = uu % nip, r4 = uu / nip;
        const T* xr = (m ? buf1 : buf0) + (4 * r4) * d;
        const float* v0 = Vs + (2 * ip) * ldv;
        const float* v1 = v0 + ldv;
        float ac[4][2];
#pragma unroll
        for (int a = 0; a < 4; ++a) ac[a][0] = ac[a][1] = 0.f;
        for (int c = 0; c < d; c += 4) {
          const float4 w0 = *reinterpret_cast<const float4*>(v0 + c);
          const float4 w1 = *reinterpret_cast<const float4*>(v1 + c);
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const float4 x = ld4<T>(xr + a * d + c);
            ac[a][0] = fmaf(x.x, w0.x, fmaf(x.y, w0.y, fmaf(x.z, w0.z, fmaf(x.w, w0.w, ac[a][0]))));
            ac[a][1] = fmaf(x.x, w1.x, fmaf(x.y, w1.y, fmaf(x.z, w1.z, fmaf(x.w, w1.w, ac[a][1]))));
          }
        }
        float* out = m == 0 ? As : Bs;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int r = 4 * r4 + a;
          if (r < d) {
            out[(2 * ip) * ldv + r] = ac[a][0];
            out[(2 * ip + 1) * ldv + r] = ac[a][1];
          }
        }
      }
    }
    __syncthreads();
    pf.mark(prof, 3);
    // ---- G: raw tables; 8 lanes per entry over d, fixed-order shuffles ----
    {
      const int nent = 2 * ntri + 2 * k;
      const int l8 = lane & 7;
      for (int eb = warp * 4; eb < nent; eb += SM_THREADS / 8) {   // warp-uniform trip count (shuffles below)
        const int e = eb + (lane >> 3);
        const float* a = Vs;
        const float* b2 = Vs;
        float* dst = nullptr;
        if (e < ntri) {                                // G'^A_ij, j <= i
          int i, j;
          sm_untri(e, i, j);
          a = Vs + i * ldv; b2 = As + j * ldv; dst = rA + e;
        } else if (e < 2 * ntri) {                     // G'^C_ij
          int i, j;
          sm_untri(e - ntri, i, j);
          a = Vs + i * ldv; b2 = Cs + j * ldv; dst = rC + (e - ntri);
        } else if (e < 2 * ntri + k) {                 // G'^B_ii
          const int i = e - 2 * ntri;
          a = Vs + i * ldv; b2 = Bs + i * ldv; dst = rB + i;
        } else if (e < nent) {                         // ||v''_i||^2
          const int i = e - 2 * ntri - k;
          a = Vs + i * ldv; b2 = a; dst = rN + i;
        }
        // G'^A, G'^B are linear in the products: with a cluster each CTA sums
        // its row partials over ALL columns (no reduce-scatter needed first);
        // G'^C, ||v''||^2 need [Bv] / the state only where they are current:
        // the own columns
        const bool own_only = e >= ntri && (e < 2 * ntri || e >= 2 * ntri + k);
        const int c_lo = own_only ? clo : 0, c_hi = own_only ? chi : d;
        float sum = 0.f;
        if (dst)
          for (int c = c_lo + l8; c < c_hi; c += 8) sum = fmaf(a[c], b2[c], sum);
        sum += __shfl_xor_sync(0xffffffffu, sum, 4);
        sum += __shfl_xor_sync(0xffffffffu, sum, 2);
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        if (dst && l8 == 0) {
          if (C > 1) dst = pt + (dst - rA);   // the cluster sum below forms rA.. from every CTA's pt
          *dst = sum;
        }
      }
    }
    if (C > 1) {
      // ONE cluster barrier: every CTA's row-partial products and partial
      // tables are complete.  The tables are summed over the ranks (rank
      // order: identical in every CTA) and the products reduce-scattered:
      // this CTA sums its own columns of every CTA's As / Bs in place (the
      // others read only their own columns of these tiles)
      cluster.sync();
      {
        const int nc = chi - clo;
        for (int e = tid; e < 2 * k * nc; e += SM_THREADS) {
          const int h = e / (k * nc), r = e - h * k * nc, i = r / nc, c = clo + (r - i * nc);
          float* loc = (h ? Bs : As) + i * ldv + c;
          float vq[8];
#pragma unroll
          for (int q2 = 0; q2 < 8; ++q2) vq[q2] = q2 < C ? *cluster.map_shared_rank(loc, q2) : 0.f;   // all in flight
          float v = 0.f;
#pragma unroll
          for (int q2 = 0; q2 < 8; ++q2) v += vq[q2];   // rank order (the zeros past C are exact)
          *loc = v;
        }
      }
      for (int e = tid; e < 2 * ntri + 2 * k; e += SM_THREADS) {
        // offsets of [tri A | tri C | B (k of KP) | N (k of KP)]
        const int oo = e < 2 * ntri + k ? e : 2 * ntri + KP + (e - 2 * ntri - k);
        float vq[8];
#pragma unroll
        for (int q2 = 0; q2 < 8; ++q2) vq[q2] = q2 < C ? *cluster.map_shared_rank(pt + oo, q2) : 0.f;
        float v = 0.f;
#pragma unroll
        for (int q2 = 0; q2 < 8; ++q2) v += vq[q2];
        rA[oo] = v;
      }
    }
    __syncthreads();
    pf.mark(prof, 4);
    // ---- C: coefficients (update.cuh phase 3a algebra; Alg. 2 l.8-11, Alg. 3 l.7/14/21) ----
    if (tid < KP) {
      const int i = tid;
      float n = 0.f, is2 = 0.f, gb = 0.f;
      if (i < k) {
        n = rsqrtf(rN[i]);
        gb = n * n * rB[i];
        const float gcii = n * rC[sm_tri(i, i)];
        if (p.smooth) {
          const float* zr = p.zbuf + ((p.zpar + t) & 1) * 64;
          const float z = zr[i];
          const float sg = 1.f / (1.f + expf(-z));
          const float br = expf(p.lnrho + (p.lnnu - p.lnrho) * sg);
          is2 = 1.f / br;
          if (rank == 0) {
            float* zw = p.zbuf + ((p.zpar + t + 1) & 1) * 64;
            zw[i] = z + p.gamma * (gcii - br) * br * (p.lnnu - p.lnrho) * sg * (1.f - sg);
          }
        } else {
          is2 = 1.f / fmaxf(gcii, p.rho);
        }
      }
      Ns[i] = n; IS2[i] = is2; D1s[i] = gb;
    }
    __syncthreads();
    if (tid < KP * KP) {
      // L_ij = G^B_ii G^A_ij / s_j^2 (j < i), Lt[j][i]
      const int j = tid / KP, i = tid - j * KP;
      float l = 0.f;
      if (i < k && j < i) l = D1s[i] * (Ns[i] * Ns[j] * rA[sm_tri(i, j)]) * IS2[j];
      Lt[j * KP + i] = l;
    } else if (tid >= 256 && tid < 256 + KP) {
      // c_i = sum_{j<i} G^A_ij G^C_ij / s_j^2, D2_i = G^A_ii - c_i
      const int i = tid - 256;
      float c = 0.f;
      if (i < k) {
        for (int j = 0; j < i; ++j)
          c = fmaf(Ns[i] * Ns[j] * rA[sm_tri(i, j)], Ns[i] * rC[sm_tri(i, j)] * IS2[j], c);
      }
      D2s[i] = i < k ? Ns[i] * Ns[i] * rA[sm_tri(i, i)] - c : 0.f;
    }
    const int nc = chi - clo;                       // this CTA's columns (all of them when C == 1)
    if (t + 1 == p.nsteps) {
      // the last step's products to global memory (before the update reuses Bs)
      for (int e = tid; e < k * nc; e += SM_THREADS) {
        const int i = e / nc, c = clo + (e - i * nc);
        p.AV[(int64_t)i * d + c] = As[i * ldv + c];
        p.BV[(int64_t)i * d + c] = Bs[i * ldv + c];
      }
    }
    __syncthreads();
    if (t + 1 == p.nsteps && rank == 0) {
      // the last step's normalised tables (geig_get_gram)
      for (int e = tid; e < k * k; e += SM_THREADS) {
        const int i = e / k, j = e - (e / k) * k;
        const bool low = j <= i;
        const int tij = sm_tri(i, low ? j : 0);
        p.gram[e] = low ? Ns[i] * Ns[j] * rA[tij] : 0.f;
        p.gram[k * k + e] = (i == j) ? D1s[i] : 0.f;
        p.gram[2 * k * k + e] = low ? Ns[i] * rC[tij] : 0.f;
      }
    }
    pf.mark(prof, 5);
    // ---- U: direction, ascent, aux moving average (new aux into Bs, then swap) ----
    for (int e = tid; e < k * nc; e += SM_THREADS) {
      const int i = e / nc, c = clo + (e - i * nc);
      const int o = i * ldv + c;
      float pen = 0.f;
      for (int j = 0; j < i; ++j) pen = fmaf(Lt[j * KP + i], Cs[j * ldv + c], pen);
      const float ni = Ns[i];
      const float d1 = D1s[i] * ni, d2 = D2s[i] * ni;
      const float bv = Bs[o], xa = Cs[o];
      Vs[o] = ni * Vs[o] + p.eta * (d1 * As[o] - d2 * bv - pen);
      Bs[o] = xa + p.gamma * (ni * bv - xa);
    }
    __syncthreads();
    if (C > 1) {
      // every CTA's next forward reads all of v'': the own columns into the
      // other CTAs' copies (distributed shared memory), then a cluster barrier
      for (int e = tid; e < k * nc; e += SM_THREADS) {
        const int i = e / nc, c = clo + (e - i * nc);
        const float v = Vs[i * ldv + c];
        for (int q2 = 0; q2 < C; ++q2)
          if (q2 != rank) *cluster.map_shared_rank(Vs + i * ldv + c, q2) = v;
      }
      cluster.sync();
    }
    pf.mark(prof, 6);
    { float* tmp = Cs; Cs = Bs; Bs = tmp; }
  }
  // ---- state back to global memory (this CTA's columns) ----
  {
    const int nc = chi - clo;
    for (int e2 = tid; e2 < k * nc; e2 += SM_THREADS) {
      const int i = e2 / nc, c = clo + (e2 - i * nc);
      const int64_t e = (int64_t)i * d + c;
      const float v = Vs[i * ldv + c];
      p.V[e] = v;
      p.AUX[e] = Cs[i * ldv + c];
      if (p.Vbf) {
        const __nv_bfloat16 hv = __float2bfloat16_rn(v);
        p.Vbf[e] = hv;
        p.Vbf[(int64_t)k * d + e] = __float2bfloat16_rn(v - __bfloat162float(hv));
      }
    }
  }
  if (prof) {
    pf.mark(true, 7);
    for (int i = 0; i < 8; ++i) p.prof[i] = (unsigned long long)pf.acc[i];
  }
  if (p.ts && tid == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.ts[1] = t;
  }
}

// Host: smem bytes of a configuration (0 = does not fit).
inline size_t small_smem_bytes(bool dense, int KP, int d, int k, int rc, int dpad, size_t es) {
  const int ntri = k * (k + 1) / 2;
  const int npt = 2 * ntri + 2 * KP;
  size_t fl = (size_t)4 * KP * (d + 4) + (dense ? 0 : (size_t)rc * (2 * KP + 4)) + 2 * ntri + 6 * KP + KP * KP + npt +
              ((KP * KP + npt) & 1) + 4;
  fl = (fl + 3) & ~(size_t)3;   // ring 16-byte aligned
  (void)dpad;
  const size_t ring = 2 * (size_t)rc * d * es;   // dense: rc = d rounded up to 4
  return fl * 4 + ring;
}

}  // namespace geig
