// simt_gemm.cuh — FFMA fp32 tiled GEMM: the exactness-check variant of the
// minibatch products (GEIG_MATH_F32).  C(m, n) = sum_kk A(m, kk) * B(n, kk)
// over kk in [kbeg, kend), with compile-time operand layouts:
//   A_K: A(m,kk) = A[m*lda + kk]   (K-major)   else A[kk*lda + m] (M-major)
//   B_K: B(n,kk) = B[n*ldb + kk]   (K-major)   else B[kk*ldb + n] (N-major)
// 64x64 output tile per 256-thread CTA, BK = 16, 4x4 outputs per thread.
// The epilogue functor receives (m, n, value) for in-range outputs.
// Split-K (gridDim.z > 1, for the tall-skinny products whose M x N grid is
// a handful of tiles, e.g. the backward X^T Z with M = d_view, N = k, K = h):
// slice z sums kk in its K chunk and writes the raw partial to
// part[(z * N + n) * M + m]; simt_splitk_reduce then adds the slices in
// fixed order (deterministic) and applies the epilogue.
#pragma once
#include "common.cuh"

namespace geig {

constexpr int SG_BM = 64, SG_BN = 64, SG_BK = 16;

template <typename TA, typename TB, bool A_K, bool B_K, class Epi>
__global__ void __launch_bounds__(256)
simt_gemm_kernel(const TA* __restrict__ A, int64_t lda, const TB* __restrict__ B, int64_t ldb,
                 int M, int N, int64_t kbeg, int64_t kend, Epi epi, float* __restrict__ part = nullptr,
                 int64_t kchunk = 0) {
  if (gridDim.z > 1) {   // split-K slice
    kbeg += (int64_t)blockIdx.z * kchunk;
    kend = min(kend, kbeg + kchunk);
  }
  __shared__ float As[SG_BK][SG_BM + 4];
  __shared__ float Bs[SG_BK][SG_BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.x * SG_BM, n0 = blockIdx.y * SG_BN;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int64_t k0 = kbeg; k0 < kend; k0 += SG_BK) {
#pragma unroll
    for (int e = tid; e < SG_BM * SG_BK; e += 256) {
      int m, kk;
      if (A_K) { m = e / SG_BK; kk = e % SG_BK; } else { kk = e / SG_BM; m = e % SG_BM; }
      const int gm = m0 + m;
      const int64_t gk = k0 + kk;
      float v = 0.f;
      if (gm < M && gk < kend) v = to_f32(A_K ? A[(int64_t)gm * lda + gk] : A[gk * lda + gm]);
      As[kk][m] = v;
    }
#pragma unroll
    for (int e = tid; e < SG_BN * SG_BK; e += 256) {
      int n, kk;
      if (B_K) { n = e / SG_BK; kk = e % SG_BK; } else { kk = e / SG_BN; n = e % SG_BN; }
      const int gn = n0 + n;
      const int64_t gk = k0 + kk;
      float v = 0.f;
      if (gn < N && gk < kend) v = to_f32(B_K ? B[(int64_t)gn * ldb + gk] : B[gk * ldb + gn]);
      Bs[kk][n] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SG_BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
      if (m < M && n < N) {
        if (gridDim.z > 1) part[((int64_t)blockIdx.z * N + n) * M + m] = acc[i][j];
        else epi(m, n, acc[i][j]);
      }
    }
}

template <class Epi>
__global__ void __launch_bounds__(256)
simt_splitk_reduce(const float* __restrict__ part, int M, int N, int splits, Epi epi) {
  const int64_t MN = (int64_t)M * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < MN; e += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += part[z * MN + e];
    const int n = (int)(e / M), m = (int)(e - (int64_t)n * M);
    epi(m, n, s);
  }
}

// Epilogue of the CCA forward product Z_v = X_v V_v^T (rows r, player n):
// rows r < h feed the OTHER view's A-half backward, rows h <= r < 2h feed
// this view's B-half backward (reading R1), stored player-major W[n][r].
struct EpiForward {
  float* w_other;  // other view's backward operand, k x ldw
  float* w_self;   // this view's backward operand, k x ldw
  int64_t ldw;
  int h;
  __device__ __forceinline__ void operator()(int r, int n, float v) const {
    if (r < h) w_other[(int64_t)n * ldw + r] = v;
    else if (r < 2 * h) w_self[(int64_t)n * ldw + r] = v;
  }
};

// Epilogue writing C^T scaled: out[n*ldo + m] = scale * v (player-major).
struct EpiTransposeScale {
  float* out;
  int64_t ldo;
  float scale;
  __device__ __forceinline__ void operator()(int m, int n, float v) const {
    out[(int64_t)n * ldo + m] = scale * v;
  }
};

}  // namespace geig
