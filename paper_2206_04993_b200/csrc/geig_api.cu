// geig_api.cu — the C ABI of include/geig.h: solver state, scratch, dispatch
// of the product kernels (SIMT fp32 / tcgen05) and the cooperative update.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <algorithm>
#include <initializer_list>

#include "../../include/geig.h"
#include "common.cuh"
#include "simt_gemm.cuh"
#include "update.cuh"
#include "tc_gemm.cuh"
#include "fused_step.cuh"
#include "small_step.cuh"

using namespace geig;

static thread_local std::string g_err;

static geig_status fail(geig_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CU(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return fail(GEIG_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,           \
                  cudaGetErrorString(e_));                                            \
  } while (0)

#define CHECK_LAUNCH() CU(cudaGetLastError())

struct geig_solver {
  int problem = 0, math = 0, dtype = 0, device = 0;
  int64_t dx = 0, dy = 0, d = 0, max_rows = 0;
  int k = 0;
  float rho = 0.f;
  cudaStream_t stream = nullptr;
  // state
  float *V = nullptr, *AUX = nullptr;
  __nv_bfloat16* Vbf = nullptr;
  char* arena = nullptr;                              // V | AUX | AV | BV | Vbf (one allocation)
  size_t arena_bytes = 0;
  // scratch
  float *AV = nullptr, *BV = nullptr, *gram = nullptr, *raw = nullptr;
  float *partial = nullptr;
  unsigned long long* ts = nullptr;                   // phase stamps of the last update (device, 6)
  float *Wx = nullptr, *Wy = nullptr;                 // fp32 backward operands k x max_rows
  __nv_bfloat16 *Wxb = nullptr, *Wyb = nullptr;       // bf16 backward operands
  void *hX = nullptr, *hY = nullptr;                  // device staging for *_host
  void *hX2 = nullptr, *hY2 = nullptr;                // second staging pair (geig_run_cca_host double buffer)
  cudaStream_t copy_stream = nullptr;                 // H2D copies of geig_run_cca_host
  cudaEvent_t ev_loaded[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
  int upd_grid = 1;
  bool upd_res = false;                               // resident (k <= 64) update kernel
  bool fused_last = false;                            // last step ran the fused cooperative kernel
  // update variants (geig_set_smooth / geig_set_adam)
  int smooth = 0;
  float nu = 0.f;
  float* zbuf = nullptr;                              // 2 x 64 (double-buffered z of Alg. 3)
  int zpar = 0;
  int adam = 0;
  float b1 = 0.9f, b2 = 0.999f, eps = 1e-8f;
  float* am = nullptr;                                // k x d Adam moments
  float* as = nullptr;
  long long adam_t = 0;
  int64_t upd_segw = 32;
  size_t upd_smem = 0;
  int64_t launches = 0;
  tc::TcPlan tc;                                      // tcgen05 plans (tensor maps, scratch)
  int opt_staged = 0;                                 // geig_set_option(GEIG_OPT_STAGED_PRODUCTS)
  int nsm = 148;
  // column-owned multi-GPU step (geig_set_partition)
  int part_world = 1, part_rank = 0;
  int64_t part_W = 0;
  __nv_bfloat16* gshadow = nullptr;                   // [world][hi|lo][k][W] gathered bf16 shadow of V
  int own_grid = 1;
  int64_t own_segw = 0;
  float* splitk = nullptr;                            // SIMT split-K partials (lazily sized)
  size_t splitk_floats = 0;
  // peer exchange of the column-owned step (geig_set_peers)
  float* precv = nullptr;                             // [world][chunk] receive slots (local)
  unsigned* pflags = nullptr;                         // flag words (local): 2 x GEIG_MAX_PEERS lines of 32
  float* peer_recv[GEIG_MAX_PEERS] = {};
  __nv_bfloat16* peer_shadow[GEIG_MAX_PEERS] = {};
  unsigned* peer_flags[GEIG_MAX_PEERS] = {};
  bool peer_on = false;
  unsigned peer_epoch = 0;                            // last completed step
  unsigned peer_pending = 0;                          // products launched, update not yet
  // one-CTA small-problem step (small_step.cuh)
  int opt_small = 1;                                  // geig_set_option(GEIG_OPT_SMALL_STEP)
  int opt_gram_tc = 1;                                // geig_set_option(GEIG_OPT_GRAM_TC)
  int opt_small_cluster = 0;                          // geig_set_option(GEIG_OPT_SMALL_CLUSTER): 0 auto, else CTAs
  const void** ptab_dev = nullptr;                    // per-step batch pointers of a run (device, pinned staging)
  const void** ptab_host = nullptr;
  cudaEvent_t ptab_ev = nullptr;
};

extern "C" const char* geig_last_error(void) { return g_err.c_str(); }
extern "C" const char* geig_version(void) { return "geig 0.1 (sm_100a)"; }
extern "C" int64_t geig_launch_count(const geig_solver* s) { return s ? s->launches : 0; }

static void set_l2_window(geig_solver* s);

extern "C" geig_status geig_create(geig_solver** out, int problem, int64_t dx, int64_t dy,
                                   int32_t k, int math, int data_dtype, double rho,
                                   int64_t max_rows, int device) {
  if (!out) return fail(GEIG_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (problem != GEIG_DENSE && problem != GEIG_CCA) return fail(GEIG_ERR_ARG, "bad problem %d", problem);
  if (k < 1) return fail(GEIG_ERR_ARG, "k must be >= 1");
  if (k > 128) return fail(GEIG_ERR_UNSUPPORTED, "k=%d > 128 not compiled", k);
  if (dx < 1 || dy < 0 || (problem == GEIG_CCA && dy < 1) || (problem == GEIG_DENSE && dy != 0))
    return fail(GEIG_ERR_ARG, "bad dims dx=%lld dy=%lld", (long long)dx, (long long)dy);
  if (math < GEIG_MATH_F32 || math > GEIG_MATH_BF16X2) return fail(GEIG_ERR_ARG, "bad math %d", math);
  if (data_dtype != GEIG_DATA_F32 && data_dtype != GEIG_DATA_BF16) return fail(GEIG_ERR_ARG, "bad dtype");
  if ((math == GEIG_MATH_BF16 || math == GEIG_MATH_BF16X2) && data_dtype != GEIG_DATA_BF16)
    return fail(GEIG_ERR_ARG, "GEIG_MATH_BF16/BF16X2 require bf16 data");
  if ((math == GEIG_MATH_TF32 || math == GEIG_MATH_3XTF32) && data_dtype != GEIG_DATA_F32)
    return fail(GEIG_ERR_ARG, "tf32 math requires fp32 data");
  if (!(rho >= 0.0)) return fail(GEIG_ERR_ARG, "rho must be >= 0");
  if (problem == GEIG_CCA && max_rows < 2) return fail(GEIG_ERR_ARG, "max_rows must be >= 2");
  if (k > dx + dy) return fail(GEIG_ERR_ARG, "k > d");

  geig_solver* s = new geig_solver();
  s->problem = problem; s->math = math; s->dtype = data_dtype; s->device = device;
  s->dx = dx; s->dy = dy; s->d = dx + dy; s->k = k; s->rho = (float)rho;
  s->max_rows = problem == GEIG_CCA ? max_rows : 0;
  auto cleanup = [&](geig_status st) { geig_destroy(s); return st; };
  if (cudaSetDevice(device) != cudaSuccess) return cleanup(fail(GEIG_ERR_CUDA, "cudaSetDevice(%d)", device));
  const size_t kd = (size_t)k * s->d;
#define ALLOC(ptr, bytes)                                                               \
  if (cudaMalloc((void**)&(ptr), (bytes)) != cudaSuccess)                              \
    return cleanup(fail(GEIG_ERR_CUDA, "cudaMalloc %zu bytes failed", (size_t)(bytes)));
  // One arena for the per-step state (V, [Bv], bf16 shadow, AV, BV: 18 B per
  // k x d element) so a single L2 persistence window can pin it while the
  // minibatch streams through L2 (see set_l2_window).
  {
    const size_t arena = kd * (4 + 4 + 4 + 4 + 4);
    char* base = nullptr;
    if (cudaMalloc((void**)&base, arena) != cudaSuccess)
      return cleanup(fail(GEIG_ERR_CUDA, "cudaMalloc state arena %zu bytes failed", arena));
    s->arena = base;
    s->arena_bytes = arena;
    s->V = (float*)base;
    s->AUX = (float*)(base + kd * 4);
    s->AV = (float*)(base + kd * 8);
    s->BV = (float*)(base + kd * 12);
    s->Vbf = (__nv_bfloat16*)(base + kd * 16);      // hi + lo planes
  }
  ALLOC(s->gram, (size_t)3 * k * k * 4);
  ALLOC(s->ts, 8 * sizeof(unsigned long long));
  cudaMemset(s->ts, 0, 8 * sizeof(unsigned long long));
  if (problem == GEIG_CCA) {
    const int64_t mr = ((max_rows + 127) / 128) * 128;
    ALLOC(s->Wx, (size_t)k * mr * 4);
    ALLOC(s->Wy, (size_t)k * mr * 4);
    ALLOC(s->Wxb, (size_t)k * mr * 2);
    ALLOC(s->Wyb, (size_t)k * mr * 2);
  }
#undef ALLOC
  cudaMemset(s->V, 0, kd * 4);
  cudaMemset(s->AUX, 0, kd * 4);
  cudaMemset(s->Vbf, 0, kd * 2 * 2);
  cudaMemset(s->gram, 0, (size_t)3 * k * k * 4);

  // cooperative update grid: one co-resident CTA per SM, contiguous column ranges
  {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    s->nsm = std::max(1, nsm);
    int64_t G = std::min<int64_t>(nsm, (s->d + UPD_XC - 1) / UPD_XC);
    G = std::max<int64_t>(G, 1);
    int64_t segw = (s->d + G - 1) / G;
    const bool res = k <= 64 && ((segw + 7) / 8) * 8 <= UPD_RES_WMAX;
    segw = res ? ((segw + 7) / 8) * 8 : ((segw + 3) / 4) * 4;
    G = (s->d + segw - 1) / segw;
    s->upd_grid = (int)G;
    s->upd_segw = segw;
    s->upd_res = res;
    const int NB = k <= 64 ? 1 : 2;
    s->upd_smem = res ? upd_res_smem_floats((int)segw) * 4 : upd_smem_floats(NB) * 4;
    void* fns[2];
    if (res) { fns[0] = (void*)update_res_kernel<true>; fns[1] = (void*)update_res_kernel<false>; }
    else {
      fns[0] = NB == 1 ? (void*)update_kernel<1, true> : (void*)update_kernel<2, true>;
      fns[1] = NB == 1 ? (void*)update_kernel<1, false> : (void*)update_kernel<2, false>;
    }
    for (void* fn : fns) {
      if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->upd_smem) != cudaSuccess)
        return cleanup(fail(GEIG_ERR_CUDA, "smem attribute for update kernel"));
      int o = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, UPD_THREADS, s->upd_smem) != cudaSuccess || o < 1)
        return cleanup(fail(GEIG_ERR_CUDA, "update kernel cannot be co-resident"));
    }
    const size_t pfl = res ? (size_t)upd_raw_floats_res(k) : upd_partial_floats(NB);
    // one partial row per CTA of any grid the fused step launches (<= #SM)
    if (cudaMalloc((void**)&s->partial, (size_t)std::max<int64_t>(G, s->nsm) * pfl * 4) != cudaSuccess ||
        cudaMalloc((void**)&s->raw, pfl * 4) != cudaSuccess)
      return cleanup(fail(GEIG_ERR_CUDA, "cudaMalloc gram partials"));
  }
  if (math != GEIG_MATH_F32) {
    geig_status st = tc::plan_create(s->tc, problem, dx, dy, k, math, max_rows, device);
    if (st != GEIG_OK) return cleanup(fail(st, "%s", tc::last_error()));
  }
  set_l2_window(s);
  if (cudaDeviceSynchronize() != cudaSuccess) return cleanup(fail(GEIG_ERR_CUDA, "create sync"));
  *out = s;
  return GEIG_OK;
}

extern "C" geig_status geig_destroy(geig_solver* s) {
  if (!s) return GEIG_OK;
  cudaSetDevice(s->device);
  if (s->tc.l2win.num_bytes > 0) cudaCtxResetPersistingL2Cache();   // no persisting lines outlive the arena
  for (void* p : {(void*)s->arena, (void*)s->precv, (void*)s->pflags,
                  (void*)s->gram, (void*)s->raw, (void*)s->partial,
                  (void*)s->Wx, (void*)s->Wy, (void*)s->ts, (void*)s->Wxb, (void*)s->Wyb, s->hX, s->hY,
                  (void*)s->zbuf, (void*)s->am, (void*)s->as, (void*)s->splitk, (void*)s->gshadow})
    if (p) cudaFree(p);
  if (s->ptab_dev) cudaFree((void*)s->ptab_dev);
  if (s->hX2) cudaFree(s->hX2);
  if (s->hY2) cudaFree(s->hY2);
  for (int i = 0; i < 2; ++i) {
    if (s->ev_loaded[i]) cudaEventDestroy(s->ev_loaded[i]);
    if (s->ev_free[i]) cudaEventDestroy(s->ev_free[i]);
  }
  if (s->copy_stream) cudaStreamDestroy(s->copy_stream);
  if (s->ptab_host) cudaFreeHost((void*)s->ptab_host);
  if (s->ptab_ev) cudaEventDestroy(s->ptab_ev);
  tc::plan_destroy(s->tc);
  delete s;
  return GEIG_OK;
}

// Persisting-L2 window over the state arena (V, [Bv], AV, BV, bf16 shadow)
// so the update phases find the state in L2 after the products have streamed
// the minibatch (> L2) through it.  The window is attached to the library's
// own cooperative launches only (a launch attribute; no stream attribute is
// changed).  Side effect (documented in geig.h): the device's persisting-L2
// set-aside is raised to the arena size (never lowered); geig_destroy resets
// the persisting lines.  Best effort: skipped when the device has no
// set-aside.
static void set_l2_window(geig_solver* s) {
  if (dev_knob("GEIG_NO_L2_PERSIST")) return;
  int max_persist = 0, max_window = 0;
  cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, s->device);
  cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, s->device);
  if (max_persist <= 0 || max_window <= 0) return;
  const size_t want = std::min<size_t>(s->arena_bytes, (size_t)max_persist);
  size_t cur = 0;
  cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
  if (cur < want) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
  cudaAccessPolicyWindow& w = s->tc.l2win;
  w.base_ptr = s->arena;
  w.num_bytes = std::min<size_t>(s->arena_bytes, (size_t)max_window);
  w.hitRatio = std::min(1.0f, (float)want / (float)w.num_bytes);
  w.hitProp = cudaAccessPropertyPersisting;
  w.missProp = cudaAccessPropertyStreaming;
  cudaGetLastError();   // best effort
}

extern "C" geig_status geig_set_stream(geig_solver* s, void* stream) {
  if (!s) return fail(GEIG_ERR_ARG, "solver is NULL");
  // the fused launches of one solver count the Gram reduction on a shared
  // counter in launch order: drain the old stream before switching
  if ((cudaStream_t)stream != s->stream) {
    CU(cudaSetDevice(s->device));
    CU(cudaStreamSynchronize(s->stream));
  }
  s->stream = (cudaStream_t)stream;
  return GEIG_OK;
}

extern "C" geig_status geig_sync(geig_solver* s) {
  if (!s) return fail(GEIG_ERR_ARG, "solver is NULL");
  CU(cudaSetDevice(s->device));
  CU(cudaStreamSynchronize(s->stream));
  return GEIG_OK;
}

// Column-owned mode: the gathered bf16 shadow [rank][hi|lo][k][W] of the
// whole state V (rank r's block = columns [r W, (r + 1) W)).
__global__ void pack_shadow_kernel(const float* __restrict__ V, __nv_bfloat16* __restrict__ g, int k, int64_t d,
                                   int64_t W) {
  const int64_t n = (int64_t)k * d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / d);
    const int64_t c = e - (int64_t)i * d, r = c / W, x = c - r * W;
    const float v = V[e];
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    __nv_bfloat16* blk = g + r * 2 * (int64_t)k * W;
    blk[(int64_t)i * W + x] = h;
    blk[(int64_t)k * W + (int64_t)i * W + x] = __float2bfloat16_rn(v - __bfloat162float(h));
  }
}

static geig_status refresh_gathered_shadow(geig_solver* s) {
  if (!s->gshadow) return GEIG_OK;
  pack_shadow_kernel<<<2 * s->nsm, 256, 0, s->stream>>>(s->V, s->gshadow, s->k, s->d, s->part_W);
  CHECK_LAUNCH();
  s->launches++;
  return GEIG_OK;
}

extern "C" geig_status geig_init_state(geig_solver* s, const float* G) {
  if (!s || !G) return fail(GEIG_ERR_ARG, "NULL argument");
  CU(cudaSetDevice(s->device));
  init_state_kernel<<<s->k, 256, 0, s->stream>>>(G, s->V, s->AUX, s->Vbf, s->d);
  CHECK_LAUNCH();
  s->launches++;
  return refresh_gathered_shadow(s);
}

extern "C" geig_status geig_set_state(geig_solver* s, const float* V, const float* AUX) {
  if (!s || !V) return fail(GEIG_ERR_ARG, "NULL argument");
  CU(cudaSetDevice(s->device));
  const size_t kd = (size_t)s->k * s->d;
  CU(cudaMemcpyAsync(s->V, V, kd * 4, cudaMemcpyDeviceToDevice, s->stream));
  if (AUX) CU(cudaMemcpyAsync(s->AUX, AUX, kd * 4, cudaMemcpyDeviceToDevice, s->stream));
  f32_to_bf16_kernel<<<256, 256, 0, s->stream>>>(s->V, s->Vbf, (int64_t)kd);   // hi + lo planes
  CHECK_LAUNCH();
  s->launches++;
  return refresh_gathered_shadow(s);
}

extern "C" geig_status geig_get(geig_solver* s, float* V, float* AUX) {
  if (!s) return fail(GEIG_ERR_ARG, "solver is NULL");
  CU(cudaSetDevice(s->device));
  const size_t kd = (size_t)s->k * s->d;
  if (V && s->part_world > 1) {
    // column-owned: only the own block is current and the retraction needs
    // the row norms over every rank's columns — return the raw v''
    CU(cudaMemcpyAsync(V, s->V, kd * 4, cudaMemcpyDeviceToDevice, s->stream));
  } else if (V) {
    // the state holds v'' (retraction folded into the next update): return v''/||v''||
    normalize_rows_kernel<<<s->k, 256, 0, s->stream>>>(s->V, V, s->d);
    CHECK_LAUNCH();
    s->launches++;
  }
  if (AUX) CU(cudaMemcpyAsync(AUX, s->AUX, kd * 4, cudaMemcpyDeviceToDevice, s->stream));
  return GEIG_OK;
}

extern "C" geig_status geig_get_gram(geig_solver* s, float* GA, float* GB, float* GC) {
  if (!s) return fail(GEIG_ERR_ARG, "solver is NULL");
  CU(cudaSetDevice(s->device));
  const size_t kk = (size_t)s->k * s->k;
  if (GA) CU(cudaMemcpyAsync(GA, s->gram, kk * 4, cudaMemcpyDeviceToDevice, s->stream));
  if (GB) CU(cudaMemcpyAsync(GB, s->gram + kk, kk * 4, cudaMemcpyDeviceToDevice, s->stream));
  if (GC) CU(cudaMemcpyAsync(GC, s->gram + 2 * kk, kk * 4, cudaMemcpyDeviceToDevice, s->stream));
  return GEIG_OK;
}

// ---------------------------------------------------------------------------
// products
// ---------------------------------------------------------------------------

// SIMT (FFMA) product launch.  When the M x N tile grid leaves most SMs idle
// and K is long (the backward X^T Z of small d with a large batch), K is
// split over gridDim.z slices into s->splitk partials and reduced in fixed
// order by simt_splitk_reduce (two launches, deterministic).
template <typename TA, bool A_K, bool B_K, class Epi>
static geig_status launch_simt(geig_solver* s, const TA* A, int64_t lda, const float* B, int64_t ldb,
                               int M, int N, int64_t kbeg, int64_t kend, Epi epi) {
  if (M <= 0 || N <= 0) return GEIG_OK;
  dim3 grid((M + SG_BM - 1) / SG_BM, (N + SG_BN - 1) / SG_BN);
  const int tiles = (int)(grid.x * grid.y);
  const int64_t K = kend - kbeg;
  int splits = 1;
  while (tiles * splits * 2 <= 2 * s->nsm && K / (splits * 2) >= 512) splits *= 2;
  if (splits > 1) {
    const size_t need = (size_t)splits * M * N;
    if (need > s->splitk_floats) {
      if (s->splitk) cudaFree(s->splitk);
      s->splitk = nullptr;
      s->splitk_floats = 0;
      CU(cudaMalloc((void**)&s->splitk, need * sizeof(float)));
      s->splitk_floats = need;
    }
    int64_t kchunk = (K + splits - 1) / splits;
    kchunk = (kchunk + SG_BK - 1) / SG_BK * SG_BK;
    grid.z = (unsigned)splits;
    simt_gemm_kernel<TA, float, A_K, B_K, Epi><<<grid, 256, 0, s->stream>>>(A, lda, B, ldb, M, N, kbeg, kend, epi,
                                                                           s->splitk, kchunk);
    CHECK_LAUNCH();
    const int rb = (int)std::min<int64_t>(2 * s->nsm, ((int64_t)M * N + 255) / 256);
    simt_splitk_reduce<Epi><<<rb, 256, 0, s->stream>>>(s->splitk, M, N, splits, epi);
    CHECK_LAUNCH();
    s->launches += 2;
    return GEIG_OK;
  }
  simt_gemm_kernel<TA, float, A_K, B_K, Epi><<<grid, 256, 0, s->stream>>>(A, lda, B, ldb, M, N, kbeg, kend, epi);
  CHECK_LAUNCH();
  s->launches++;
  return GEIG_OK;
}

template <typename T>
static geig_status products_cca_simt(geig_solver* s, const T* X, const T* Y, int64_t b, float scale,
                                     float* AV, float* BV) {
  const int h = (int)(b / 2);
  const int k = s->k;
  const int64_t ldw = b;
  geig_status st;
  // forward: Z_x = X V_x^T (b x k), scattered into the backward operands
  st = launch_simt<T, true, true>(s, X, s->dx, s->V, s->d, (int)(2 * h), k, 0, s->dx,
                                  EpiForward{s->Wy, s->Wx, ldw, h});
  if (st) return st;
  st = launch_simt<T, true, true>(s, Y, s->dy, s->V + s->dx, s->d, (int)(2 * h), k, 0, s->dy,
                                  EpiForward{s->Wx, s->Wy, ldw, h});
  if (st) return st;
  // backward: AV_x = X1^T W_x[:, :h], BV_x = X2^T W_x[:, h:2h], same for y
  for (int view = 0; view < 2; ++view) {
    const T* Xv = view == 0 ? X : Y;
    const int64_t dv = view == 0 ? s->dx : s->dy;
    const int64_t off = view == 0 ? 0 : s->dx;
    const float* W = view == 0 ? s->Wx : s->Wy;
    st = launch_simt<T, false, true>(s, Xv, dv, W, ldw, (int)dv, k, 0, h,
                                     EpiTransposeScale{AV + off, s->d, scale});
    if (st) return st;
    st = launch_simt<T, false, true>(s, Xv, dv, W, ldw, (int)dv, k, h, 2 * h,
                                     EpiTransposeScale{BV + off, s->d, scale});
    if (st) return st;
  }
  return GEIG_OK;
}

static bool fused_ok(const geig_solver* s, const void* X, const void* Y);
static UpdateArgs update_args(geig_solver* s, double eta, double gamma);
static void advance_variant_state(geig_solver* s, int64_t n);

extern "C" geig_status geig_products_cca(geig_solver* s, const void* X, const void* Y, int64_t b,
                                         float scale, float* AV, float* BV) {
  if (!s || !X || !Y || !AV || !BV) return fail(GEIG_ERR_ARG, "NULL argument");
  if (s->problem != GEIG_CCA) return fail(GEIG_ERR_STATE, "solver is not a CCA solver");
  if (b < 2 || b > s->max_rows) return fail(GEIG_ERR_ARG, "b=%lld outside [2, max_rows=%lld]",
                                            (long long)b, (long long)s->max_rows);
  CU(cudaSetDevice(s->device));
  if (s->math == GEIG_MATH_F32) {
    if (s->dtype == GEIG_DATA_F32)
      return products_cca_simt(s, (const float*)X, (const float*)Y, b, scale, AV, BV);
    return products_cca_simt(s, (const __nv_bfloat16*)X, (const __nv_bfloat16*)Y, b, scale, AV, BV);
  }
  if (fused_ok(s, X, Y) && !s->opt_staged) {
    // phases F, S, B of the fused step kernel in one launch, AV / BV to the
    // caller's buffers (e.g. before a cross-GPU all-reduce and geig_update)
    geig_status st = tc::fused_cca_step(s->tc, &X, &Y, 1, b, scale, s->Vbf, AV, BV, update_args(s, 0.0, 0.0),
                                        s->upd_grid, s->upd_smem, s->stream, /*products_only=*/true);
    if (st) return fail(st, "%s", tc::last_error());
    s->launches++;
    return GEIG_OK;
  }
  int64_t nl = 0;
  geig_status st = tc::products_cca(s->tc, X, Y, b, scale, s->Vbf, s->V, AV, BV, s->stream, &nl);
  s->launches += nl;
  if (st) return fail(st, "%s", tc::last_error());
  return GEIG_OK;
}

extern "C" int64_t geig_table_floats(const geig_solver* s) {
  if (!s) return 0;
  const int64_t ntri = (int64_t)s->k * (s->k + 1) / 2;
  return (ntri + s->k + 3) & ~(int64_t)3;
}

extern "C" geig_status geig_products_cca_tables(geig_solver* s, const void* X, const void* Y, int64_t b,
                                                float scale, float* AV, float* BV, float* T) {
  if (!s || !X || !Y || !AV || !BV || !T) return fail(GEIG_ERR_ARG, "NULL argument");
  if (s->problem != GEIG_CCA) return fail(GEIG_ERR_STATE, "solver is not a CCA solver");
  if (b < 2 || b > s->max_rows) return fail(GEIG_ERR_ARG, "b=%lld outside [2, max_rows=%lld]",
                                            (long long)b, (long long)s->max_rows);
  if (!fused_ok(s, X, Y))
    return fail(GEIG_ERR_UNSUPPORTED, "products with tables need the fused path (bf16 math, k <= 64, d %% 4 == 0)");
  CU(cudaSetDevice(s->device));
  UpdateArgs a = update_args(s, 0.0, 0.0);
  a.raw_a = T;
  geig_status st = tc::fused_cca_step(s->tc, &X, &Y, 1, b, scale, s->Vbf, AV, BV, a, s->upd_grid, s->upd_smem,
                                      s->stream, /*products_only=*/true, /*tables=*/true);
  if (st) return fail(st, "%s", tc::last_error());
  s->launches++;
  return GEIG_OK;
}

extern "C" geig_status geig_update_tables(geig_solver* s, const float* AV, const float* BV, const float* T,
                                          double eta, double gamma) {
  if (!s || !AV || !BV || !T) return fail(GEIG_ERR_ARG, "NULL argument");
  if (!s->upd_res || s->d % 4 != 0) return fail(GEIG_ERR_UNSUPPORTED, "update from tables needs k <= 64, d %% 4 == 0");
  CU(cudaSetDevice(s->device));
  UpdateArgs a = update_args(s, eta, gamma);
  a.AV = AV; a.BV = BV;
  a.raw_a = const_cast<float*>(T);
  a.pre_reduced = 1;
  if ((s->math == GEIG_MATH_BF16 || s->math == GEIG_MATH_BF16X2) && !dev_knob("GEIG_NO_FUSED") &&
      ((uintptr_t)AV | (uintptr_t)BV) % 16 == 0) {
    // phase U of the fused kernel alone (TMA-staged tiles, early table staging)
    const void* none[1] = {nullptr};
    geig_status st = tc::fused_cca_step(s->tc, none, none, 1, 0, 1.f, s->Vbf, const_cast<float*>(AV),
                                        const_cast<float*>(BV), a, s->upd_grid, s->upd_smem, s->stream,
                                        /*products_only=*/false, /*tables=*/false, /*update_only=*/true);
    if (st) return fail(st, "%s", tc::last_error());
    s->launches++;
    s->fused_last = false;
    advance_variant_state(s, 1);
    return GEIG_OK;
  }
  void* args[] = {&a};
  const bool vec = ((uintptr_t)AV | (uintptr_t)BV) % 16 == 0;
  void* fn = vec ? (void*)update_res_kernel<true> : (void*)update_res_kernel<false>;
  CU(tc::launch_coop(fn, dim3(s->upd_grid), dim3(UPD_THREADS), args, s->upd_smem, s->stream, s->tc.l2win));
  s->launches++;
  s->fused_last = false;
  advance_variant_state(s, 1);
  return GEIG_OK;
}

extern "C" geig_status geig_products_dense(geig_solver* s, const void* A, const void* B, int64_t r0,
                                           int64_t r1, float* AV, float* BV) {
  if (!s || !A || !B || !AV || !BV) return fail(GEIG_ERR_ARG, "NULL argument");
  if (s->problem != GEIG_DENSE) return fail(GEIG_ERR_STATE, "solver is not a dense solver");
  if (r0 < 0 || r1 > s->d || r0 >= r1) return fail(GEIG_ERR_ARG, "bad row range");
  CU(cudaSetDevice(s->device));
  const int M = (int)(r1 - r0);
  if (s->math == GEIG_MATH_F32) {
    geig_status st;
    if (s->dtype == GEIG_DATA_F32) {
      st = launch_simt<float, true, true>(s, (const float*)A, s->d, s->V, s->d, M, s->k, 0, s->d,
                                          EpiTransposeScale{AV + r0, s->d, 1.f});
      if (st) return st;
      return launch_simt<float, true, true>(s, (const float*)B, s->d, s->V, s->d, M, s->k, 0, s->d,
                                            EpiTransposeScale{BV + r0, s->d, 1.f});
    }
    st = launch_simt<__nv_bfloat16, true, true>(s, (const __nv_bfloat16*)A, s->d, s->V, s->d, M, s->k, 0,
                                                s->d, EpiTransposeScale{AV + r0, s->d, 1.f});
    if (st) return st;
    return launch_simt<__nv_bfloat16, true, true>(s, (const __nv_bfloat16*)B, s->d, s->V, s->d, M, s->k, 0,
                                                  s->d, EpiTransposeScale{BV + r0, s->d, 1.f});
  }
  int64_t nl = 0;
  geig_status st = tc::products_dense(s->tc, A, B, r0, r1, s->Vbf, s->V, AV, BV, s->stream, &nl);
  s->launches += nl;
  if (st) return fail(st, "%s", tc::last_error());
  return GEIG_OK;
}

// ---------------------------------------------------------------------------
// update
// ---------------------------------------------------------------------------

extern "C" geig_status geig_update(geig_solver* s, const float* AV, const float* BV, double eta,
                                   double gamma) {
  if (!s || !AV || !BV) return fail(GEIG_ERR_ARG, "NULL argument");
  CU(cudaSetDevice(s->device));
  UpdateArgs a = update_args(s, eta, gamma);
  a.AV = AV; a.BV = BV;
  const bool vec = (s->d % 4 == 0) && (((uintptr_t)AV | (uintptr_t)BV) % 16 == 0);
  if (!s->upd_res && s->opt_gram_tc && s->tc.ready && (s->math == GEIG_MATH_TF32 || s->math == GEIG_MATH_3XTF32) &&
      vec && (s->d + 31) / 32 >= s->upd_grid) {
    // k > 64: the G'^A, G'^C partial rows on the tensor cores (one split per
    // update CTA), the update's phase 1 only forms the diagonals
    int64_t nl = 0;
    const int KP = 128;
    geig_status st = tc::gram_dense_tc(s->tc, s->V, AV, s->AUX, s->partial, (int64_t)upd_partial_floats(2), KP,
                                       s->upd_grid, s->stream, &nl);
    s->launches += nl;
    if (st) return fail(st, "%s", tc::last_error());
    a.gram_tc = 1;
  }
  void* args[] = {&a};
  void* fn;
  if (s->upd_res) fn = vec ? (void*)update_res_kernel<true> : (void*)update_res_kernel<false>;
  else if (s->k <= 64) fn = vec ? (void*)update_kernel<1, true> : (void*)update_kernel<1, false>;
  else fn = vec ? (void*)update_kernel<2, true> : (void*)update_kernel<2, false>;
  CU(tc::launch_coop(fn, dim3(s->upd_grid), dim3(UPD_THREADS), args, s->upd_smem, s->stream, s->tc.l2win));
  s->launches++;
  advance_variant_state(s, 1);
  return GEIG_OK;
}

static bool fused_ok(const geig_solver* s, const void* X, const void* Y) {
  if ((s->math != GEIG_MATH_BF16 && s->math != GEIG_MATH_BF16X2) || !s->upd_res || s->d % 4 != 0) return false;
  if (dev_knob("GEIG_NO_FUSED")) return false;
  return (((uintptr_t)X | (uintptr_t)Y) % 16) == 0;
}

static UpdateArgs update_args(geig_solver* s, double eta, double gamma) {
  UpdateArgs a{};
  a.V = s->V; a.AUX = s->AUX; a.AV = s->AV; a.BV = s->BV;
  a.Vbf = s->Vbf; a.partial = s->partial; a.raw = s->raw; a.gram = s->gram;
  a.k = s->k; a.d = s->d; a.segw = s->upd_segw;
  a.eta = (float)eta; a.gamma = (float)gamma; a.rho = s->rho; a.ts = s->ts;
  a.smooth = s->smooth; a.zbuf = s->zbuf; a.zpar = s->zpar;
  a.lnrho = logf(std::max(s->rho, 1e-30f)); a.lnnu = logf(std::max(s->nu, 1e-30f));
  a.adam = s->adam; a.am = s->am; a.as = s->as; a.b1 = s->b1; a.b2 = s->b2; a.eps = s->eps;
  a.adam_t0 = s->adam_t;
  return a;
}

// the variant state advances with every update launched (n steps)
static void advance_variant_state(geig_solver* s, int64_t n) {
  s->zpar = (int)((s->zpar + n) & 1);
  s->adam_t += n;
}

// ---------------------------------------------------------------------------
// one-CTA small-problem step (small_step.cuh): fp32 FFMA math, k <= 16, the
// state (4 k x d fp32 arrays) and a chunk of rows (CCA) or A and B (dense)
// resident in one SM's shared memory.  Otherwise the staged path runs.
// ---------------------------------------------------------------------------
struct SmallPlan {
  bool ok = false;
  int KP = 8, rc = 0, dpad = 0, RG = 1;
  int C = 1, bq = 0, dq = 0;                           // cluster CTAs, rows / columns per CTA
  size_t smem = 0;
};

static SmallPlan small_plan(const geig_solver* s, int64_t b) {
  SmallPlan pl;
  if (!s->opt_small || s->math != GEIG_MATH_F32 || s->k > 16 || s->adam) return pl;
  const size_t es = s->dtype == GEIG_DATA_BF16 ? 2 : 4;
  const int E = (int)(16 / es);
  const int64_t d = s->d;
  pl.KP = s->k <= 8 ? 8 : 16;
  if (d % E != 0 || s->dx % E != 0 || (pl.KP / 4) * ((d / 4 + 7) / 8) * 8 > SM_THREADS) return pl;
  pl.dpad = (int)d;
  // backward tiles: (KP / 4) player quads x 8-quad column groups, RG row groups
  const int tiles = (pl.KP / 4) * (int)((d / 4 + 7) / 8) * 8;
  pl.RG = 1;
  while (pl.RG < 4 && tiles * pl.RG * 2 <= SM_THREADS) pl.RG *= 2;
  if (s->problem == GEIG_DENSE) {
    pl.rc = (int)((d + 3) / 4 * 4);                    // A, B resident: d rows each (rounded to 4)
    pl.smem = small_smem_bytes(true, pl.KP, (int)d, s->k, pl.rc, pl.dpad, es);
    pl.ok = pl.smem <= (size_t)SM_SMEM_MAX;
    return pl;
  }
  // a cluster of C CTAs splits the rows of every batch (and owns column
  // blocks of the update): auto = the largest power of 2 <= 8 leaving >= 64
  // rows and >= 16 columns per CTA
  if (s->opt_small_cluster > 0) pl.C = s->opt_small_cluster;
  else
    while (pl.C < 8 && b / (2 * pl.C) >= 64 && d / (2 * pl.C) >= 16) pl.C *= 2;
  pl.bq = (int)(((b + pl.C - 1) / pl.C + 3) / 4 * 4);
  pl.dq = (int)(((d + pl.C - 1) / pl.C + 3) / 4 * 4);
  if ((int64_t)(pl.C - 1) * pl.bq >= b || (int64_t)(pl.C - 1) * pl.dq >= d) { pl.C = 1; pl.bq = (int)b; pl.dq = (int)d; }
  const int b4 = (int)((pl.bq + 3) / 4 * 4);
  for (int rc = std::min(b4, 1024); rc >= 4; rc -= 4) {
    const size_t need = small_smem_bytes(false, pl.KP, (int)d, s->k, rc, pl.dpad, es);
    if (need <= (size_t)SM_SMEM_MAX) { pl.rc = rc; pl.smem = need; pl.ok = true; break; }
  }
  return pl;
}

// nsteps steps of the small path; batches: X[i], Y[i] (CCA) or A, B (dense, X[0], Y[0])
static geig_status small_launch(geig_solver* s, const SmallPlan& pl, const void* const* X, const void* const* Y,
                                int64_t nsteps, int64_t b, double eta, double gamma) {
  SmallParams p{};
  const bool dense = s->problem == GEIG_DENSE;
  p.dense = dense ? 1 : 0;
  p.k = s->k; p.KPr = pl.KP;
  p.dx = (int)s->dx; p.dy = (int)s->dy; p.d = (int)s->d;
  p.b = dense ? 0 : (int)b;
  p.h = (int)(b / 2);
  p.nsteps = (int)nsteps;
  p.x0 = X[0]; p.y0 = Y[0];
  p.xs = nullptr;
  bool same = true;
  for (int64_t i = 1; i < nsteps && same && !dense; ++i) same = X[i] == X[0] && Y[i] == Y[0];
  if (!same) {
    if (!s->ptab_dev) {
      CU(cudaMalloc((void**)&s->ptab_dev, (size_t)tc::TC_RUN_CHUNK * 2 * sizeof(void*)));
      CU(cudaMallocHost((void**)&s->ptab_host, (size_t)tc::TC_RUN_CHUNK * 2 * sizeof(void*)));
      CU(cudaEventCreateWithFlags(&s->ptab_ev, cudaEventDisableTiming));
    }
    CU(cudaEventSynchronize(s->ptab_ev));               // the previous run's copy out of the staging buffer is done
    for (int64_t i = 0; i < nsteps; ++i) { s->ptab_host[2 * i] = X[i]; s->ptab_host[2 * i + 1] = Y[i]; }
    CU(cudaMemcpyAsync((void*)s->ptab_dev, (const void*)s->ptab_host, (size_t)nsteps * 2 * sizeof(void*),
                       cudaMemcpyHostToDevice, s->stream));
    CU(cudaEventRecord(s->ptab_ev, s->stream));
    p.xs = s->ptab_dev;
  }
  p.scale = dense ? 1.f : 1.0f / (float)(b / 2);
  p.eta = (float)eta; p.gamma = (float)gamma; p.rho = s->rho;
  p.V = s->V; p.AUX = s->AUX; p.AV = s->AV; p.BV = s->BV; p.Vbf = s->Vbf; p.gram = s->gram;
  p.smooth = s->smooth; p.zbuf = s->zbuf; p.zpar = s->zpar;
  p.lnrho = logf(std::max(s->rho, 1e-30f)); p.lnnu = logf(std::max(s->nu, 1e-30f));
  p.rc = pl.rc; p.dpad = pl.dpad; p.RG = pl.RG;
  p.cl = dense ? 1 : pl.C;
  p.bq = dense ? 0 : pl.bq;
  p.dq = dense ? p.d : pl.dq;
  p.ts = nullptr;
  p.prof = tc::dbg_ptr();   // developer hook (geig_debug_set_tc_stamps): per-phase cycles
  const bool bf = s->dtype == GEIG_DATA_BF16;
  const void* fn = bf ? (pl.KP == 8 ? (const void*)small_step_kernel<__nv_bfloat16, 8>
                                    : (const void*)small_step_kernel<__nv_bfloat16, 16>)
                      : (pl.KP == 8 ? (const void*)small_step_kernel<float, 8> : (const void*)small_step_kernel<float, 16>);
  static std::atomic<uint64_t> attr[4];
  const int ai = (bf ? 2 : 0) + (pl.KP == 8 ? 0 : 1);
  CU(set_smem_attr_once(attr[ai], fn, SM_SMEM_MAX));
  void* args[] = {&p};
  if (p.cl > 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.cl);
    cfg.blockDim = dim3(SM_THREADS);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = s->stream;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = (unsigned)p.cl; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    CU(cudaLaunchKernelExC(&cfg, fn, args));
  } else {
    CU(cudaLaunchKernel(fn, dim3(1), dim3(SM_THREADS), args, pl.smem, s->stream));
  }
  s->launches++;
  s->fused_last = false;
  advance_variant_state(s, nsteps);
  return GEIG_OK;
}

static bool aligned16(const void* p) { return ((uintptr_t)p % 16) == 0; }

extern "C" geig_status geig_step_cca(geig_solver* s, const void* X, const void* Y, int64_t b, double eta,
                                     double gamma) {
  if (!s) return fail(GEIG_ERR_ARG, "solver is NULL");
  if (s->problem == GEIG_CCA && b >= 2 && b <= s->max_rows && X && Y && aligned16(X) && aligned16(Y)) {
    const SmallPlan pl = small_plan(s, b);
    if (pl.ok) {
      CU(cudaSetDevice(s->device));
      return small_launch(s, pl, &X, &Y, 1, b, eta, gamma);
    }
  }
  if (s->problem == GEIG_CCA && b >= 2 && b <= s->max_rows && X && Y && fused_ok(s, X, Y)) {
    // whole step in one persistent cooperative launch (fused_step.cuh)
    CU(cudaSetDevice(s->device));
    const UpdateArgs a = update_args(s, eta, gamma);
    geig_status st = tc::fused_cca_step(s->tc, &X, &Y, 1, b, 1.0f / (float)(b / 2), s->Vbf, s->AV, s->BV, a,
                                        s->upd_grid, s->upd_smem, s->stream, false, false, false, nullptr,
                                        s->nsm & ~1);
    if (st) return fail(st, "%s", tc::last_error());
    s->launches++;
    s->fused_last = true;
    advance_variant_state(s, 1);
    return GEIG_OK;
  }
  geig_status st = geig_products_cca(s, X, Y, b, 1.0f / (float)(b / 2), s->AV, s->BV);
  if (st) return st;
  s->fused_last = false;
  return geig_update(s, s->AV, s->BV, eta, gamma);
}

extern "C" geig_status geig_run_cca(geig_solver* s, const void* const* X, const void* const* Y, int64_t b,
                                    int64_t nsteps, double eta, double gamma) {
  if (!s || !X || !Y) return fail(GEIG_ERR_ARG, "NULL argument");
  if (nsteps < 0 || nsteps > (1 << 20)) return fail(GEIG_ERR_ARG, "nsteps = %lld out of range", (long long)nsteps);
  if (nsteps == 0) return GEIG_OK;
  bool fused = s->problem == GEIG_CCA && b >= 2 && b <= s->max_rows;
  {
    // one-CTA small path: up to TC_RUN_CHUNK steps per launch
    const SmallPlan pl = fused ? small_plan(s, b) : SmallPlan{};
    bool small = pl.ok;
    for (int64_t i = 0; small && i < nsteps; ++i) small = X[i] && Y[i] && aligned16(X[i]) && aligned16(Y[i]);
    if (small) {
      CU(cudaSetDevice(s->device));
      for (int64_t i0 = 0; i0 < nsteps; i0 += tc::TC_RUN_CHUNK) {
        const int64_t n = std::min<int64_t>(tc::TC_RUN_CHUNK, nsteps - i0);
        geig_status st = small_launch(s, pl, X + i0, Y + i0, n, b, eta, gamma);
        if (st) return st;
      }
      return GEIG_OK;
    }
  }
  for (int64_t i = 0; fused && i < nsteps; ++i) fused = X[i] && Y[i] && fused_ok(s, X[i], Y[i]);
  if (!fused) {
    for (int64_t i = 0; i < nsteps; ++i) {
      geig_status st = geig_step_cca(s, X[i], Y[i], b, eta, gamma);
      if (st) return st;
    }
    return GEIG_OK;
  }
  // Alg. 2's loop over t in persistent cooperative launches of up to
  // TC_RUN_CHUNK steps each (fused_step.cuh)
  CU(cudaSetDevice(s->device));
  for (int64_t i0 = 0; i0 < nsteps; i0 += tc::TC_RUN_CHUNK) {
    const int n = (int)std::min<int64_t>(tc::TC_RUN_CHUNK, nsteps - i0);
    geig_status st = tc::fused_cca_step(s->tc, X + i0, Y + i0, n, b, 1.0f / (float)(b / 2), s->Vbf, s->AV, s->BV,
                                        update_args(s, eta, gamma), s->upd_grid, s->upd_smem, s->stream, false,
                                        false, false, nullptr, s->nsm & ~1);
    if (st) return fail(st, "%s", tc::last_error());
    s->launches++;
    advance_variant_state(s, n);
  }
  s->fused_last = true;
  return GEIG_OK;
}

extern "C" geig_status geig_step_dense(geig_solver* s, const void* A, const void* B, double eta,
                                       double gamma) {
  if (!s) return fail(GEIG_ERR_ARG, "solver is NULL");
  return geig_run_dense(s, A, B, 1, eta, gamma);
}

extern "C" geig_status geig_run_dense(geig_solver* s, const void* A, const void* B, int64_t nsteps, double eta,
                                      double gamma) {
  if (!s || !A || !B) return fail(GEIG_ERR_ARG, "NULL argument");
  if (s->problem != GEIG_DENSE) return fail(GEIG_ERR_STATE, "solver is not a dense solver");
  if (nsteps < 0 || nsteps > (1 << 30)) return fail(GEIG_ERR_ARG, "nsteps = %lld out of range", (long long)nsteps);
  if (nsteps == 0) return GEIG_OK;
  const SmallPlan pl = small_plan(s, 0);
  if (pl.ok && aligned16(A) && aligned16(B)) {
    // A, B resident in one SM's shared memory for the whole launch
    CU(cudaSetDevice(s->device));
    for (int64_t i0 = 0; i0 < nsteps; i0 += tc::TC_RUN_CHUNK) {
      const int64_t n = std::min<int64_t>(tc::TC_RUN_CHUNK, nsteps - i0);
      geig_status st = small_launch(s, pl, &A, &B, n, 0, eta, gamma);
      if (st) return st;
    }
    return GEIG_OK;
  }
  for (int64_t i = 0; i < nsteps; ++i) {
    geig_status st = geig_products_dense(s, A, B, 0, s->d, s->AV, s->BV);
    if (st) return st;
    st = geig_update(s, s->AV, s->BV, eta, gamma);
    if (st) return st;
  }
  return GEIG_OK;
}

extern "C" geig_status geig_step_cca_host(geig_solver* s, const void* X_host, const void* Y_host, int64_t b,
                                          double eta, double gamma, float* ga_host, int64_t* h2d,
                                          int64_t* d2h) {
  if (!s || !X_host || !Y_host) return fail(GEIG_ERR_ARG, "NULL argument");
  if (s->problem != GEIG_CCA) return fail(GEIG_ERR_STATE, "solver is not a CCA solver");
  if (b < 2 || b > s->max_rows) return fail(GEIG_ERR_ARG, "bad b");
  CU(cudaSetDevice(s->device));
  const size_t es = s->dtype == GEIG_DATA_BF16 ? 2 : 4;
  if (!s->hX) {
    CU(cudaMalloc(&s->hX, (size_t)s->max_rows * s->dx * es));
    CU(cudaMalloc(&s->hY, (size_t)s->max_rows * s->dy * es));
  }
  const size_t bx = (size_t)b * s->dx * es, by = (size_t)b * s->dy * es;
  CU(cudaMemcpyAsync(s->hX, X_host, bx, cudaMemcpyHostToDevice, s->stream));
  CU(cudaMemcpyAsync(s->hY, Y_host, by, cudaMemcpyHostToDevice, s->stream));
  geig_status st = geig_step_cca(s, s->hX, s->hY, b, eta, gamma);
  if (st) return st;
  const size_t gb = (size_t)s->k * s->k * 4;
  if (ga_host) CU(cudaMemcpyAsync(ga_host, s->gram, gb, cudaMemcpyDeviceToHost, s->stream));
  CU(cudaStreamSynchronize(s->stream));
  if (h2d) *h2d = (int64_t)(bx + by);
  if (d2h) *d2h = ga_host ? (int64_t)gb : 0;
  return GEIG_OK;
}

extern "C" geig_status geig_run_cca_host(geig_solver* s, const void* const* X_host, const void* const* Y_host,
                                         int64_t b, int64_t nsteps, double eta, double gamma, float* ga_host,
                                         int64_t* h2d, int64_t* d2h) {
  if (!s || !X_host || !Y_host) return fail(GEIG_ERR_ARG, "NULL argument");
  if (s->problem != GEIG_CCA) return fail(GEIG_ERR_STATE, "solver is not a CCA solver");
  if (b < 2 || b > s->max_rows) return fail(GEIG_ERR_ARG, "bad b");
  if (nsteps < 0) return fail(GEIG_ERR_ARG, "nsteps < 0");
  CU(cudaSetDevice(s->device));
  const size_t es = s->dtype == GEIG_DATA_BF16 ? 2 : 4;
  const size_t bx = (size_t)b * s->dx * es, by = (size_t)b * s->dy * es;
  if (!s->hX) {
    CU(cudaMalloc(&s->hX, (size_t)s->max_rows * s->dx * es));
    CU(cudaMalloc(&s->hY, (size_t)s->max_rows * s->dy * es));
  }
  if (!s->hX2) {
    CU(cudaMalloc(&s->hX2, (size_t)s->max_rows * s->dx * es));
    CU(cudaMalloc(&s->hY2, (size_t)s->max_rows * s->dy * es));
    CU(cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CU(cudaEventCreateWithFlags(&s->ev_loaded[i], cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&s->ev_free[i], cudaEventDisableTiming));
    }
  }
  void* dX[2] = {s->hX, s->hX2};
  void* dY[2] = {s->hY, s->hY2};
  const size_t gb = (size_t)s->k * s->k * 4;
  // the staging pairs are free when this call starts (previous work on the solver's stream)
  for (int i = 0; i < 2; ++i) CU(cudaEventRecord(s->ev_free[i], s->stream));
  for (int64_t t = 0; t < nsteps; ++t) {
    const int q = (int)(t & 1);
    // copy engine: batch t into pair q once step t - 2 has released it
    CU(cudaStreamWaitEvent(s->copy_stream, s->ev_free[q], 0));
    CU(cudaMemcpyAsync(dX[q], X_host[t], bx, cudaMemcpyHostToDevice, s->copy_stream));
    CU(cudaMemcpyAsync(dY[q], Y_host[t], by, cudaMemcpyHostToDevice, s->copy_stream));
    CU(cudaEventRecord(s->ev_loaded[q], s->copy_stream));
    // compute: step t (overlaps the copy of batch t + 1), then its Gram table back
    CU(cudaStreamWaitEvent(s->stream, s->ev_loaded[q], 0));
    geig_status st = geig_step_cca(s, dX[q], dY[q], b, eta, gamma);
    if (st) return st;
    CU(cudaEventRecord(s->ev_free[q], s->stream));
    if (ga_host) CU(cudaMemcpyAsync(ga_host, s->gram, gb, cudaMemcpyDeviceToHost, s->stream));
  }
  CU(cudaStreamSynchronize(s->stream));
  if (h2d) *h2d = (int64_t)(bx + by) * nsteps;
  if (d2h) *d2h = ga_host ? (int64_t)gb * nsteps : 0;
  return GEIG_OK;
}

extern "C" geig_status geig_set_smooth(geig_solver* s, double nu) {
  if (!s) return fail(GEIG_ERR_ARG, "solver is NULL");
  if (!(nu > 0.0)) { s->smooth = 0; return GEIG_OK; }
  if (!(nu > (double)s->rho) || !(s->rho > 0.f))
    return fail(GEIG_ERR_ARG, "Alg. 3 needs 0 < rho < nu (rho=%g, nu=%g)", (double)s->rho, nu);
  if (!s->upd_res) return fail(GEIG_ERR_UNSUPPORTED, "Alg. 3 needs the resident update (k <= 64)");
  CU(cudaSetDevice(s->device));
  if (!s->zbuf) CU(cudaMalloc((void**)&s->zbuf, 2 * 64 * sizeof(float)));
  CU(cudaMemsetAsync(s->zbuf, 0, 2 * 64 * sizeof(float), s->stream));   // Alg. 3 l.4: z_i = 0
  s->zpar = 0;
  s->nu = (float)nu;
  s->smooth = 1;
  return GEIG_OK;
}

extern "C" geig_status geig_smooth_state(geig_solver* s, const float* z_in, float* z_out) {
  if (!s) return fail(GEIG_ERR_ARG, "solver is NULL");
  if (!s->smooth) return fail(GEIG_ERR_STATE, "Alg. 3 is not enabled (geig_set_smooth)");
  CU(cudaSetDevice(s->device));
  float* cur = s->zbuf + (s->zpar & 1) * 64;
  if (z_in) CU(cudaMemcpyAsync(cur, z_in, (size_t)s->k * sizeof(float), cudaMemcpyDeviceToDevice, s->stream));
  if (z_out) CU(cudaMemcpyAsync(z_out, cur, (size_t)s->k * sizeof(float), cudaMemcpyDeviceToDevice, s->stream));
  return GEIG_OK;
}

extern "C" geig_status geig_set_adam(geig_solver* s, double b1, double b2, double eps) {
  if (!s) return fail(GEIG_ERR_ARG, "solver is NULL");
  if (b1 < 0.0) { s->adam = 0; return GEIG_OK; }
  if (!(b1 < 1.0) || !(b2 >= 0.0 && b2 < 1.0) || !(eps >= 0.0)) return fail(GEIG_ERR_ARG, "bad Adam parameters");
  if (!s->upd_res || s->d % 4 != 0)
    return fail(GEIG_ERR_UNSUPPORTED, "Adam needs the resident update (k <= 64) and d %% 4 == 0");
  CU(cudaSetDevice(s->device));
  const size_t kd = (size_t)s->k * s->d;
  if (!s->am) CU(cudaMalloc((void**)&s->am, kd * sizeof(float)));
  if (!s->as) CU(cudaMalloc((void**)&s->as, kd * sizeof(float)));
  CU(cudaMemsetAsync(s->am, 0, kd * sizeof(float), s->stream));
  CU(cudaMemsetAsync(s->as, 0, kd * sizeof(float), s->stream));
  s->adam_t = 0;
  s->b1 = (float)b1; s->b2 = (float)b2; s->eps = (float)eps;
  s->adam = 1;
  return GEIG_OK;
}


// ---------------------------------------------------------------------------
// column-owned multi-GPU step (reduce-scatter of the products, update of the
// own columns, all-gather of the bf16 shadow)
// ---------------------------------------------------------------------------

extern "C" geig_status geig_set_partition(geig_solver* s, int world, int rank) {
  if (!s) return fail(GEIG_ERR_ARG, "solver is NULL");
  if (world < 1 || rank < 0 || rank >= world) return fail(GEIG_ERR_ARG, "bad partition world=%d rank=%d", world, rank);
  CU(cudaSetDevice(s->device));
  if (s->gshadow) { CU(cudaStreamSynchronize(s->stream)); cudaFree(s->gshadow); s->gshadow = nullptr; }
  if (s->precv) { cudaFree(s->precv); s->precv = nullptr; }
  if (s->pflags) { cudaFree(s->pflags); s->pflags = nullptr; }
  s->peer_on = false;
  s->peer_epoch = 0;
  s->peer_pending = 0;
  s->part_world = 1; s->part_rank = 0; s->part_W = 0;
  if (world == 1) return GEIG_OK;
  if (s->problem != GEIG_CCA || !(s->math == GEIG_MATH_BF16 || s->math == GEIG_MATH_BF16X2) || !s->upd_res)
    return fail(GEIG_ERR_UNSUPPORTED, "column-owned step needs CCA, bf16 / bf16x2 math and k <= 64");
  if (s->d % ((int64_t)world * 64) != 0 || s->dx % 64 != 0)
    return fail(GEIG_ERR_UNSUPPORTED, "column-owned step needs d %% (64 world) == 0 and dx %% 64 == 0");
  const int64_t W = s->d / world;
  CU(cudaMalloc((void**)&s->gshadow, (size_t)2 * s->k * s->d * sizeof(__nv_bfloat16)));
  s->part_world = world; s->part_rank = rank; s->part_W = W;
  // update grid over the W own columns (segment width a multiple of 8, <= UPD_RES_WMAX)
  int64_t G = std::max<int64_t>(1, std::min<int64_t>(s->nsm, (W + 7) / 8));
  int64_t segw = ((W + G - 1) / G + 7) / 8 * 8;
  if (segw > UPD_RES_WMAX) return fail(GEIG_ERR_UNSUPPORTED, "own block too wide for the resident update");
  s->own_segw = segw;
  s->own_grid = (int)((W + segw - 1) / segw);
  // receive slots and flag words of the peer exchange (used after geig_set_peers)
  const int64_t chunk = geig_owned_chunk_floats(s);
  CU(cudaMalloc((void**)&s->precv, (size_t)world * chunk * sizeof(float)));
  CU(cudaMalloc((void**)&s->pflags, (size_t)2 * GEIG_MAX_PEERS * 32 * sizeof(unsigned)));
  CU(cudaMemsetAsync(s->pflags, 0, (size_t)2 * GEIG_MAX_PEERS * 32 * sizeof(unsigned), s->stream));
  return refresh_gathered_shadow(s);
}

extern "C" geig_status geig_peer_buffers(geig_solver* s, void** recv, int64_t* recv_bytes, void** flags,
                                         int64_t* flags_bytes) {
  if (!s || !recv || !flags) return fail(GEIG_ERR_ARG, "NULL argument");
  if (!s->precv) return fail(GEIG_ERR_STATE, "no partition (geig_set_partition)");
  *recv = s->precv;
  *flags = s->pflags;
  if (recv_bytes) *recv_bytes = (int64_t)s->part_world * geig_owned_chunk_floats(s) * (int64_t)sizeof(float);
  if (flags_bytes) *flags_bytes = (int64_t)2 * GEIG_MAX_PEERS * 32 * (int64_t)sizeof(unsigned);
  return GEIG_OK;
}

extern "C" geig_status geig_set_peers(geig_solver* s, void* const* recv, void* const* shadow, void* const* flags) {
  if (!s || !recv || !shadow || !flags) return fail(GEIG_ERR_ARG, "NULL argument");
  if (!s->precv) return fail(GEIG_ERR_STATE, "no partition (geig_set_partition)");
  if (s->part_world > GEIG_MAX_PEERS) return fail(GEIG_ERR_UNSUPPORTED, "peer exchange: at most %d ranks", GEIG_MAX_PEERS);
  for (int q = 0; q < s->part_world; ++q) {
    if (!recv[q] || !shadow[q] || !flags[q]) return fail(GEIG_ERR_ARG, "NULL peer pointer for rank %d", q);
    if (((uintptr_t)recv[q] | (uintptr_t)shadow[q] | (uintptr_t)flags[q]) % 16) return fail(GEIG_ERR_ARG, "unaligned peer pointer");
  }
  if (recv[s->part_rank] != s->precv || shadow[s->part_rank] != s->gshadow || flags[s->part_rank] != s->pflags)
    return fail(GEIG_ERR_ARG, "the entries of this rank must be its own buffers (geig_peer_buffers, geig_shadow_buffer)");
  CU(cudaSetDevice(s->device));
  for (int q = 0; q < s->part_world; ++q) {
    s->peer_recv[q] = (float*)recv[q];
    s->peer_shadow[q] = (__nv_bfloat16*)shadow[q];
    s->peer_flags[q] = (unsigned*)flags[q];
  }
  s->peer_on = true;
  s->peer_epoch = 0;   // every rank starts here (its flags are zero after geig_set_partition)
  s->peer_pending = 0;
  return GEIG_OK;
}

static tc::OwnedCfg peer_cfg(geig_solver* s, unsigned epoch) {
  tc::OwnedCfg own{(int)s->part_W, s->part_world, s->part_rank, geig_owned_chunk_floats(s), s->precv, s->gshadow};
  own.recv = s->peer_recv;
  own.shadows = s->peer_shadow;
  own.flags = s->peer_flags;
  own.epoch = epoch;
  return own;
}

extern "C" geig_status geig_products_cca_peer(geig_solver* s, const void* X, const void* Y, int64_t b, float scale) {
  if (!s || !X || !Y) return fail(GEIG_ERR_ARG, "NULL argument");
  if (!s->peer_on) return fail(GEIG_ERR_STATE, "no peers (geig_set_peers)");
  if (s->peer_pending) return fail(GEIG_ERR_STATE, "geig_products_cca_peer twice without geig_update_peer");
  if (b < 2 || b > s->max_rows) return fail(GEIG_ERR_ARG, "b=%lld outside [2, max_rows]", (long long)b);
  if (!fused_ok(s, X, Y)) return fail(GEIG_ERR_ARG, "unaligned views");
  CU(cudaSetDevice(s->device));
  const unsigned epoch = s->peer_epoch + 1;
  tc::OwnedCfg own = peer_cfg(s, epoch);
  // forward from the gathered shadow (after every rank's shadow flag of the
  // previous step), backward AV | BV and the table row straight into the
  // owners' receive slots, then this rank's flag at every owner
  UpdateArgs a = update_args(s, 0.0, 0.0);
  geig_status st = tc::fused_cca_step(s->tc, &X, &Y, 1, b, scale, s->Vbf, s->AV, s->BV, a, s->upd_grid, s->upd_smem,
                                      s->stream, /*products_only=*/true, /*tables=*/true, false, &own);
  if (st) return fail(st, "%s", tc::last_error());
  s->launches++;
  s->peer_pending = epoch;
  return GEIG_OK;
}

extern "C" geig_status geig_update_peer(geig_solver* s, double eta, double gamma) {
  if (!s) return fail(GEIG_ERR_ARG, "NULL argument");
  if (!s->peer_on) return fail(GEIG_ERR_STATE, "no peers (geig_set_peers)");
  if (!s->peer_pending) return fail(GEIG_ERR_STATE, "geig_update_peer without geig_products_cca_peer");
  CU(cudaSetDevice(s->device));
  const unsigned epoch = s->peer_pending;
  const int64_t W = s->part_W, k = s->k;
  tc::OwnedCfg own = peer_cfg(s, epoch);
  geig_status st;
  // update: waits for every sender's slot, sums them, updates the own columns,
  // writes the shadow block into every rank's gathered shadow, flags there
  const int64_t c0 = (int64_t)s->part_rank * W;
  UpdateArgs u = update_args(s, eta, gamma);
  u.V = s->V + c0;
  u.AUX = s->AUX + c0;
  u.d = W;
  u.ld = s->d;
  u.segw = s->own_segw;
  u.Vbf = s->gshadow + (int64_t)s->part_rank * 2 * k * W;
  u.vbf_ld = W;
  u.vbf_lo = k * W;
  if (u.am) { u.am += c0; u.as += c0; }
  float* AV = s->precv;   // slot 0 holds the sum after the slot pass
  float* BV = AV + k * W;
  u.AV = AV; u.BV = BV;
  u.raw_a = AV + 2 * k * W;
  u.raw = u.raw_a;
  u.pre_reduced = 1;
  own.buf = AV;
  const void* none[1] = {nullptr};
  st = tc::fused_cca_step(s->tc, none, none, 1, 0, 1.f, s->Vbf, AV, BV, u, s->own_grid,
                          upd_res_smem_floats((int)s->own_segw) * 4, s->stream, /*products_only=*/false,
                          /*tables=*/false, /*update_only=*/true, &own);
  if (st) return fail(st, "%s", tc::last_error());
  s->launches++;
  s->fused_last = false;
  s->peer_epoch = epoch;
  s->peer_pending = 0;
  advance_variant_state(s, 1);
  return GEIG_OK;
}

extern "C" geig_status geig_step_cca_peer(geig_solver* s, const void* X, const void* Y, int64_t b, float scale,
                                          double eta, double gamma) {
  geig_status st = geig_products_cca_peer(s, X, Y, b, scale);
  if (st) return st;
  return geig_update_peer(s, eta, gamma);
}

// CUDA IPC of the peer buffers (one process per GPU): the handle of a
// device allocation of this process, and the mapping of another process's
// handle into this one (peer access enabled lazily).
extern "C" geig_status geig_ipc_handle(const void* dev_ptr, void* handle64) {
  if (!dev_ptr || !handle64) return fail(GEIG_ERR_ARG, "NULL argument");
  cudaIpcMemHandle_t h;
  CU(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle64, &h, 64);
  return GEIG_OK;
}

extern "C" geig_status geig_ipc_open(const void* handle64, void** dev_ptr) {
  if (!handle64 || !dev_ptr) return fail(GEIG_ERR_ARG, "NULL argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  CU(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return GEIG_OK;
}

extern "C" geig_status geig_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return fail(GEIG_ERR_ARG, "NULL argument");
  CU(cudaIpcCloseMemHandle(dev_ptr));
  return GEIG_OK;
}

extern "C" int64_t geig_owned_chunk_floats(const geig_solver* s) {
  if (!s || s->part_world <= 1) return 0;
  const int64_t ntri = (int64_t)s->k * (s->k + 1) / 2, hA = (ntri + s->k + 3) & ~(int64_t)3;
  return 2 * (int64_t)s->k * s->part_W + 2 * hA;
}

extern "C" geig_status geig_shadow_buffer(geig_solver* s, void** ptr, int64_t* bytes_per_rank) {
  if (!s || !ptr) return fail(GEIG_ERR_ARG, "NULL argument");
  if (!s->gshadow) return fail(GEIG_ERR_STATE, "no partition (geig_set_partition)");
  *ptr = s->gshadow;
  if (bytes_per_rank) *bytes_per_rank = 2 * (int64_t)s->k * s->part_W * (int64_t)sizeof(__nv_bfloat16);
  return GEIG_OK;
}

extern "C" geig_status geig_products_cca_owned(geig_solver* s, const void* X, const void* Y, int64_t b, float scale,
                                               float* buf) {
  if (!s || !X || !Y || !buf) return fail(GEIG_ERR_ARG, "NULL argument");
  if (!s->gshadow) return fail(GEIG_ERR_STATE, "no partition (geig_set_partition)");
  if (b < 2 || b > s->max_rows) return fail(GEIG_ERR_ARG, "b=%lld outside [2, max_rows]", (long long)b);
  if (!fused_ok(s, X, Y) || ((uintptr_t)buf % 16)) return fail(GEIG_ERR_ARG, "unaligned views or buffer");
  CU(cudaSetDevice(s->device));
  tc::OwnedCfg own{(int)s->part_W, s->part_world, s->part_rank, geig_owned_chunk_floats(s), buf, s->gshadow};
  UpdateArgs a = update_args(s, 0.0, 0.0);
  geig_status st = tc::fused_cca_step(s->tc, &X, &Y, 1, b, scale, s->Vbf, s->AV, s->BV, a, s->upd_grid, s->upd_smem,
                                      s->stream, /*products_only=*/true, /*tables=*/true, false, &own);
  if (st) return fail(st, "%s", tc::last_error());
  s->launches++;
  return GEIG_OK;
}

extern "C" geig_status geig_update_owned(geig_solver* s, const float* chunk, double eta, double gamma) {
  if (!s || !chunk) return fail(GEIG_ERR_ARG, "NULL argument");
  if (!s->gshadow) return fail(GEIG_ERR_STATE, "no partition (geig_set_partition)");
  if ((uintptr_t)chunk % 16) return fail(GEIG_ERR_ARG, "chunk must be 16-byte aligned");
  CU(cudaSetDevice(s->device));
  const int64_t W = s->part_W, c0 = (int64_t)s->part_rank * W, k = s->k;
  UpdateArgs a = update_args(s, eta, gamma);
  a.V = s->V + c0;
  a.AUX = s->AUX + c0;
  a.d = W;
  a.ld = s->d;
  a.segw = s->own_segw;
  a.Vbf = s->gshadow + (int64_t)s->part_rank * 2 * k * W;   // this rank's block of the gathered shadow
  a.vbf_ld = W;
  a.vbf_lo = k * W;
  if (a.am) { a.am += c0; a.as += c0; }
  float* AV = const_cast<float*>(chunk);
  float* BV = AV + k * W;
  a.AV = AV; a.BV = BV;
  a.raw_a = AV + 2 * k * W;
  a.raw = a.raw_a;
  a.pre_reduced = 1;
  tc::OwnedCfg own{(int)W, s->part_world, s->part_rank, geig_owned_chunk_floats(s), AV, s->gshadow};
  const void* none[1] = {nullptr};
  geig_status st = tc::fused_cca_step(s->tc, none, none, 1, 0, 1.f, s->Vbf, AV, BV, a, s->own_grid,
                                      upd_res_smem_floats((int)s->own_segw) * 4, s->stream,
                                      /*products_only=*/false, /*tables=*/false, /*update_only=*/true, &own);
  if (st) return fail(st, "%s", tc::last_error());
  s->launches++;
  s->fused_last = false;
  advance_variant_state(s, 1);
  return GEIG_OK;
}

extern "C" geig_status geig_set_option(geig_solver* s, int option, int64_t value) {
  if (!s) return fail(GEIG_ERR_ARG, "solver is NULL");
  switch (option) {
    case GEIG_OPT_FUSED_M_TILES:
      if (value < 0 || value > 2) return fail(GEIG_ERR_ARG, "GEIG_OPT_FUSED_M_TILES must be 0, 1 or 2");
      s->tc.opt_m_tiles = (int)value;
      return GEIG_OK;
    case GEIG_OPT_FUSED_PAIRS:
      if (value < 0 || value > 2) return fail(GEIG_ERR_ARG, "GEIG_OPT_FUSED_PAIRS must be 0, 1 or 2");
      s->tc.opt_pairs = (int)value;
      return GEIG_OK;
    case GEIG_OPT_SMALL_CLUSTER:
      if (value < 0 || value > 8 || (value & (value - 1))) return fail(GEIG_ERR_ARG, "GEIG_OPT_SMALL_CLUSTER: 0 (auto), 1, 2, 4 or 8");
      s->opt_small_cluster = (int)value;
      return GEIG_OK;
    case GEIG_OPT_GRAM_TC:
      if (value != 0 && value != 1) return fail(GEIG_ERR_ARG, "GEIG_OPT_GRAM_TC must be 0 or 1");
      s->opt_gram_tc = (int)value;
      return GEIG_OK;
    case GEIG_OPT_SMALL_STEP:
      if (value != 0 && value != 1) return fail(GEIG_ERR_ARG, "GEIG_OPT_SMALL_STEP must be 0 or 1");
      s->opt_small = (int)value;
      return GEIG_OK;
    case GEIG_OPT_STAGED_PRODUCTS:
      if (value != 0 && value != 1) return fail(GEIG_ERR_ARG, "GEIG_OPT_STAGED_PRODUCTS must be 0 or 1");
      s->opt_staged = (int)value;
      return GEIG_OK;
    default:
      return fail(GEIG_ERR_ARG, "unknown option %d", option);
  }
}

extern "C" geig_status geig_update_phase_ns(geig_solver* s, int64_t* out) {
  if (!s || !out) return fail(GEIG_ERR_ARG, "NULL argument");
  CU(cudaSetDevice(s->device));
  unsigned long long t[8];
  CU(cudaMemcpyAsync(t, s->ts, sizeof(t), cudaMemcpyDeviceToHost, s->stream));
  CU(cudaStreamSynchronize(s->stream));
  for (int i = 0; i < 3; ++i) out[i] = (int64_t)(t[i + 1] - t[i]);
  out[3] = s->fused_last ? (int64_t)(t[5] - t[4]) : 0;      // fused: forward phase
  out[4] = s->fused_last ? (int64_t)(t[7] - t[5]) : 0;      // fused: reshuffle + backward phases
  return GEIG_OK;
}

// Developer hook (not part of the documented ABI): per-CTA %globaltimer stamps
// of the tensor-core product kernels are written to `buf` (4 x uint64 per CTA,
// launch after launch overwrite), NULL disables.
extern "C" void geig_debug_set_tc_stamps(void* buf) { tc::dbg_ptr() = (unsigned long long*)buf; }

// Developer hook (not part of the documented ABI): device pointers of the
// solver's internal AV / BV scratch (k x d fp32 each).
extern "C" void geig_debug_products(geig_solver* s, float** av, float** bv) {
  if (av) *av = s ? s->AV : nullptr;
  if (bv) *bv = s ? s->BV : nullptr;
}
