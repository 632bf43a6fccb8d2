// dataflow_step.cuh — the CCA step as ONE persistent cooperative kernel with
// a dataflow schedule instead of grid-wide phases (bf16 tcgen05, k <= 64).
//
// The batch is cut into row chunks of CH rows (CH | h, so a chunk lies in one
// half: reading R1).  Work items:
//   F(c, v, rt, sp)  forward partial Z_v[rows of tile rt of chunk c] over the
//                    sp-th K slice of the features (DRAM-streamed, K-major TMA)
//   B(c) of tile f   backward K-slice "chunk c" of feature tile f: accumulate
//                    X_v[chunk c]^T Z (MN-major TMA, rows just streamed by the
//                    forward items -> L2 hits) into the CTA's TMEM accumulator
//                    (A-half chunks -> AV accumulator, B-half -> BV)
// Every CTA walks a host-built schedule F(0) F(1) B(0) F(2) B(1) ... B(n-1),
// so DRAM streaming of chunk c+1 overlaps the L2-fed backward of chunk c and
// the pipeline ramps up once per step.  Split-K partials are reduced by the
// LAST finishing item of a row tile ("fix-up": per-tile arrival counter),
// which writes the bf16 backward operand and bumps the chunk's ready counter;
// the TMA producer of a B(c) item polls that counter (acquire) before its
// loads.  The two TMEM accumulators of the forward items are double-buffered
// so the MMA issuer never waits for the epilogue drain.  After all items a
// grid barrier hands over to the Gram / update phases (update_res_phases).
#pragma once
#include <cooperative_groups.h>
#include <algorithm>
#include <string>
#include <vector>
#include "tc_gemm.cuh"
#include "update.cuh"

namespace geig { namespace tc {

namespace cg = cooperative_groups;

constexpr int DF_THREADS = 256;
constexpr int DF_MAXSCHED = 96;     // schedule entries per CTA

struct DfMaps {
  CUtensorMap aF[2];   // X, Y K-major (box {64, 128})
  CUtensorMap bF[2];   // V_x, V_y K-major (box {64, BN})
  CUtensorMap aB[2];   // X, Y MN-major over all rows (box {64, 64})
  CUtensorMap bB[4];   // Zb planes [view][half] K-major (box {64, BN})
};

struct DfParams {
  int rows, h, k, BN, stages, CH, nchunks, RT, SPL, kbF[2], kbslice[2];
  int64_t dv[2], d, ldz, hpad;
  float scale;
  uint32_t idescF, idescB;
  const int* sched;      // [G][1 + DF_MAXSCHED]: count, then entries
  const int* btile;      // [G]: feature tile owned for the backward (-1: none)
  int mtB0;              // feature tiles of view x (tiles >= mtB0 belong to view y)
  float* Zp;             // SPL x 2 x k x ldz fp32 split-K partials (player-major)
  __nv_bfloat16* Zb;     // 4 x k x hpad
  int* tile_cnt;         // [2][rows/128] arrival counters (self-resetting)
  int* ready;            // [nchunks] reduced row tiles per chunk (reset at the end)
  float* AV;
  float* BV;
  UpdateArgs upd;
  unsigned long long* dbg;   // optional per-CTA stamps: [start, producer done, MMA done, epilogue done, F done]
};

// schedule entry: bit 31 = B item; F: chunk << 16 | item-in-chunk ; B: chunk
__device__ __forceinline__ bool sched_is_b(int e) { return e < 0; }
__device__ __forceinline__ int sched_chunk(int e) { return (e & 0x7fffffff) >> 16; }
__device__ __forceinline__ int sched_item(int e) { return e & 0xffff; }

struct FItem { int v, rt, sp, row0, kb0, kbn; };
__device__ __forceinline__ FItem decode_f(const DfParams& p, int c, int j) {
  FItem f;
  f.sp = j % p.SPL;
  const int t = j / p.SPL;
  f.rt = t % p.RT;
  f.v = t / p.RT;
  f.row0 = c * p.CH + f.rt * TC_BM;
  const int kb = f.v == 0 ? p.kbF[0] : p.kbF[1];
  f.kb0 = (int)((int64_t)kb * f.sp / p.SPL);
  f.kbn = (int)((int64_t)kb * (f.sp + 1) / p.SPL) - f.kb0;
  return f;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int EB>
__global__ void __launch_bounds__(DF_THREADS, 1)
cca_step_df_kernel(const __grid_constant__ DfMaps maps, const DfParams p) {
  static_assert(EB == 2, "bf16 only");
  constexpr int ATOM = 64, BK = 64, UK = 16;
  constexpr uint32_t A_BYTES = TC_BM * 128;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned view of the dynamic smem that stays in the shared
  // address space (integer pointer round-trips would turn every later smem
  // access into a generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t STAGE_BYTES = A_BYTES + (uint32_t)p.BN * 128;
  const int S = p.stages;
  uint8_t* ring = smem;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + TC_MAX_STAGES;
  uint64_t* accF_full = empty_bar + TC_MAX_STAGES;   // [2]
  uint64_t* accF_empty = accF_full + 2;              // [2]
  uint64_t* accB_full = accF_empty + 2;              // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accB_full + 1);
  int* fix_flag = reinterpret_cast<int*>(tmem_slot + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t NCOLS = 256;       // F slots at cols 0 and 64, B accumulators at 128 (A-half), 192 (B-half)
  const int* my = p.sched + (size_t)blockIdx.x * (1 + DF_MAXSCHED);
  const int nsched = my[0];
  const int bt = p.btile[blockIdx.x];
  const int bview = bt >= p.mtB0 ? 1 : 0;
  const int bm0 = (bt >= p.mtB0 ? bt - p.mtB0 : bt) * TC_BM;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
    mbar_init(&accF_full[0], 1); mbar_init(&accF_full[1], 1);
    mbar_init(&accF_empty[0], 128); mbar_init(&accF_empty[1], 128);
    mbar_init(accB_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int v = 0; v < 2; ++v) { tma_prefetch_desc(&maps.aF[v]); tma_prefetch_desc(&maps.bF[v]); tma_prefetch_desc(&maps.aB[v]); }
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(NCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  stamp(p.upd, 4);
  if (p.dbg && threadIdx.x == 0) p.dbg[blockIdx.x * 8 + 0] = gtimer();

  // This CTA's F items (schedule entries that are not B) in schedule order.
  // The producer issues them eagerly and slots in the CTA's backward chunk c
  // as soon as ready[c] is complete (non-blocking probe between items), so a
  // late chunk never stalls this SM's DRAM stream.  The order actually taken
  // is published per stage (stage_meta) to the MMA issuer, and per forward
  // accumulator slot (accF_item) to the epilogue warps.
  volatile int* stage_meta = reinterpret_cast<volatile int*>(fix_flag + 1);   // [TC_MAX_STAGES]
  volatile int* accF_item = stage_meta + TC_MAX_STAGES;                         // [2]
  int nfm = 0, total_stages = 0;
  for (int si = 0; si < nsched; ++si) {
    const int e = my[1 + si];
    if (!sched_is_b(e)) { ++nfm; total_stages += decode_f(p, sched_chunk(e), sched_item(e)).kbn; }
  }
  const int nbchunks = bt >= 0 ? p.nchunks : 0;
  total_stages += nbchunks * (p.CH / BK);
  // stage meta: F: (fidx << 8) | j  with bit 30 = last k-block ; B: bit 31 | half << 29 | first << 28
  if (threadIdx.x == 0) {
    // ======================= TMA producer =======================
    int it = 0, fi = 0, si = 0, bc = 0;
    const int need = 2 * p.RT;
    while (fi < nfm || bc < nbchunks) {
      bool doB = false;
      if (bc < nbchunks) {
        if (fi >= nfm) {
          while (ld_acquire(&p.ready[bc]) < need) __nanosleep(64);
          doB = true;
        } else {
          doB = ld_acquire(&p.ready[bc]) >= need;
        }
      }
      if (doB) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        const int c = bc++;
        const int half = (c * p.CH) >= p.h ? 1 : 0;
        const int r0 = c * p.CH;
        const int rz = r0 - half * p.h;
        const bool first_of_half = (c * p.CH) == half * p.h;
        const CUtensorMap* mb = &maps.bB[bview * 2 + half];
        for (int j = 0; j < p.CH / BK; ++j, ++it) {
          const int st = it % S;
          if (it >= S) mbar_wait(&empty_bar[st], ((it / S) + 1) & 1);
          stage_meta[st] = (int)(0x80000000u | ((unsigned)half << 29) | ((first_of_half && j == 0) ? (1u << 28) : 0u));
          uint8_t* sa = ring + st * STAGE_BYTES;
          mbar_expect_tx(&full_bar[st], STAGE_BYTES);
#pragma unroll
          for (int q = 0; q < TC_BM / ATOM; ++q)
            tma_load_2d(sa + q * (BK * 128), &maps.aB[bview], &full_bar[st], bm0 + q * ATOM, r0 + j * BK);
          tma_load_2d(sa + A_BYTES, mb, &full_bar[st], rz + j * BK, 0);
        }
      } else {
        // next F entry of the schedule
        while (sched_is_b(my[1 + si])) ++si;
        const int e = my[1 + si++];
        const FItem f = decode_f(p, sched_chunk(e), sched_item(e));
        ++fi;
        for (int j = 0; j < f.kbn; ++j, ++it) {
          const int st = it % S;
          if (it >= S) mbar_wait(&empty_bar[st], ((it / S) + 1) & 1);
          stage_meta[st] = ((si - 1) << 8) | j | (j == f.kbn - 1 ? (1 << 30) : 0);
          uint8_t* sa = ring + st * STAGE_BYTES;
          mbar_expect_tx(&full_bar[st], STAGE_BYTES);
          const int k0 = (f.kb0 + j) * BK;
          tma_load_2d(sa, &maps.aF[f.v], &full_bar[st], k0, f.row0);
          tma_load_2d(sa + A_BYTES, &maps.bF[f.v], &full_bar[st], k0, 0);
        }
        if (p.dbg && fi == nfm) p.dbg[blockIdx.x * 8 + 4] = gtimer();
      }
    }
    if (p.dbg) p.dbg[blockIdx.x * 8 + 1] = gtimer();
  } else if (threadIdx.x == 32) {
    // ======================= MMA issuer =======================
    int nf = 0;
    uint32_t dF = 0;
    for (int it = 0; it < total_stages; ++it) {
      const int st = it % S;
      mbar_wait(&full_bar[st], (it / S) & 1);
      const int meta = stage_meta[st];
      tc_fence_after();
      const uint32_t sa = smem_u32(ring + st * STAGE_BYTES);
      if (meta < 0) {
        const int half = (meta >> 29) & 1;
        const bool first = (meta >> 28) & 1;
        const uint32_t d = tmem_base + 128u + (uint32_t)(half * 64);
#pragma unroll
        for (int kk = 0; kk < BK / UK; ++kk)
          umma<2>(d, make_sdesc(sa + kk * UK * 128, BK * 128, 1024), make_sdesc(sa + A_BYTES + kk * 32, 16, 1024),
                  p.idescB, (!first || kk > 0) ? 1u : 0u);
        umma_commit(&empty_bar[st]);
      } else {
        const int j = meta & 0xff;
        const bool last = (meta >> 30) & 1;
        const int slot = nf & 1;
        if (j == 0) {
          if (nf >= 2) mbar_wait(&accF_empty[slot], ((nf >> 1) - 1) & 1);
          tc_fence_after();
          accF_item[slot] = (meta >> 8) & 0x3fff;      // schedule position of the item
          __threadfence_block();
          dF = tmem_base + (uint32_t)(slot * 64);
        }
#pragma unroll
        for (int kk = 0; kk < BK / UK; ++kk)
          umma<2>(dF, make_sdesc(sa + kk * 32, 16, 1024), make_sdesc(sa + A_BYTES + kk * 32, 16, 1024), p.idescF,
                  (j > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&empty_bar[st]);
        if (last) { umma_commit(&accF_full[slot]); ++nf; }
      }
    }
    if (bt >= 0) umma_commit(accB_full);
    if (p.dbg) p.dbg[blockIdx.x * 8 + 2] = gtimer();
  } else if (warp >= 4) {
    // ======================= epilogue warps =======================
    const int ew = warp - 4;
    const int et = threadIdx.x - 128;         // 0..127
    unsigned long long t_red_acc = 0, t_fix_acc = 0;
    for (int nf = 0; nf < nfm; ++nf) {
      const int slot = nf & 1;
      mbar_wait(&accF_full[slot], (nf >> 1) & 1);
      __syncwarp();
      tc_fence_after();
      const int e = my[1 + accF_item[slot]];
      const int c = sched_chunk(e);
      const FItem f = decode_f(p, c, sched_item(e));
      unsigned long long t_red0 = (p.dbg && et == 0) ? gtimer() : 0ull;
      // partial Z of this split -> Zp[sp][v][n][row] (plain coalesced stores)
      {
        const int row = f.row0 + ew * 32 + lane;
        float* out = p.Zp + ((int64_t)(2 * f.sp + f.v) * p.k) * p.ldz + row;
        for (int c0 = 0; c0 < p.BN; c0 += 16) {
          uint32_t r[16];
          tmem_ld16(tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)(slot * 64 + c0), r);
          if (row < p.rows) {
#pragma unroll
            for (int jn = 0; jn < 16; ++jn)
              if (c0 + jn < p.k) out[(int64_t)(c0 + jn) * p.ldz] = __uint_as_float(r[jn]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&accF_empty[slot]);
      // ---- the last arriving split of this row tile reduces it (fix-up) ----
      // bar.sync makes the 128 threads' stores visible to thread 0, whose
      // gpu-scope fence is cumulative over them before the arrival count.
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (et == 0) {
        __threadfence();
        int* cnt = p.tile_cnt + f.v * (p.rows / TC_BM) + (f.row0 / TC_BM);
        const int old = atomicAdd(cnt, 1);
        const bool lastsp = old == p.SPL - 1;
        if (lastsp) { *cnt = 0; __threadfence(); }   // self-reset for the next step
        *fix_flag = lastsp ? 1 : 0;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (p.dbg && et == 0) { t_red_acc += gtimer() - t_red0; t_red0 = gtimer(); }
      if (*fix_flag) {
        const int half = f.row0 >= p.h ? 1 : 0;
        // half 0: Z_x feeds the Y backward, Z_y the X backward; half 1: own view
        const int dview = half == 0 ? 1 - f.v : f.v;
        __nv_bfloat16* dst = p.Zb + (int64_t)(dview * 2 + half) * p.k * p.hpad;
        const int rbase = f.row0 - half * p.h;
        const int64_t vstride = (int64_t)p.k * p.ldz;
        const float* zsrc = p.Zp + (int64_t)f.v * vstride;
        constexpr int Q = TC_BM / 4;            // float4 per player row of the tile
        for (int u0 = 0; u0 < 16; u0 += 4) {    // 16 x 128 = 2048 = 64 players x 32 quads (k <= 64)
          float4 acc[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int sp = 0; sp < TC_MAX_SPLITS; ++sp) {
            if (sp < p.SPL) {
              float4 v4[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int idx = et + 128 * (u0 + u);
                const int n = idx / Q, q = 4 * (idx % Q);
                const bool ok = n < p.k && f.row0 + q < p.rows;
                v4[u] = ok ? *reinterpret_cast<const float4*>(zsrc + (int64_t)(2 * sp) * vstride + (int64_t)n * p.ldz +
                                                              f.row0 + q)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
              }
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                acc[u].x += v4[u].x; acc[u].y += v4[u].y; acc[u].z += v4[u].z; acc[u].w += v4[u].w;
              }
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int idx = et + 128 * (u0 + u);
            const int n = idx / Q, q = 4 * (idx % Q);
            if (n < p.k && f.row0 + q < p.rows)
              store4<__nv_bfloat16>(dst + (int64_t)n * p.hpad + rbase + q, acc[u].x, acc[u].y, acc[u].z, acc[u].w);
          }
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (et == 0) {
          __threadfence();
          atomicAdd(p.ready + c, 1);
        }
        if (p.dbg && et == 0) t_fix_acc += gtimer() - t_red0;
      }
    }
    if (p.dbg && et == 0) { p.dbg[blockIdx.x * 8 + 6] = t_red_acc; p.dbg[blockIdx.x * 8 + 7] = t_fix_acc; }
    if (p.dbg && et == 0) p.dbg[blockIdx.x * 8 + 5] = gtimer();
    // ---- backward accumulators of the owned feature tile -> AV, BV ----
    if (bt >= 0) {
      mbar_wait(accB_full, 0);
      __syncwarp();
      tc_fence_after();
      const int m = bm0 + ew * 32 + lane;
      const int64_t off = bview == 0 ? 0 : p.dv[0];
      const bool mok = m < (int)p.dv[bview];
      for (int half = 0; half < 2; ++half) {
        float* out = (half == 0 ? p.AV : p.BV) + off + m;
        for (int c0 = 0; c0 < p.BN; c0 += 16) {
          uint32_t r[16];
          tmem_ld16(tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)(128 + half * 64 + c0), r);
          if (mok) {
#pragma unroll
            for (int jn = 0; jn < 16; ++jn)
              if (c0 + jn < p.k) out[(int64_t)(c0 + jn) * p.d] = p.scale * __uint_as_float(r[jn]);
          }
        }
      }
    }
  }
  if (p.dbg && threadIdx.x == 128) p.dbg[blockIdx.x * 8 + 3] = gtimer();
  tc_fence_before();
  __syncwarp();   // reconverge the role lanes before the CTA barrier inside grid.sync
  grid.sync();
  stamp(p.upd, 7);
  if (blockIdx.x == 0)
    for (int c = threadIdx.x; c < p.nchunks; c += blockDim.x) p.ready[c] = 0;
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(NCOLS));
  }
  update_res_phases<true>(p.upd, reinterpret_cast<float*>(smem), grid);
}

// ----------------------------------------------------------------------------
// host side
// ----------------------------------------------------------------------------
struct DfPlan {
  bool ready = false;
  int G = 0, CH = 0, nchunks = 0, RT = 0, SPL = 0, mtB = 0, mtB0 = 0;
  int64_t b = 0;
  int* d_sched = nullptr;
  int* d_btile = nullptr;
  int* d_tile_cnt = nullptr;
  int* d_ready = nullptr;
  float* d_Zp = nullptr;
};

inline void df_destroy(DfPlan& q) {
  for (void* x : {(void*)q.d_sched, (void*)q.d_btile, (void*)q.d_tile_cnt, (void*)q.d_ready, (void*)q.d_Zp})
    if (x) cudaFree(x);
  q = DfPlan();
}

// Build (or reuse) the schedule for batch size b.  Returns false when the
// shape is not covered (caller falls back to the phase-ordered fused kernel).
inline bool df_prepare(DfPlan& q, const TcPlan& t, int64_t b, int G) {
  if (q.ready && q.b == b && q.G == G) return true;
  df_destroy(q);
  const int h = (int)(b / 2);
  int CH = 0;
  for (int c : {512, 256, 128})
    if (h % c == 0) { CH = c; break; }
  if (CH == 0 || t.k > 64 || t.dx % 128 || t.dy % 128) return false;
  const int rows = 2 * h;
  const int nchunks = rows / CH, RT = CH / TC_BM;
  const int mtx = (int)(t.dx / TC_BM), mty = (int)(t.dy / TC_BM), mtB = mtx + mty;
  if (mtB > G || nchunks > 127) return false;
  const int kbx = (int)((t.dx + 63) / 64), kby = (int)((t.dy + 63) / 64);
  // split so that an F item is ~16 k-blocks
  int SPL = std::max(1, std::min(kbx, kby) / 16);
  SPL = std::min(SPL, TC_MAX_SPLITS);
  const int nF = 2 * RT * SPL;                // F items per chunk
  const int Fk = std::min(kbx, kby) / SPL;    // ~stages per F item
  const int Bk = CH / 64;                     // stages per B(c)
  // F items of every chunk are dealt round-robin over all CTAs (the DRAM
  // stream is the bottleneck; the L2-fed backward chunks fill the gaps), so
  // each chunk's forward work is spread over many SMs and completes early.
  std::vector<int> btile(G, -1);
  for (int f = 0; f < mtB; ++f) btile[f] = f;
  std::vector<int> rot;
  for (int g = 0; g < G; ++g) rot.push_back(g);
  (void)Fk; (void)Bk;
  std::vector<std::vector<std::vector<int>>> per_chunk(G, std::vector<std::vector<int>>(nchunks));
  size_t ptr = 0;
  for (int c = 0; c < nchunks; ++c)
    for (int j = 0; j < nF; ++j) {
      per_chunk[rot[ptr % rot.size()]][c].push_back(j);
      ++ptr;
    }
  std::vector<int> sched((size_t)G * (1 + DF_MAXSCHED), 0);
  for (int g = 0; g < G; ++g) {
    std::vector<int> e;
    for (int c = 0; c <= nchunks; ++c) {
      if (c < nchunks)
        for (int j : per_chunk[g][c]) e.push_back((c << 16) | j);
      if (c >= 1 && btile[g] >= 0) e.push_back((int)(0x80000000u | (unsigned)((c - 1) << 16)));
    }
    if ((int)e.size() > DF_MAXSCHED) return false;
    sched[(size_t)g * (1 + DF_MAXSCHED)] = (int)e.size();
    for (size_t i = 0; i < e.size(); ++i) sched[(size_t)g * (1 + DF_MAXSCHED) + 1 + i] = e[i];
  }
  if (cudaMalloc(&q.d_sched, sched.size() * 4) != cudaSuccess || cudaMalloc(&q.d_btile, G * 4) != cudaSuccess ||
      cudaMalloc(&q.d_tile_cnt, 2 * (rows / TC_BM) * 4) != cudaSuccess ||
      cudaMalloc(&q.d_ready, nchunks * 4) != cudaSuccess ||
      cudaMalloc(&q.d_Zp, (size_t)SPL * 2 * t.k * t.ldz * 4) != cudaSuccess) {
    df_destroy(q);
    return false;
  }
  cudaMemcpy(q.d_sched, sched.data(), sched.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(q.d_btile, btile.data(), G * 4, cudaMemcpyHostToDevice);
  cudaMemset(q.d_tile_cnt, 0, 2 * (rows / TC_BM) * 4);
  cudaMemset(q.d_ready, 0, nchunks * 4);

  q.G = G; q.CH = CH; q.nchunks = nchunks; q.RT = RT; q.SPL = SPL; q.mtB = mtB; q.mtB0 = mtx; q.b = b;
  q.ready = true;
  return true;
}

inline geig_status df_cca_step(TcPlan& t, DfPlan& q, const void* X, const void* Y, int64_t b, float scale,
                               const __nv_bfloat16* Vbf, float* AV, float* BV, UpdateArgs upd, size_t upd_bytes,
                               cudaStream_t st) {
  const int eb = 2, ATOM = 64;
  const int h = (int)(b / 2), rows = 2 * h, k = t.k;
  const int64_t dv[2] = {t.dx, t.dy};
  const void* Xv[2] = {X, Y};
  DfMaps maps;
  DfParams p{};
  for (int v = 0; v < 2; ++v) {
    const char* vb = (const char*)Vbf + (v == 0 ? 0 : t.dx * eb);
    if (!make_map(&maps.aF[v], Xv[v], eb, dv[v], rows, dv[v], ATOM, TC_BM) ||
        !make_map(&maps.bF[v], vb, eb, dv[v], k, t.d, ATOM, t.BN) ||
        !make_map(&maps.aB[v], Xv[v], eb, dv[v], rows, dv[v], ATOM, ATOM))
      return tc_fail(GEIG_ERR_CUDA, "tensor map encode (dataflow) failed");
    for (int s = 0; s < 2; ++s) {
      const char* zb = (const char*)t.Zb + (int64_t)(v * 2 + s) * k * t.hpad * eb;
      if (!make_map(&maps.bB[v * 2 + s], zb, eb, h, k, t.hpad, ATOM, t.BN))
        return tc_fail(GEIG_ERR_CUDA, "tensor map encode (dataflow Zb) failed");
    }
    p.dv[v] = dv[v];
    p.kbF[v] = (int)((dv[v] + ATOM - 1) / ATOM);
  }
  p.rows = rows; p.h = h; p.k = k; p.BN = t.BN; p.d = t.d; p.ldz = t.ldz; p.hpad = t.hpad; p.scale = scale;
  p.CH = q.CH; p.nchunks = q.nchunks; p.RT = q.RT; p.SPL = q.SPL;
  p.idescF = make_idesc(eb, false, t.BN, TC_BM);
  p.idescB = make_idesc(eb, true, t.BN, TC_BM);
  p.sched = q.d_sched; p.btile = q.d_btile; p.mtB0 = q.mtB0;
  p.Zp = q.d_Zp; p.Zb = (__nv_bfloat16*)t.Zb; p.tile_cnt = q.d_tile_cnt; p.ready = q.d_ready;
  p.AV = AV; p.BV = BV; p.upd = upd; p.dbg = dbg_ptr();
  const size_t stage_bytes = TC_BM * 128 + (size_t)t.BN * 128;
  p.stages = (int)std::min<size_t>(TC_MAX_STAGES, (196 * 1024) / stage_bytes);
  const size_t ring = (size_t)p.stages * stage_bytes + (2 * TC_MAX_STAGES + 8) * 8 + 16 + (TC_MAX_STAGES + 4) * 4;
  const size_t smem = 1024 + std::max(ring, upd_bytes);
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(cca_step_df_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess)
      return tc_fail(GEIG_ERR_CUDA, "cudaFuncSetAttribute(cca_step_df_kernel) failed");
    attr = true;
  }
  void* args[] = {(void*)&maps, (void*)&p};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)cca_step_df_kernel<2>, dim3(q.G), dim3(DF_THREADS), args, smem, st);
  if (e != cudaSuccess) return tc_fail(GEIG_ERR_CUDA, std::string("cca_step_df_kernel launch: ") + cudaGetErrorString(e));
  return GEIG_OK;
}

}}  // namespace geig::tc
