// fused_step.cuh — one persistent cooperative kernel per CCA step on the
// tensor-core path: every stage of the hot path in a single launch.
//
//   phase F  forward products Z_v = X_v V_v^T (tcgen05, K-major TMA, split-K
//            partials in fp32)                                    [row a1]
//   phase S  sum the split-K partials, route the halves (reading R1) and cast
//            the backward operands to bf16 (all threads, grid-stride)
//   phase B  backward products AV = X_1^T Z, BV = X_2^T Z (tcgen05, MN-major
//            TMA straight from the sample-major views, 2 TMEM accumulators)
//   phase U  Gram tables, coefficients, fused update (update_res_phases)
//                                                                  [rows a2-a4]
// ordered by a grid barrier S -> B and between steps, and by per-tile
// dependency counters F -> S (a CTA's phase S waits for the forward items of
// its row tiles) and B -> U (its update waits for the Gram reduction and the
// backward items of its columns).  One CTA per SM (256 threads): warp 0 lane 0
// issues TMA, warp 1 lane 0 issues tcgen05.mma, warp 2 owns TMEM, warps 4-7
// drain the accumulators (tcgen05.ld -> registers -> coalesced stores); the
// smem ring and its mbarrier phases persist across the work items of F and B,
// so the producer runs ahead into the next item while the epilogue drains.
// Removes, per step, 3 kernel launches, 2 TMEM allocations / pipeline
// prologues and the separate reshuffle launch of the unfused path.
#pragma once
#include <cooperative_groups.h>
#include "tc_gemm.cuh"
#include "update.cuh"
#include <algorithm>
#include <string>

namespace geig { namespace tc {

namespace cg = cooperative_groups;

constexpr int FS_THREADS = 256;
constexpr int GEIG_COEF_FLOATS = 64 * UPD_LTS + 4 * 64;   // Lt | N | 1/s^2 | D1 | D2 (coef_early)
constexpr int TC_RUN_CHUNK = 4096;   // steps per persistent launch (per-step A maps: 3 MiB device + pinned)

struct FusedMaps {
  CUtensorMap a[6];    // A operands of the batch: [0..1] forward X, Y (K-major, box {ATOM, 128});
                       // [2..5] backward X[0:h], X[h:2h], Y[0:h], Y[h:2h] (MN-major, box {ATOM, ATOM})
  CUtensorMap bF[2];   // forward B: V_x, V_y (K-major, box {ATOM, BN})
  CUtensorMap bB[4];   // backward B: Zb planes (K-major, box {ATOM, BN})
  CUtensorMap bFlo[2]; // bf16x2: low halves of V_x, V_y
  CUtensorMap bBlo[4]; // bf16x2: low halves of the Zb planes
  UpdMaps um;          // phase U: fp32 state tiles (V'', AV, [Bv], BV)
};

// wait until *c >= target (acquire); a lost count traps (seconds) instead of hanging
__device__ __forceinline__ void spin_geq_trap(const int* c, int target) {
  int v;
  long long polls = 0;
  do {
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
    if (++polls > (1ll << 22)) __trap();
  } while (v - target < 0);
}

// Peer-exchange flags (system scope: the writers are kernels on other GPUs)
__device__ __forceinline__ void peer_flag_wait(const unsigned* f, unsigned epoch) {
  unsigned v;
  long long polls = 0;
  do {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    if (++polls > (1ll << 26)) __trap();   // a peer that never signals: fail instead of hanging
  } while ((int)(v - epoch) < 0);
}
__device__ __forceinline__ void peer_flag_set(unsigned* f, unsigned epoch) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
}

// Grid barrier of the CTA-pair launches, which are NOT cooperative launches
// (the profiler cannot replay a cooperative launch with thread-block
// clusters; co-residency of the grid is checked on the host with
// cudaOccupancyMaxActiveClusters instead): the cooperative-groups algorithm —
// CTA 0 adds 2^31 - (n - 1), every other CTA 1, so the counter's top bit
// flips exactly once per barrier and the counter never needs a reset.
__device__ __forceinline__ void grid_bar(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned n = gridDim.x;
    const unsigned add = blockIdx.x == 0 ? 0x80000000u - (n - 1) : 1u;
    unsigned old, cur;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(bar), "r"(add) : "memory");
    long long polls = 0;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
      if (++polls > (1ll << 26)) __trap();   // a CTA that never arrives: fail instead of hanging
    } while (((old ^ cur) & 0x80000000u) == 0);
  }
  __syncthreads();
}

struct FusedParams {
  int rows, h, k, BN, stages, splitsF, mtF, mtB[2], split, bwd_y_first, dbg_nostore, dbg_mode, l2_keep;
  // Dependency counters (zero at launch start; CTA 0 zeroes them again after
  // the last step's B barrier, when nothing reads them any more):
  //  rcnt: CTAs whose slice of the Gram reduction is done — step t needs
  //        G (t + 1); warps 2-3 wait for it during phase B and form the
  //        update's coefficients there (coef_early);
  //  fcnt[r]: forward items done on 128-row tile r — step t needs
  //        fper (t + 1) (2 views x splitsF items cover a tile); phase S of a
  //        CTA waits for the tiles of its rows instead of a grid barrier.
  //  bcnt[v * btiles + c]: backward items done on 128-column tile c of view
  //        v — step t needs 2 (t + 1) (the A-half and B-half items); the
  //        update phase of a CTA waits for the tiles of its columns
  int* rcnt;
  int* fcnt;
  int* bcnt;
  int btiles;
  int fper;
  int early_coef;
  int splitB;                      // backward: z as hi + lo bf16 (bf16x2), else hi only
  int tmF, tmB;                    // 128-row M tiles per work item (forward: sample rows; backward: feature
                                   // columns): tm tiles share one B-operand tile per K step, so the ring
                                   // holds tm x more batch bytes in flight per byte of V / Z re-read
  int nsteps;                      // steps of Alg. 2 run by this launch (one batch each)
  // column-owned products (geig_products_cca_owned): 0 = off, else the block
  // width W — the forward's V operand is the gathered shadow [rank][hi|lo][k][W]
  // (3D maps), the backward epilogue writes AV | BV of column c into rank
  // c / W's chunk of `chunk` floats ([AV k x W | BV k x W | tables])
  int ownW;
  int64_t chunk;
  int products_only;               // 1: phases F, S, B only (AV, BV to global; multi-GPU: all-reduce, then geig_update)
  int update_only;                 // phase U only (multi-GPU: from the all-reduced products and tables)
  int tables;                      // products-only launch that also forms the Gram tables (G^A, G^B of the
                                   // local rows into upd.raw_a, G^C of the state into upd.raw)
  uint32_t bar_off;                // smem offset of the ring mbarriers (past the ring AND the update arena)
  const CUtensorMap* xmaps;        // nsteps x 6 A-operand maps in global memory (nullptr: maps.a, one step)
  int kbF[2], kbB;                 // K blocks: forward per view, backward per half
  // CTA pairs (thread-block clusters of 2; 0 = off): the backward items of
  // CTAs 2m, 2m + 1 are the two halves of one 256-column tile (AV, BV), and
  // each CTA updates 128 of those columns: the backward accumulators go
  // straight from TMEM into the update's shared-memory tiles — own columns
  // locally, the partner's through distributed shared memory — instead of
  // through AV / BV in global memory and the B -> U tile counters
  int pair;
  unsigned* gbar;                  // non-null: grid barriers by grid_bar (non-cooperative cluster launch)
  // Peer exchange of the column-owned step (geig_set_peers): the products
  // launch stores each column's AV | BV and the table row straight into the
  // owner's receive buffer (slot = this rank) over peer memory and then
  // raises this rank's flag at every owner; the update launch waits for the
  // flags of all senders, sums the slots in rank order, updates the own
  // columns, writes its shadow block into every rank's gathered shadow and
  // raises its shadow flag at every rank; the next products launch waits for
  // the shadow flags.  Flags carry the step epoch (monotonic, never reset):
  // flag words [q * 32] (receive, from sender q) and [(GEIG_MAX_PEERS + q) * 32]
  // (shadow, from owner q), one 128-byte line each.
  int peer, prank, pworld;
  unsigned epoch;
  float* precv[GEIG_MAX_PEERS];    // owner r's receive buffer (peer-mapped; this rank's own: local)
  unsigned* pflags[GEIG_MAX_PEERS];// rank q's flag words (peer-mapped; this rank's own: local)
  int64_t dv[2], d, ldz, hpad;
  float scale;
  uint32_t idescF, idescB;
  float* Zt;                       // splitsF x 2 x k x ldz fp32 partials
  __nv_bfloat16* Zb;               // 4 x k x hpad
  float* AV;
  float* BV;
  UpdateArgs upd;
};

struct Item {
  int64_t coff;       // global column offset of the item's view
  int nseg, m0, mbound;
  int view;           // backward item: view of the feature columns
  int mt;             // M tiles of this item (<= tm of the phase; fewer at the ragged end)
  int kb0[2], kbn[2];
  const CUtensorMap* ma[2];
  const CUtensorMap* mb[2];
  const CUtensorMap* mblo[2];
  float* out[2];
  int64_t ldo;
  float scale;
  bool keep_a;        // A operand (a view of the batch) is read again in phase B: keep it in L2
};

__device__ __forceinline__ void decode_forward(const FusedMaps& M, const CUtensorMap* A, const FusedParams& p, int idx,
                                               Item& it) {
  const int per_view = p.mtF * p.splitsF;
  const int v = idx / per_view, r = idx % per_view;
  const int mt = r / p.splitsF, sp = r % p.splitsF;
  it.nseg = 1;
  it.m0 = mt * p.tmF * TC_BM;
  it.mbound = p.rows;
  it.mt = min(p.tmF, (p.rows - it.m0 + TC_BM - 1) / TC_BM);
  const int kb = v == 0 ? p.kbF[0] : p.kbF[1];
  it.kb0[0] = (int)((int64_t)kb * sp / p.splitsF);
  it.kbn[0] = (int)((int64_t)kb * (sp + 1) / p.splitsF) - it.kb0[0];
  it.kb0[1] = it.kbn[1] = 0;
  it.ma[0] = &A[v];
  it.mb[0] = v == 0 ? &M.bF[0] : &M.bF[1];
  it.ma[1] = it.ma[0];
  it.mb[1] = it.mb[0];
  it.mblo[0] = it.mblo[1] = v == 0 ? &M.bFlo[0] : &M.bFlo[1];
  it.keep_a = p.l2_keep && v == 1;    // view Y is streamed last in F and first in B
  it.view = v;
  it.coff = v == 0 ? 0 : p.dv[0];
  it.out[0] = p.Zt + ((int64_t)(2 * sp + v) * p.k) * p.ldz;
  it.out[1] = nullptr;
  it.ldo = p.ldz;
  it.scale = 1.f;
}

__device__ __forceinline__ void decode_backward(const FusedMaps& M, const CUtensorMap* A, const FusedParams& p, int idx,
                                                Item& it) {
  // view Y first: phase F streamed Y last, so part of it is still in L2.
  // Item = (feature tile of tmB x 128 columns, half): half 0 (rows [0,h))
  // accumulates AV, half 1 (rows [h,2h)) BV (reading R1).
  const int first = p.bwd_y_first ? 1 : 0;
  const int nfirst = 2 * p.mtB[first];
  const int v = idx < nfirst ? first : 1 - first;
  const int r = v == first ? idx : idx - nfirst;
  const int mt = r >> 1, seg = r & 1;
  it.nseg = 1;
  it.view = v;
  it.m0 = mt * p.tmB * TC_BM;
  it.mbound = (int)(v == 0 ? p.dv[0] : p.dv[1]);
  it.mt = min(p.tmB, (it.mbound - it.m0 + TC_BM - 1) / TC_BM);
  it.kb0[0] = it.kb0[1] = 0;
  it.kbn[0] = p.kbB;
  it.kbn[1] = 0;
  it.ma[0] = it.ma[1] = &A[2 + 2 * v + seg];
  it.mb[0] = it.mb[1] = &M.bB[2 * v + seg];       // Zb planes: y1, x2 (view x); x1, y2 (view y)
  it.mblo[0] = it.mblo[1] = &M.bBlo[2 * v + seg];
  const int64_t off = v == 0 ? 0 : p.dv[0];
  it.keep_a = false;
  it.coff = off;
  it.out[0] = (seg == 0 ? p.AV : p.BV) + (p.ownW ? 0 : off);
  it.out[1] = nullptr;
  it.ldo = p.ownW ? p.ownW : p.d;
  it.scale = p.scale;
}

// developer NaN tracing (dev-knob builds with the stamp buffer set): slot
// 56 + what of this CTA records step + 1 of the first non-finite value
__device__ __forceinline__ void nan_rec(const FusedParams& p, int what, int, float v) {
  // records after the G x 64 stamp slots: 8 per CTA, [7] = the current step
  if (kDevKnobs && p.upd.dbg && !isfinite(v)) {
    unsigned long long* r = p.upd.dbg + (size_t)gridDim.x * 64 + (size_t)blockIdx.x * 8;
    atomicCAS(&r[what], 0ull, *(volatile unsigned long long*)&r[7] + 1ull);
  }
}

__device__ __forceinline__ bool dev_tbar_in_ring(const FusedParams& p) { return kDevKnobs && (p.dbg_mode & 8192); }

struct RingState {
  int it_prod = 0, it_mma = 0, items = 0;   // per-role running counters (persist across phases)
};

// One GEMM phase over this CTA's items (idx = blockIdx.x, +gridDim.x, ...).
template <int EB, bool A_MN>
__device__ __forceinline__ void gemm_phase(const FusedMaps& M, const CUtensorMap* A, const FusedParams& p, int nitems,
                                           uint8_t* ring,
                                           uint64_t* full_bar, uint64_t* empty_bar, uint64_t* accf_bar,
                                           uint64_t* acce_bar, uint32_t tmem_base, RingState& rs, float* epi,
                                           uint64_t* tbar_init = nullptr, const CUtensorMap* Anext = nullptr) {
  constexpr int ATOM = 128 / EB;
  constexpr int BK = ATOM;
  constexpr int UK = 32 / EB;
  constexpr uint32_t A_TILE = TC_BM * 128;         // one 128-row M tile of A for one K block (16 KB)
  const int tm = A_MN ? p.tmB : p.tmF;
  const uint32_t A_BYTES = (uint32_t)tm * A_TILE;   // stage: tm A tiles, then the (shared) B tile(s)
  const uint32_t B_BYTES = (uint32_t)p.BN * 128;
  const bool split = (A_MN ? p.splitB : p.split) != 0;   // hi + lo B operands of this phase
  const uint32_t STAGE_BYTES = A_BYTES + B_BYTES * (split ? 2 : 1);
  const int S = p.stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t idesc = A_MN ? p.idescB : p.idescF;
  Item it;
  if (threadIdx.x == 0) {
    // ---------------- TMA producer (lane 0 of the converged warp 0) ----------------
    const uint64_t pol_keep = l2_policy_evict_last(), pol_stream = l2_policy_evict_first();
    for (int idx = blockIdx.x; idx < nitems; idx += gridDim.x) {
      if (A_MN) decode_backward(M, A, p, idx, it); else decode_forward(M, A, p, idx, it);
      for (int s = 0; s < it.nseg; ++s) {
        for (int j = 0; j < it.kbn[s]; ++j, ++rs.it_prod) {
          const int st = rs.it_prod % S;
          if (rs.it_prod >= S) mbar_wait(&empty_bar[st], ((rs.it_prod / S) + 1) & 1);
          uint8_t* sa = ring + st * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          const bool nob = (kDevKnobs && (p.dbg_mode & 2) != 0);
          const uint32_t abytes = (uint32_t)it.mt * A_TILE;
          mbar_expect_tx(&full_bar[st], abytes + (nob ? 0u : STAGE_BYTES - A_BYTES));
          const int k0 = (it.kb0[s] + j) * BK;
          const uint64_t pa = it.keep_a ? pol_keep : pol_stream;
          for (int mtile = 0; mtile < it.mt; ++mtile) {
            const int mm = it.m0 + mtile * TC_BM;
            uint8_t* sat = sa + mtile * A_TILE;
            if (A_MN) {
#pragma unroll
              for (int q = 0; q < TC_BM / ATOM; ++q)
                tma_load_2d_hint(sat + q * (BK * 128), it.ma[s], &full_bar[st], mm + q * ATOM, k0, pa);
            } else {
              tma_load_2d_hint(sat, it.ma[s], &full_bar[st], k0, mm, pa);
            }
          }
          if (!nob) {   // V / Z tiles: small, re-read by every CTA
            if (!A_MN && p.ownW) {
              // column-owned: V from the gathered shadow, block g / W of rank g / W
              const int64_t g = it.coff + k0;
              const int gw = (int)(g % p.ownW), gr = (int)(g / p.ownW);
              tma_load_3d_hint(sb, it.mb[s], &full_bar[st], gw, 0, gr, pol_keep);
              if (split) tma_load_3d_hint(sb + B_BYTES, it.mblo[s], &full_bar[st], gw, 0, gr, pol_keep);
            } else {
              tma_load_2d_hint(sb, it.mb[s], &full_bar[st], k0, 0, pol_keep);
              if (split) tma_load_2d_hint(sb + B_BYTES, it.mblo[s], &full_bar[st], k0, 0, pol_keep);
            }
          }
        }
      }
    }
    if (!A_MN) {
      // off the critical path (this thread now only waits for the phase to
      // end): the descriptors of phase B and of the update tiles
      for (int v = 0; v < 4; ++v) {
        tma_prefetch_desc(&A[2 + v]);
        tma_prefetch_desc(&M.bB[v]);
        if (split) tma_prefetch_desc(&M.bBlo[v]);
      }
      tma_prefetch_desc(&M.um.t[0]);
      tma_prefetch_desc(&M.um.t[2]);
    } else if (Anext) {
      // the next step's forward descriptors, while this thread waits for the
      // backward to end
      for (int v = 0; v < 2; ++v) tma_prefetch_desc(Anext + v);
    }
  } else if (warp == 1 && elect_one()) {
    // ---------------- MMA issuer (lane 0 of the converged warp 1) ----------------
    for (int idx = blockIdx.x; idx < nitems; idx += gridDim.x, ++rs.items) {
      if (A_MN) decode_backward(M, A, p, idx, it); else decode_forward(M, A, p, idx, it);
      if (rs.items > 0) mbar_wait(acce_bar, (rs.items - 1) & 1);   // epilogue drained the accumulator
      tc_fence_after();
      // bf16x2: the hi and lo tiles of the B operand sit back to back in smem
      // and form ONE N = 2 BN operand, so each K step is a single MMA whose
      // accumulator holds A.B_hi^T in columns [0, BN) and A.B_lo^T in [BN, 2BN)
      // (summed by the epilogue): half the MMA issues and A-operand smem reads
      // of two N = BN MMAs.
      // tm M tiles per K step share the B tile; accumulator of M tile mtile
      // (segment s) at TMEM columns (s * mt + mtile) * acols
      const uint32_t acols = (uint32_t)(p.BN * (split ? 2 : 1));
      for (int s = 0; s < it.nseg; ++s) {
        for (int j = 0; j < it.kbn[s]; ++j, ++rs.it_mma) {
          const int st = rs.it_mma % S;
          mbar_wait(&full_bar[st], (rs.it_mma / S) & 1);
          tc_fence_after();
          const uint32_t sa0 = smem_u32(ring + st * STAGE_BYTES);
          const uint32_t sb = sa0 + A_BYTES;
          for (int mtile = 0; mtile < it.mt; ++mtile) {
            const uint32_t d_tmem = tmem_base + (uint32_t)(s * it.mt + mtile) * acols;
            const uint32_t sa = sa0 + (uint32_t)mtile * A_TILE;
#pragma unroll
            for (int kk = 0; kk < BK / UK; ++kk) {
              if (kDevKnobs && (p.dbg_mode & 1)) break;
              const uint64_t ad = A_MN ? make_sdesc(sa + kk * UK * 128, BK * 128, 1024) : make_sdesc(sa + kk * 32, 16, 1024);
              const uint64_t bd = make_sdesc(sb + kk * 32, 16, 1024);
              umma<EB>(d_tmem, ad, bd, idesc, (j > 0 || kk > 0) ? 1u : 0u);
            }
          }
          umma_commit(&empty_bar[st]);
        }
      }
      umma_commit(accf_bar);
    }
    if (!A_MN && tbar_init) {
      // this step's update-tile barrier, with its init and shared-memory proxy
      // fences, by the MMA thread once its forward issues are done (it only
      // waits for the phase to end): off the B -> U hand-off and off the start
      // of the backward's stream (CTA pairs: pair_exchange arms it and nothing
      // arrives on it before this CTA's announcement there; else the update
      // phase arms it)
      mbar_init(tbar_init, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
  } else if (warp >= 4 && !(A_MN && p.pair)) {   // (CTA pairs: the backward drain is pair_exchange)
    // ---------------- epilogue warps: TMEM -> registers -> smem -> global ----------------
    // Each warp drains its 32 TMEM lanes (32 consecutive m) 16 columns (n) at
    // a time, transposes the 32 x 16 block through its 2 KB of smem and
    // writes it as float4 rows (one instruction: 4 rows x 128 B): a quarter
    // of the store instructions of lane-per-m scalar stores, no per-element
    // bounds branches on full tiles.
    const int ew = warp - 4;
    float* ws = epi + ew * (16 * 32);              // [16 n][32 m]
    for (int idx = blockIdx.x; idx < nitems; idx += gridDim.x, ++rs.items) {
      if (A_MN) decode_backward(M, A, p, idx, it); else decode_forward(M, A, p, idx, it);
      mbar_wait(accf_bar, rs.items & 1);
      __syncwarp();
      tc_fence_after();
      if (threadIdx.x == 128) tstamp(p.upd, A_MN ? 11 : 9);
      const int acols = p.BN * (split ? 2 : 1);
      for (int s = 0; s < it.nseg * it.mt; ++s) {
        const int seg = s / it.mt, mtile = s - seg * it.mt;
        const int mw = it.m0 + mtile * TC_BM + ew * 32;           // this warp's first m
        float* __restrict__ outw = it.out[seg] + mw;
        const uint32_t tb = tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)(s * acols);
        const int q = lane & 7, rr = lane >> 3;                    // float4 column q, row offset rr
        const bool full_m = mw + 32 <= it.mbound;
        const bool q_ok = mw + 4 * q + 3 < it.mbound;
        for (int c0 = 0; c0 < p.BN; c0 += 16) {
          uint32_t r[16], rl[16];
          tmem_ld16(tb + (uint32_t)c0, r);
          if (split) tmem_ld16(tb + (uint32_t)(p.BN + c0), rl);
#pragma unroll
          for (int j = 0; j < 16; ++j)
            ws[j * 32 + lane] = it.scale * (split ? __uint_as_float(r[j]) + __uint_as_float(rl[j]) : __uint_as_float(r[j]));
          __syncwarp();
          if (!(kDevKnobs && p.dbg_nostore)) {
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              const int jn = 4 * g + rr, n = c0 + jn;
              if (n < p.k) {
                const float4 v = *reinterpret_cast<const float4*>(ws + jn * 32 + 4 * q);
                float* o = outw + (int64_t)n * it.ldo + 4 * q;
                if (A_MN && p.ownW) {   // rank-blocked chunk of column gc's owner
                  const int64_t gc = it.coff + mw + 4 * q;
                  const int64_t r = gc / p.ownW;
                  o = (p.peer ? p.precv[r] + (int64_t)p.prank * p.chunk + (it.out[seg] - p.AV)   // owner r's slot
                              : it.out[seg] + r * p.chunk) +
                      (int64_t)n * p.ownW + (gc - r * p.ownW);
                }
                if (kDevKnobs) nan_rec(p, A_MN ? 0 : 1, 0, v.x + v.y + v.z + v.w);
                if (full_m || q_ok) {
                  __stcg(reinterpret_cast<float4*>(o), v);
                } else {
                  const float vv[4] = {v.x, v.y, v.z, v.w};
                  for (int e = 0; e < 4; ++e)
                    if (mw + 4 * q + e < it.mbound) o[e] = vv[e];
                }
              }
            }
          }
          __syncwarp();
        }
      }
      tc_fence_before();
      mbar_arrive(acce_bar);
      if (!A_MN && p.fcnt) {
        // this item's split-K partials are stored: count them on its row tiles (release)
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (threadIdx.x == 128) {
          __threadfence();
          for (int mtile = 0; mtile < it.mt; ++mtile) atomicAdd(p.fcnt + it.m0 / TC_BM + mtile, 1);
        }
      }
      if (A_MN && p.bcnt) {
        // this item's AV / BV columns are final: count them on its column tiles
        // (release; the update phases stage them through TMA, the async proxy)
        asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (threadIdx.x == 128) {
          __threadfence();
          for (int mtile = 0; mtile < it.mt; ++mtile) atomicAdd(p.bcnt + it.view * p.btiles + it.m0 / TC_BM + mtile, 1);
        }
      }
    }
  }
  // Reconverge warps 0/1 (lane 0 ran a role, lanes 1-31 did not) before any
  // CTA barrier: bar.sync counts whole warps, so a divergent warp arriving
  // early would release the barrier before the epilogue warps finished.
  __syncwarp();
}

// CTA pairs: after phase B, the backward accumulators of this CTA (half
// `rank` of the pair's 256-column tile: rank 0 AV, rank 1 BV; M tile 0 =
// the columns of rank 0, M tile 1 those of rank 1) go into the update tiles
// [64 players][W + 4] of the CTA that owns the columns:
//  * own columns: TMEM -> registers -> this CTA's tile (generic stores);
//  * the partner's columns: TMEM -> a staging tile in this CTA's free ring
//    space, then ONE bulk copy (TMA engine, shared::cta -> the partner's
//    shared::cluster tile) that completes on the partner's tile barrier,
//    issued once the partner has announced (remote arrive on this CTA's
//    `freebar`) that its ring is free and its tile barrier is armed.
// No cluster-wide barrier: each CTA waits only for its own MMAs, the
// announcement of its partner and, in the update, its tile barrier (V'' and
// [Bv] by TMA from global memory + the partner's pushed tile).
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ uint32_t cluster_map(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}

__device__ __forceinline__ void pair_exchange(const FusedParams& p, const UpdMaps& um, uint8_t* smem,
                                              uint64_t* accf_bar, uint64_t* acce_bar, uint64_t* tbar,
                                              uint64_t* freebar, uint32_t tmem_base, RingState& rs, int t,
                                              int nitemsB) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool has = (int)blockIdx.x < nitemsB;      // both CTAs of a pair have an item or neither
  const uint32_t rank = blockIdx.x & 1u, peer = rank ^ 1u;   // cluster (2, 1, 1)
  const int W = (int)p.upd.segw, S = W + 4;
  float* Vt = reinterpret_cast<float*>(smem);
  float* At = Vt + 64 * S;
  float* Ct = At + 64 * S;
  float* Bt = Ct + 64 * S;
  float* stage = Bt + 64 * S;                       // the partner's columns (inside the free ring)
  float* tile = rank == 0 ? At : Bt;                // the half this CTA computed (AV or BV)
  const uint32_t push_bytes = (uint32_t)(p.k * S * 4);
  if (warp >= 4 && has) {
    mbar_wait(accf_bar, rs.items & 1);   // this CTA's MMAs are complete: its ring is free
    __syncwarp();
    tc_fence_after();
    if (threadIdx.x == 128) tstamp(p.upd, 11);
  }
  __syncthreads();
  if (threadIdx.x == 128) tstamp(p.upd, 15);
  if (threadIdx.x == 0) {
    // this step's tile barrier (initialised, with its fences, by the MMA
    // thread at the end of phase F — off this critical path): V'' and [Bv]
    // of the own columns (TMA) and the partner's pushed tile; then announce
    // to the partner that it may push.
    // (V'' and [Bv] were last written by the previous step's update with
    // generic stores: ordered for the async proxy by this thread's
    // fence.proxy.async.global at the start of this step's phase F)
    mbar_expect_tx(tbar, (uint32_t)(2 * 64 * S * 4) + (has ? push_bytes : 0u));
    const int c0 = (int)((int64_t)blockIdx.x * W);
    tma_load_2d(Vt, &um.t[0], tbar, c0, 0);
    tma_load_2d(Ct, &um.t[2], tbar, c0, 0);
    // relaxed: the announcement publishes no data of this CTA — the partner's
    // push writes this CTA's tile through the async proxy, the MMAs that read
    // that smem have completed (accf), and the tile barrier's init was released
    // to the cluster by the fence.mbarrier_init at the end of phase F (a
    // release fence followed by this strong relaxed arrive is a release
    // pattern).  A release here cost ~0.7 us/step on the B -> U hand-off.
    if (has)
      asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_map(freebar, peer))
                   : "memory");
    tstamp(p.upd, 16);
  }
  if (has) {
    // all 8 warps drain, the partner's M tile first (its push then crosses
    // DSMEM while the own tile is drained): warps w and w + 4 reach TMEM lanes
    // 32 (w % 4) .. + 31 and split the players in blocks of 32
    __syncwarp();                                   // (thread 0 ran the tile-barrier block alone)
    if (warp < 4) tc_fence_after();
    const int ew = warp & 3;
    const int acols = p.BN * (p.splitB ? 2 : 1);
    const int m = ew * 32 + lane;                   // this thread's column within the M tile (TMEM lane)
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
      const int mtile = (int)(pass == 0 ? peer : rank);
      float* dst = (pass == 0 ? stage : tile) + m;
      const uint32_t tb = tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)(mtile * acols);
      for (int c0 = (warp >> 2) * 32; c0 < p.BN; c0 += 64) {
        uint32_t r0[16], r1[16], l0[16], l1[16];
        tmem_ld16_nw(tb + (uint32_t)c0, r0);
        tmem_ld16_nw(tb + (uint32_t)(c0 + 16), r1);
        if (p.splitB) {
          tmem_ld16_nw(tb + (uint32_t)(p.BN + c0), l0);
          tmem_ld16_nw(tb + (uint32_t)(p.BN + c0 + 16), l1);
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // lanes = 32 consecutive columns: each store is one 128-byte row segment
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int n0 = c0 + j, n1 = c0 + 16 + j;
          const float a0 = p.splitB ? __uint_as_float(r0[j]) + __uint_as_float(l0[j]) : __uint_as_float(r0[j]);
          const float a1 = p.splitB ? __uint_as_float(r1[j]) + __uint_as_float(l1[j]) : __uint_as_float(r1[j]);
          if (n0 < p.k) dst[n0 * S] = p.scale * a0;
          if (n1 < p.k) dst[n1 * S] = p.scale * a1;
        }
      }
      if (pass == 0) {
        // the staged tile is read by the bulk copy (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 3, 256;" ::: "memory");
        if (threadIdx.x == 128) {
          tstamp(p.upd, 17);
          mbar_wait(freebar, (uint32_t)(t & 1));    // the partner's ring is free, its tile barrier armed
          asm volatile(
              "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  cluster_map(tile, peer)),
              "r"(smem_u32(stage)), "r"(push_bytes), "r"(cluster_map(tbar, peer))
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        __syncwarp();
      }
    }
    if (threadIdx.x == 128) tstamp(p.upd, 18);
    tc_fence_before();
    if (warp >= 4) {
      mbar_arrive(acce_bar);
      ++rs.items;
    }
    // without early coefficients the update stages its tables right after
    // the four tiles, i.e. over the staging tile: the push must have read it
    if (threadIdx.x == 128 && !p.early_coef) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  __syncthreads();                                   // the own-column tile (generic stores) is complete
}

template <int EB, bool ADAM>
__global__ void __launch_bounds__(FS_THREADS, 1)
cca_step_kernel(const __grid_constant__ FusedMaps maps, const FusedParams p) {
  cg::grid_group grid = cg::this_grid();
  auto gsync = [&]() {
    if (p.gbar) grid_bar(p.gbar); else grid.sync();
  };
  dstamp(p.upd, 0);
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned view of the dynamic smem that stays in the shared
  // address space (integer pointer round-trips would turn every later smem
  // access into a generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring = smem;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  uint64_t* empty_bar = full_bar + TC_MAX_STAGES;
  uint64_t* accf_bar = empty_bar + TC_MAX_STAGES;
  uint64_t* acce_bar = accf_bar + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce_bar + 1);
  float* side_scratch = reinterpret_cast<float*>(acce_bar + 3);   // 64 floats for warps 2-3
  uint64_t* freebar = reinterpret_cast<uint64_t*>(side_scratch + 64);   // CTA pairs: "the partner's ring is free"
  float* epi_stage = reinterpret_cast<float*>(smem + p.bar_off + 512);   // 4 x 2 KB epilogue transpose tiles
  float* coef_smem = epi_stage + 4 * 16 * 32;                              // early coefficients (GEIG_COEF_FLOATS)
  const int warp = threadIdx.x >> 5;
  constexpr uint32_t NCOLS = 256;   // >= tm * BN * (split ? 2 : 1): one accumulator per M tile of an item

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(accf_bar, 1);
    mbar_init(acce_bar, 128);
    if (p.pair) mbar_init(freebar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int v = 0; v < 2; ++v) tma_prefetch_desc(&maps.bF[v]);
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
  dstamp(p.upd, 1);
  RingState rs;

  // Alg. 2's loop over t: one batch per step, the state stays in HBM/L2, the
  // TMEM allocation, mbarrier ring and its phase counters persist.
  for (int t = 0; t < p.nsteps; ++t) {
  if (kDevKnobs && p.upd.dbg && threadIdx.x == 0) p.upd.dbg[(size_t)gridDim.x * 64 + (size_t)blockIdx.x * 8 + 7] = t;
  const CUtensorMap* A = p.xmaps ? p.xmaps + 6 * t : maps.a;
  if (t > 0) stamp(p.upd, 4);
  if (!p.update_only) {   // (update-only launch: phase U alone, from given products and tables)
  if (p.peer && threadIdx.x == 0)   // every rank's shadow block of the previous update has landed here
    for (int q = 0; q < p.pworld; ++q) peer_flag_wait(p.pflags[p.prank] + (GEIG_MAX_PEERS + q) * 32, p.epoch - 1);
  if (threadIdx.x == 0) {
    // consumer-side proxy fence: the V shadow read by this step's TMA was
    // written with generic stores by every CTA's phase U of the previous step
    // (ordered by the grid barrier); the async proxy must see them
    asm volatile("fence.proxy.async.global;" ::: "memory");
    // (later steps: prefetched at the end of the previous backward, or the
    // same descriptors as before)
    if (t == 0) for (int v = 0; v < 2; ++v) tma_prefetch_desc(&A[v]);
  }

  // ---- phase F: forward split-K partials; warps 2-3: G^C, ||v''||^2 partials ----
  if (warp == 2 || warp == 3) {
    if (!p.products_only || p.tables) gram_c_side(p.upd, threadIdx.x - 64);
    if (threadIdx.x == 64) tstamp(p.upd, 31);
  } else if (!(kDevKnobs && (p.dbg_mode & 8))) {
    gemm_phase<EB, false>(maps, A, p, 2 * p.mtF * p.splitsF, ring, full_bar, empty_bar, accf_bar, acce_bar, tmem_base, rs,
                          epi_stage, (!p.products_only && !dev_tbar_in_ring(p)) ? acce_bar + 2 : nullptr);
    if (threadIdx.x == 32) tstamp(p.upd, 29);
    if (threadIdx.x == 128) tstamp(p.upd, 30);
  }
  __syncthreads();
  dstamp(p.upd, 2);
  if (p.fcnt) {
    // phase S of this CTA reads the split-K partials of its own rows only:
    // wait for the forward items of those 128-row tiles (both halves)
    __syncthreads();
    if (threadIdx.x == 0 || threadIdx.x == 32) {
      // thread 0 polls the tiles of the rows in half 0, thread 32 those in
      // half 1: the two L2 round trips overlap (the CTA barrier below joins them)
      const int U = (((p.h & 3) == 0) && ((p.ldz & 3) == 0) && ((p.hpad & 3) == 0)) ? 4 : 1;   // as phase S
      const int nu = p.h / U;
      const int ua = (int)((int64_t)nu * blockIdx.x / gridDim.x), ub = (int)((int64_t)nu * (blockIdx.x + 1) / gridDim.x);
      const int target = (t + 1) * p.fper;
      if (ub > ua) {
        const int half = threadIdx.x >> 5;
        const int r0 = half * p.h + ua * U, r1 = half * p.h + ub * U - 1;
        for (int tile = r0 / TC_BM; tile <= r1 / TC_BM; ++tile) spin_geq_trap(p.fcnt + tile, target);
      }
    }
    __syncthreads();
  } else {
    gsync();
  }
  stamp(p.upd, 5);
  dstamp(p.upd, 3);

  // ---- phase S: sum partials, route halves, cast to bf16; Gram tables G^A, G^B ----
  // CTA c owns a contiguous range of sample rows of each half.  For every
  // row it sums the split-K partials of z = X_v v''^T (both views, both
  // halves), routes the halves (reading R1) and writes the bf16 (hi, lo)
  // backward operands.  From the same fp32 z it accumulates, by linearity
  // (reading R3), the Gram tables that the update would otherwise form from
  // AV and BV over all d columns:
  //   <v''_i, AV''_j> = scale (zx1_i . zy1_j + zy1_i . zx1_j)     (rows [0,h))
  //   <v''_i, BV''_i> = scale (|zx2_i|^2 + |zy2_i|^2)             (rows [h,2h))
  // (zx1 = X[0:h] v''_x, zy2 = Y[h:2h] v''_y, ...), i.e. k^2 h instead of
  // k^2 d multiply-adds.  The CTA's sums go to the first half of its Gram
  // partial row; the update phase adds G^C and ||v''||^2 and reduces.
  {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // ring smem: async-proxy writes before
    const int64_t vstride = (int64_t)p.k * p.ldz;
    const int64_t plane = (int64_t)p.k * p.hpad;
    const int h = p.h, k = p.k;
    const int tid = threadIdx.x;
    const bool vec = ((h & 3) == 0) && ((p.ldz & 3) == 0) && ((p.hpad & 3) == 0);
    const int U = vec ? 4 : 1;                               // rows per work unit
    const int nu = h / U;
    const int ua = (int)((int64_t)nu * blockIdx.x / gridDim.x), ub = (int)((int64_t)nu * (blockIdx.x + 1) / gridDim.x);
    constexpr int ZR = 16;                                   // rows per chunk
    float* zs = reinterpret_cast<float*>(smem);              // [4 planes: x1, x2, y1, y2][ZR][64]
    float* Ps = zs + 4 * ZR * 64;                            // [64][65]
    float* pst = Ps + 64 * 65;                               // [hA]
    const int ntri = k * (k + 1) / 2;
    const int hA = (ntri + k + 3) & ~3;
    if (k < 64)   // z of players n >= k stays zero (the loops below read all 64 columns)
      for (int e = tid; e < 4 * ZR * 64; e += FS_THREADS) zs[e] = 0.f;
    const int ib = tid & 15, jb = tid >> 4;                  // P tile rows 4ib.., cols 4jb..
    float P[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) P[a][c] = 0.f;
    float gB = 0.f;
    __syncthreads();
    dstamp(p.upd, 23);
    for (int u0 = ua; u0 < ub; u0 += ZR / U) {
      const int nuc = min(ZR / U, ub - u0);
      for (int e = tid; e < k * nuc; e += FS_THREADS) {
        const int n = e / nuc, uu = e - n * nuc;
        const int r = (u0 + uu) * U;
        float z[4][4];                                       // [plane][row]
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int w = 0; w < 4; ++w) z[q][w] = 0.f;
        // split-K partials: 4 splits per round, all 16 loads of a round issued
        // before the adds (one L2 round trip per round, not per split)
        for (int sp0 = 0; sp0 < p.splitsF; sp0 += 4) {
          if (vec) {
            float4 ld[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int sp = sp0 + u;
              if (sp < p.splitsF) {
                const float* zx = p.Zt + (int64_t)(2 * sp) * vstride + (int64_t)n * p.ldz;
                const float* zy = zx + vstride;
                ld[u][0] = __ldcg(reinterpret_cast<const float4*>(zx + r));
                ld[u][1] = __ldcg(reinterpret_cast<const float4*>(zx + h + r));
                ld[u][2] = __ldcg(reinterpret_cast<const float4*>(zy + r));
                ld[u][3] = __ldcg(reinterpret_cast<const float4*>(zy + h + r));
              } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) ld[u][q] = make_float4(0.f, 0.f, 0.f, 0.f);
              }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                z[q][0] += ld[u][q].x; z[q][1] += ld[u][q].y; z[q][2] += ld[u][q].z; z[q][3] += ld[u][q].w;
              }
          } else {
            for (int sp = sp0; sp < min(sp0 + 4, p.splitsF); ++sp) {
              const float* zx = p.Zt + (int64_t)(2 * sp) * vstride + (int64_t)n * p.ldz;
              const float* zy = zx + vstride;
              z[0][0] += zx[r]; z[1][0] += zx[h + r]; z[2][0] += zy[r]; z[3][0] += zy[h + r];
            }
          }
        }
        // Zb planes: 0 = y1 (-> AV_x), 1 = x2 (-> BV_x), 2 = x1 (-> AV_y), 3 = y2 (-> BV_y)
        const int64_t o = (int64_t)n * p.hpad + r;
        if (kDevKnobs)
          nan_rec(p, 2, 0, z[0][0] + z[1][0] + z[2][0] + z[3][0] + z[0][3] + z[1][3] + z[2][3] + z[3][3]);
        if (vec) {
          store4<__nv_bfloat16>(p.Zb + 0 * plane + o, z[2][0], z[2][1], z[2][2], z[2][3]);
          store4<__nv_bfloat16>(p.Zb + 1 * plane + o, z[1][0], z[1][1], z[1][2], z[1][3]);
          store4<__nv_bfloat16>(p.Zb + 2 * plane + o, z[0][0], z[0][1], z[0][2], z[0][3]);
          store4<__nv_bfloat16>(p.Zb + 3 * plane + o, z[3][0], z[3][1], z[3][2], z[3][3]);
          if (p.splitB) {
            store4_lo<__nv_bfloat16>(p.Zb + 4 * plane + o, z[2][0], z[2][1], z[2][2], z[2][3]);
            store4_lo<__nv_bfloat16>(p.Zb + 5 * plane + o, z[1][0], z[1][1], z[1][2], z[1][3]);
            store4_lo<__nv_bfloat16>(p.Zb + 6 * plane + o, z[0][0], z[0][1], z[0][2], z[0][3]);
            store4_lo<__nv_bfloat16>(p.Zb + 7 * plane + o, z[3][0], z[3][1], z[3][2], z[3][3]);
          }
        } else {
          const float zv[4] = {z[2][0], z[1][0], z[0][0], z[3][0]};
          for (int q = 0; q < 4; ++q) {
            const __nv_bfloat16 hv = __float2bfloat16_rn(zv[q]);
            p.Zb[q * plane + o] = hv;
            if (p.splitB) p.Zb[(4 + q) * plane + o] = __float2bfloat16_rn(zv[q] - __bfloat162float(hv));
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int w = 0; w < 4; ++w)
            if (w < U) zs[(q * ZR + uu * U + w) * 64 + n] = z[q][w];
      }
      __syncthreads();
      dstamp(p.upd, 24);
      const int nr = nuc * U;
      for (int r = 0; r < nr; ++r) {
        const float4 xi = *reinterpret_cast<const float4*>(zs + (0 * ZR + r) * 64 + 4 * ib);
        const float4 yi = *reinterpret_cast<const float4*>(zs + (2 * ZR + r) * 64 + 4 * ib);
        const float4 xj = *reinterpret_cast<const float4*>(zs + (0 * ZR + r) * 64 + 4 * jb);
        const float4 yj = *reinterpret_cast<const float4*>(zs + (2 * ZR + r) * 64 + 4 * jb);
        const float xa[4] = {xi.x, xi.y, xi.z, xi.w}, ya[4] = {yi.x, yi.y, yi.z, yi.w};
        const float xb[4] = {xj.x, xj.y, xj.z, xj.w}, yb[4] = {yj.x, yj.y, yj.z, yj.w};
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) P[a][c] = fmaf(xa[a], yb[c], fmaf(ya[a], xb[c], P[a][c]));
      }
      if (tid < 64)
        for (int r = 0; r < nr; ++r) {
          const float x2 = zs[(1 * ZR + r) * 64 + tid], y2 = zs[(3 * ZR + r) * 64 + tid];
          gB = fmaf(x2, x2, fmaf(y2, y2, gB));
        }
      __syncthreads();
      dstamp(p.upd, 25);
    }
    // first half of this CTA's Gram partial row: [tri(G^A) | diag(G^B) | pad]
    if (!p.products_only || p.tables) {
      float* pr = pst;
      const float sc = p.scale;
      // the z-Gram is symmetric: each thread writes the lower-triangle entries of its 4x4 tile
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int i = 4 * ib + a, j = 4 * jb + c;
          if (i < k && j <= i) pr[tri_index(i, j)] = sc * P[a][c];
        }
      if (tid < k) pr[ntri + tid] = sc * gB;
      for (int e = ntri + k + tid; e < hA; e += FS_THREADS) pr[e] = 0.f;
      __syncthreads();
      dstamp(p.upd, 26);
      float* out = p.upd.partial + (size_t)blockIdx.x * (2 * hA);
      for (int e = 4 * tid; e < hA; e += 4 * FS_THREADS)
        *reinterpret_cast<float4*>(out + e) = *reinterpret_cast<const float4*>(pr + e);
    }
    // generic smem writes before the next TMA writes into the ring; generic
    // global writes (Zb) consumed by the async proxy (TMA) after the barrier
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  __syncthreads();
  dstamp(p.upd, 4);
  gsync();
  stamp(p.upd, 6);
  dstamp(p.upd, 5);

  // ---- phase B: backward products into AV, BV ----
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.global;" ::: "memory");   // Zb of every CTA's phase S, read by TMA below
    // (the backward's descriptors were prefetched by this thread at the end
    // of its forward producer loop, where it only waits for the epilogue)
  }
  if (warp == 2 || warp == 3) {    // warps 2-3: reduce the (now complete) Gram partial rows
    if (!p.products_only || p.tables) {
      reduce_side(p.upd, threadIdx.x - 64, side_scratch);
      if (threadIdx.x == 64) tstamp(p.upd, 27);
      if (p.rcnt) {
        asm volatile("bar.sync 1, 64;" ::: "memory");
        if (threadIdx.x == 64) {
          __threadfence();
          atomicAdd(p.rcnt, 1);
        }
        if (p.early_coef) {
          if (threadIdx.x == 64) spin_geq_trap(p.rcnt, (t + 1) * (int)gridDim.x);
          asm volatile("bar.sync 1, 64;" ::: "memory");
          if (threadIdx.x == 64) tstamp(p.upd, 12);
          coef_early(p.upd, coef_smem, t, threadIdx.x - 64);
          if (threadIdx.x == 64) tstamp(p.upd, 10);
        }
      }
    }
  } else if (!(kDevKnobs && (p.dbg_mode & 32))) {
    gemm_phase<EB, true>(maps, A, p, 2 * (p.mtB[0] + p.mtB[1]), ring, full_bar, empty_bar, accf_bar, acce_bar, tmem_base, rs,
                         epi_stage, nullptr, (p.xmaps && t + 1 < p.nsteps) ? p.xmaps + 6 * (t + 1) : nullptr);
  }
  tc_fence_before();
  if (p.upd.dbg && threadIdx.x >= 128) {
    if (threadIdx.x == 128) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) :: "memory");
      p.upd.dbg[(size_t)blockIdx.x * 64 + 17] = t;
      p.upd.dbg[(size_t)blockIdx.x * 64 + 49] = clock64();
    }
    __threadfence();
    if (threadIdx.x == 128) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) :: "memory");
      p.upd.dbg[(size_t)blockIdx.x * 64 + 16] = t;
      p.upd.dbg[(size_t)blockIdx.x * 64 + 48] = clock64();
    }
  }
  __syncthreads();
  dstamp(p.upd, 6);
  if (p.upd.dbg && threadIdx.x == 0) {
    p.upd.dbg[(size_t)blockIdx.x * 64 + 18] = *(volatile unsigned long long*)&p.upd.dbg[(size_t)blockIdx.x * 64 + 17];
    __threadfence(); dstamp(p.upd, 15);
  }
  if (p.pair) {
    // the update needs the Gram reduction of every CTA (coefficients) and the
    // backward accumulators of the pair (exchanged through DSMEM)
    // (with early coefficients warps 2-3 have waited for it in phase B)
    if (threadIdx.x == 0 && p.rcnt && !p.early_coef) spin_geq_trap(p.rcnt, (t + 1) * (int)gridDim.x);
    pair_exchange(p, maps.um, smem, accf_bar, acce_bar, acce_bar + 2, freebar, tmem_base, rs, t,
                  2 * (p.mtB[0] + p.mtB[1]));
    if (kDevKnobs && (p.dbg_mode & 16384)) {   // developer: the exchanged tiles to AV / BV (global)
      mbar_wait(acce_bar + 2, 0);
      const int W = (int)p.upd.segw, S = W + 4;
      const float* At = reinterpret_cast<const float*>(smem) + 64 * S;
      const float* Bt = At + 2 * 64 * S;
      const int64_t c0 = (int64_t)blockIdx.x * W;
      for (int e = threadIdx.x; e < p.k * W; e += FS_THREADS) {
        const int i = e / W, c = e - i * W;
        if (c0 + c < p.d) { p.AV[i * p.d + c0 + c] = At[i * S + c]; p.BV[i * p.d + c0 + c] = Bt[i * S + c]; }
      }
      __syncthreads();
    }
  } else if (p.bcnt && !p.products_only) {
    // the update phase of this CTA needs the Gram reduction of every CTA and
    // the backward items of its own columns [c W, (c + 1) W) only
    if (threadIdx.x == 0) {
      // (with early coefficients warps 2-3 have waited for the reduction in phase B)
      if (p.rcnt && !p.early_coef) spin_geq_trap(p.rcnt, (t + 1) * (int)gridDim.x);
      const int64_t W = p.upd.segw;
      const int64_t c0 = (int64_t)blockIdx.x * W, c1 = min(p.d, c0 + W);
      for (int v = 0; v < 2; ++v) {
        const int64_t lo = v == 0 ? 0 : p.dv[0], hi = v == 0 ? p.dv[0] : p.d;
        const int64_t a = max(c0, lo), b = min(c1, hi);
        if (a < b)
          for (int tile = (int)((a - lo) / TC_BM); tile <= (int)((b - 1 - lo) / TC_BM); ++tile)
            spin_geq_trap(p.bcnt + v * p.btiles + tile, 2 * (t + 1));
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    __syncthreads();
  } else {
    if (p.peer) __threadfence_system();   // this thread's peer stores performed before the flags below
    gsync();
    if (p.peer && blockIdx.x == 0 && threadIdx.x == 0)   // this rank's slot is complete at every owner
      for (int r = 0; r < p.pworld; ++r) peer_flag_set(p.pflags[r] + p.prank * 32, p.epoch);
  }
  stamp(p.upd, 7);
  dstamp(p.upd, 7);
  }  // !update_only

  if (p.peer && p.update_only) {
    // the senders' slots of this step have landed: sum them in rank order
    // into slot 0 (the own columns of this CTA; CTA 0 also the table row)
    if (threadIdx.x == 0)
      for (int q = 0; q < p.pworld; ++q) peer_flag_wait(p.pflags[p.prank] + q * 32, p.epoch);
    __syncthreads();
    float* rb = p.precv[p.prank];
    const int64_t W = p.ownW, kW = (int64_t)p.k * W;
    const int64_t c0 = (int64_t)blockIdx.x * p.upd.segw, c1 = min(W, c0 + p.upd.segw);
    const int nc = c1 > c0 ? (int)(c1 - c0) : 0;
    for (int e = threadIdx.x; e < 2 * p.k * nc; e += FS_THREADS) {
      const int h = e / (p.k * nc), r = e - h * p.k * nc, i = r / nc, c = r - i * nc;
      const int64_t o = h * kW + (int64_t)i * W + c0 + c;
      float v = rb[o];
      for (int q = 1; q < p.pworld; ++q) v += rb[(int64_t)q * p.chunk + o];
      rb[o] = v;
    }
    if (blockIdx.x == 0) {
      const int ntri = p.k * (p.k + 1) / 2, hA = (ntri + p.k + 3) & ~3;
      for (int e = threadIdx.x; e < 2 * hA; e += FS_THREADS) {
        float v = rb[2 * kW + e];
        for (int q = 1; q < p.pworld; ++q) v += rb[(int64_t)q * p.chunk + 2 * kW + e];
        rb[2 * kW + e] = v;
      }
    }
    __threadfence();
    gsync();
  }

  // ---- phase U: Gram tables + fused update ----
  if (!p.products_only && !(kDevKnobs && (p.dbg_mode & 64)))
    update_res_phases<true, 1, ADAM>(p.upd, reinterpret_cast<float*>(smem), grid, &maps.um, t,
                                     p.early_coef ? coef_smem : nullptr,
                                     dev_tbar_in_ring(p) ? nullptr : acce_bar + 2,
                                     !p.update_only && !dev_tbar_in_ring(p));
  if (p.pair && threadIdx.x == 128) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // staging reusable
  if (t + 1 < p.nsteps) {
    // next step: its forward TMA reads the new bf16 shadow of V (generic
    // stores above) and refills the smem ring the update phase used
    asm volatile("fence.proxy.async.global;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    gsync();
    tc_fence_after();
  }
  }  // steps

  if (p.peer && p.update_only) {
    __threadfence_system();               // this thread's shadow stores into the peers performed
    gsync();
    if (blockIdx.x == 0 && threadIdx.x == 0)   // this rank's shadow block is in every rank's copy
      for (int q = 0; q < p.pworld; ++q) peer_flag_set(p.pflags[q] + (GEIG_MAX_PEERS + p.prank) * 32, p.epoch);
  }
  if (p.rcnt || p.fcnt || p.bcnt) {
    // every CTA is past its last counter read: back to zero for the next launch
    gsync();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (p.rcnt) *p.rcnt = 0;
      if (p.fcnt)
        for (int r = 0; r < (p.rows + TC_BM - 1) / TC_BM; ++r) p.fcnt[r] = 0;
      if (p.bcnt)
        for (int r = 0; r < 2 * p.btiles; ++r) p.bcnt[r] = 0;
    }
  }

  // ---- release TMEM ----
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(NCOLS));
  }
}


// ----------------------------------------------------------------------------
// host side
// ----------------------------------------------------------------------------

// Whole CCA step in one cooperative launch (bf16 tensor cores, k <= 64).
// `upd` carries the update arguments (state, AV/BV scratch, eta, gamma...);
// its grid partition (gridDim = G, segw) is reused by the GEMM phases.
// The six A-operand maps of one batch (X, Y sample-major, b = 2h rows):
// [0..1] forward K-major boxes, [2..5] backward MN-major boxes of the halves.
// Cooperative launch with the solver's persisting-L2 window attached to THIS
// launch only (no stream attribute is changed, so the caller's later kernels
// on the same stream do not inherit it).
inline cudaError_t launch_coop(const void* fn, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t st,
                               const cudaAccessPolicyWindow& win, int cluster = 0, bool coop = true) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[3];
  int n = 0;
  if (coop) {
    attr[n].id = cudaLaunchAttributeCooperative;
    attr[n++].val.cooperative = 1;
  }
  if (cluster > 1) {   // thread-block clusters (CTA pairs of the fused step)
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = (unsigned)cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n++].val.clusterDim.z = 1;
  }
  if (win.num_bytes > 0) {
    attr[n].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[n++].val.accessPolicyWindow = win;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

inline bool make_batch_maps(CUtensorMap* a, const TcPlan& t, const void* X, const void* Y, int h) {
  const int eb = 2, ATOM = 64;
  const int64_t dv[2] = {t.dx, t.dy};
  const void* Xv[2] = {X, Y};
  for (int v = 0; v < 2; ++v) {
    if (!make_map(&a[v], Xv[v], eb, dv[v], 2 * h, dv[v], ATOM, TC_BM)) return false;
    for (int s = 0; s < 2; ++s) {
      const char* xb = (const char*)Xv[v] + (int64_t)s * h * dv[v] * eb;
      if (!make_map(&a[2 + 2 * v + s], xb, eb, dv[v], h, dv[v], ATOM, ATOM)) return false;
    }
  }
  return true;
}

// Column-owned multi-GPU step (geig_set_partition): rank `rank` of `world`
// owns columns [rank W, (rank + 1) W) of d.  products launch: the forward's
// V operand is the gathered bf16 shadow `gathered` ([world][hi|lo][k][W]),
// AV | BV | tables go to `buf` (world chunks of `chunk` floats, one per
// owner, for the reduce-scatter); update launch: AV, BV and the tables come
// from the rank's summed chunk `buf` and the update covers the own columns.
struct OwnedCfg {
  int W, world, rank;
  int64_t chunk;
  float* buf;
  __nv_bfloat16* gathered;
  // peer exchange (geig_set_peers): nullptr = NCCL-style buffers
  float* const* recv = nullptr;              // [world] receive buffers (peer-mapped)
  __nv_bfloat16* const* shadows = nullptr;   // [world] gathered shadows (peer-mapped)
  unsigned* const* flags = nullptr;          // [world] flag words (peer-mapped)
  unsigned epoch = 0;
};

// Whole CCA step(s) in one cooperative launch (bf16 tensor cores, k <= 64):
// nsteps consecutive steps of Alg. 2, step i on batch (X[i], Y[i]) (device
// pointers, b rows each).  `upd` carries the update arguments (state, AV/BV
// scratch, eta, gamma...); its grid partition (gridDim = G, segw) is reused
// by the GEMM phases.
inline geig_status fused_cca_step(TcPlan& t, const void* const* X, const void* const* Y, int nsteps, int64_t b,
                                  float scale, const __nv_bfloat16* Vbf, float* AV, float* BV, UpdateArgs upd,
                                  int grid_ctas, size_t upd_bytes, cudaStream_t st, bool products_only = false,
                                  bool tables = false, bool update_only = false, const OwnedCfg* own = nullptr,
                                  int pair_grid = 0) {
  if (!t.ready || t.math != GEIG_MATH_BF16) return tc_fail(GEIG_ERR_STATE, "fused step needs the bf16 plan");
  if (nsteps < 1) return tc_fail(GEIG_ERR_ARG, "nsteps < 1");
  // (t.math is BF16 for both GEIG_MATH_BF16 and GEIG_MATH_BF16X2; t.splitb selects hi+lo operands)
  const int eb = 2, ATOM = 64;
  const int h = (int)(b / 2), rows = 2 * h, k = t.k;
  const int64_t dv[2] = {t.dx, t.dy};
  FusedMaps maps;
  FusedParams p{};
  if (update_only && (products_only || nsteps != 1)) return tc_fail(GEIG_ERR_ARG, "update-only launch: one step");
  const UpdateArgs upd_in = upd;                     // (the fallback below relaunches with the caller's arguments)
  const int grid_in = grid_ctas;
  const size_t upd_bytes_in = upd_bytes;
  // CTA pairs (full steps): every 256-column backward tile of both views is
  // one pair's item and each CTA of the pair updates 128 of its columns
  // (the update then covers d / 128 CTAs: used where that is most of the grid)
  const int64_t pair_ctas = (t.dx + t.dy) / 128;
  const bool pair = pair_grid > 0 && t.opt_pairs && !products_only && !update_only && !own && t.dx % 256 == 0 &&
                    t.dy % 256 == 0 && pair_ctas <= pair_grid && 4 * pair_ctas >= 3 * (int64_t)pair_grid &&
                    (pair_grid & 1) == 0 && t.opt_m_tiles != 1 && 128 <= UPD_RES_WMAX;
  if (pair) {
    grid_ctas = pair_grid;
    upd.segw = 128;
    upd.pair_tiles = 1;
    upd_bytes = upd_res_smem_floats(128) * 4;
  } else if (pair_grid > 0 && !products_only && !update_only && !own && 2 * grid_ctas <= pair_grid) {
    // small d (config 2: 49 CTAs of 32 columns): the update's column
    // partition would leave most SMs idle in phases F, S and B — a finer
    // partition (8-column multiples) widens the grid (98 CTAs of 16
    // columns: 27.05 vs 27.55 us/step, same-box A/B)
    int64_t segw = ((t.dx + t.dy + pair_grid - 1) / pair_grid + 7) / 8 * 8;
    grid_ctas = (int)((t.dx + t.dy + segw - 1) / segw);
    upd.segw = segw;
    upd_bytes = upd_res_smem_floats((int)segw) * 4;
  }
  if (!update_only && !make_batch_maps(maps.a, t, X[0], Y[0], h))
    return tc_fail(GEIG_ERR_CUDA, "tensor map encode (batch) failed");
  p.nsteps = nsteps;
  p.products_only = products_only ? 1 : 0;
  p.tables = (products_only && tables) ? 1 : 0;
  p.update_only = update_only ? 1 : 0;
  // Gram-reduction counter: every launch that runs the reduction (full steps,
  // products + tables) counts it; the full steps also use it for the early
  // coefficients.  The solver's epoch advances only with a launch that was
  // enqueued (below), so targets always match the counts.
  p.rcnt = p.fcnt = p.bcnt = nullptr;
  p.btiles = 0;
  p.fper = 0;
  p.early_coef = 0;
  if (!update_only) {
    const int ntiles = (int)((t.max_rows + TC_BM - 1) / TC_BM);
    const int btiles = (int)((std::max(t.dx, t.dy) + TC_BM - 1) / TC_BM);
    if (!t.dep) {   // [rcnt | pad][grid barrier | pad][fcnt per 128-row tile | bcnt per view x 128-column tile]
                    // (128-byte lines; the counts are zero between launches, the barrier word persists)
      const size_t words = 64 + (size_t)ntiles + 2 * (size_t)btiles;
      if (cudaMalloc((void**)&t.dep, words * sizeof(int)) != cudaSuccess ||
          cudaMemsetAsync(t.dep, 0, words * sizeof(int), st) != cudaSuccess)
        return tc_fail(GEIG_ERR_CUDA, "allocating the dependency counters failed");
    }
    const bool runs_reduce = !products_only || tables;
    if (runs_reduce && !dev_knob("GEIG_NO_EARLY_COEF")) {
      p.rcnt = t.dep;
      p.early_coef = products_only ? 0 : 1;
    }
    if (!dev_knob("GEIG_F_BARRIER")) p.fcnt = t.dep + 64;   // GEIG_F_BARRIER: developer A/B (grid barrier after F)
    p.btiles = btiles;
    if (!products_only && !pair && !dev_knob("GEIG_BU_BARRIER")) p.bcnt = t.dep + 64 + ntiles;   // (grid barrier after B)
  }
  if (products_only && nsteps != 1) return tc_fail(GEIG_ERR_ARG, "products-only launch runs one step");
  p.xmaps = nullptr;
  bool same_batch = true;   // every step on one batch: the param-space maps serve all steps
  for (int i = 1; i < nsteps && same_batch; ++i) same_batch = X[i] == X[0] && Y[i] == Y[0];
  if (dev_knob("GEIG_XMAPS_ALWAYS")) same_batch = false;
  if (nsteps > 1 && !same_batch) {
    // per-step A maps in global memory (distinct batches encoded once)
    if (nsteps > TC_RUN_CHUNK) return tc_fail(GEIG_ERR_ARG, "fused run: more than TC_RUN_CHUNK steps per launch");
    if (!t.xm_dev) {   // fixed capacity, allocated once (never inside a timed loop of later calls)
      if (cudaMalloc((void**)&t.xm_dev, (size_t)TC_RUN_CHUNK * 6 * sizeof(CUtensorMap)) != cudaSuccess ||
          cudaMallocHost((void**)&t.xm_host, (size_t)TC_RUN_CHUNK * 6 * sizeof(CUtensorMap)) != cudaSuccess)
        return tc_fail(GEIG_ERR_CUDA, "allocating per-step tensor maps failed");
      t.xm_cap = TC_RUN_CHUNK;
    }
    if (!t.xm_ev && cudaEventCreateWithFlags(&t.xm_ev, cudaEventDisableTiming) != cudaSuccess)
      return tc_fail(GEIG_ERR_CUDA, "cudaEventCreate failed");
    cudaEventSynchronize(t.xm_ev);   // the previous call's copy out of the pinned staging buffer is done
    for (int i = 0; i < nsteps; ++i) {
      int j = 0;
      while (j < i && !(X[j] == X[i] && Y[j] == Y[i])) ++j;
      if (j < i) {
        memcpy(&t.xm_host[6 * i], &t.xm_host[6 * j], 6 * sizeof(CUtensorMap));
      } else if (!make_batch_maps(&t.xm_host[6 * i], t, X[i], Y[i], h)) {
        return tc_fail(GEIG_ERR_CUDA, "tensor map encode (batch) failed");
      }
    }
    if (cudaMemcpyAsync(t.xm_dev, t.xm_host, (size_t)nsteps * 6 * sizeof(CUtensorMap), cudaMemcpyHostToDevice, st) !=
            cudaSuccess ||
        cudaEventRecord(t.xm_ev, st) != cudaSuccess)
      return tc_fail(GEIG_ERR_CUDA, "copying per-step tensor maps failed");
    p.xmaps = t.xm_dev;
  }
  for (int v = 0; v < 2; ++v) {
    const char* vb = (const char*)Vbf + (v == 0 ? 0 : t.dx * eb);
    if (own && !update_only) {   // the gathered shadow [world][hi|lo][k][W]
      const int64_t W = own->W;
      if (!make_map3(&maps.bF[v], own->gathered, W, k, own->world, W, 2 * (int64_t)k * W, ATOM, t.BN) ||
          (t.splitb && !make_map3(&maps.bFlo[v], own->gathered + (int64_t)k * W, W, k, own->world, W, 2 * (int64_t)k * W,
                                  ATOM, t.BN)))
        return tc_fail(GEIG_ERR_CUDA, "tensor map encode (owned forward) failed");
    } else {
      if (!make_map(&maps.bF[v], vb, eb, dv[v], k, t.d, ATOM, t.BN))
        return tc_fail(GEIG_ERR_CUDA, "tensor map encode (fused forward) failed");
      if (t.splitb && !make_map(&maps.bFlo[v], vb + (int64_t)k * t.d * eb, eb, dv[v], k, t.d, ATOM, t.BN))
        return tc_fail(GEIG_ERR_CUDA, "tensor map encode (fused forward lo) failed");
    }
    for (int s = 0; s < 2 && !update_only; ++s) {
      const char* zb = (const char*)t.Zb + (int64_t)(v * 2 + s) * k * t.hpad * eb;
      if (!make_map(&maps.bB[v * 2 + s], zb, eb, h, k, t.hpad, ATOM, t.BN))
        return tc_fail(GEIG_ERR_CUDA, "tensor map encode (fused backward) failed");
      if (t.splitb && !make_map(&maps.bBlo[v * 2 + s], zb + (int64_t)4 * k * t.hpad * eb, eb, h, k, t.hpad, ATOM, t.BN))
        return tc_fail(GEIG_ERR_CUDA, "tensor map encode (fused backward lo) failed");
    }
    p.dv[v] = dv[v];
    p.kbF[v] = (int)((dv[v] + ATOM - 1) / ATOM);
  }
  // M tiles per work item: 2 where the grid stays busy (the B-operand tile of
  // each K step then serves 256 rows / columns), else 1
  {
    const int fixed = t.opt_m_tiles;   // geig_set_option(GEIG_OPT_FUSED_M_TILES), 0 = auto
    int nB2 = 0;
    for (int v = 0; v < 2; ++v) nB2 += 2 * (int)((dv[v] + 2 * TC_BM - 1) / (2 * TC_BM));
    p.tmB = fixed ? fixed : (2 * nB2 >= grid_ctas ? 2 : 1);
    // forward: 2 tiles only beside a 2-tile backward or for a long batch — with
    // a 1-tile backward the smaller stage of 1-tile items gives the ring up to
    // 8 stages (config 2: all 8 K blocks of a backward item in flight at once)
    // and halves the forward's split-K partials (same-box A/B over 7 shapes,
    // scripts/mtiles_time.py: 1.5-10 % faster except b = 8192)
    p.tmF = fixed ? fixed : ((rows >= 8 * TC_BM && (p.tmB == 2 || rows >= 64 * TC_BM)) ? 2 : 1);
    if (dev_knob("GEIG_TMF")) p.tmF = std::max(1, std::min(2, atoi(dev_knob("GEIG_TMF"))));   // developer A/B knobs
    if (dev_knob("GEIG_TMB")) p.tmB = std::max(1, std::min(2, atoi(dev_knob("GEIG_TMB"))));
    for (int v = 0; v < 2; ++v) p.mtB[v] = (int)((dv[v] + p.tmB * TC_BM - 1) / (p.tmB * TC_BM));
  }
  {
    // phase U tiles: V'', AV, [Bv], BV over upd.d columns (the own block when
    // column-owned: V, [Bv] pre-offset with row stride upd.ld, AV / BV from
    // the rank's chunk with row stride W)
    const float* src[4] = {upd.V, AV, upd.AUX, BV};
    const int64_t lds = upd.ld ? upd.ld : upd.d, ldp = (own && update_only) ? own->W : upd.d;
    const int64_t lda[4] = {lds, ldp, lds, ldp};
    for (int a = 0; a < 4; ++a)
      if (!make_map(&maps.um.t[a], src[a], 4, upd.d, k, lda[a], (int)upd.segw + 4, 64, false))
        return tc_fail(GEIG_ERR_CUDA, "tensor map encode (update tiles) failed");
  }
  p.rows = rows; p.h = h; p.k = k; p.BN = t.BN; p.d = t.d; p.ldz = t.ldz; p.hpad = t.hpad;
  p.scale = scale;
  p.mtF = (rows + p.tmF * TC_BM - 1) / (p.tmF * TC_BM);
  p.splitsF = std::min(TC_MAX_SPLITS, choose_splits_deep(2 * p.mtF, std::min(p.kbF[0], p.kbF[1]), grid_ctas));
  p.fper = 2 * p.splitsF;   // forward items covering each 128-row tile per step
  p.kbB = (h + ATOM - 1) / ATOM;
  p.idescF = make_idesc(eb, false, t.BN * (t.splitb ? 2 : 1), TC_BM);
  p.idescB = make_idesc(eb, true, t.BN * (t.splitb ? 2 : 1), TC_BM);
  p.Zt = t.Zt;
  p.Zb = (__nv_bfloat16*)t.Zb;
  p.AV = AV;
  p.BV = BV;
  p.upd = upd;
  p.ownW = 0;
  p.chunk = 0;
  p.peer = 0;
  if (own && own->recv) {
    if (own->world > GEIG_MAX_PEERS) return tc_fail(GEIG_ERR_UNSUPPORTED, "peer exchange: more than 8 ranks");
    p.peer = 1;
    p.prank = own->rank;
    p.pworld = own->world;
    p.epoch = own->epoch;
    for (int q = 0; q < own->world; ++q) { p.precv[q] = own->recv[q]; p.pflags[q] = own->flags[q]; }
    if (update_only) {
      p.ownW = own->W;   // the slot sum reads these
      p.chunk = own->chunk;
      int n = 0;
      for (int q = 0; q < own->world; ++q)
        if (q != own->rank) p.upd.vpeer[n++] = own->shadows[q] + (int64_t)own->rank * 2 * k * own->W;
      p.upd.vpeer_n = n;
    } else {
      for (int q = 0; q < own->world; ++q) p.upd.tpeer[q] = own->recv[q];
      p.upd.tpeer_off = (int64_t)own->rank * own->chunk + 2 * (int64_t)k * own->W;
    }
  }
  if (own && !update_only) {
    p.ownW = own->W;
    p.chunk = own->chunk;
    p.AV = own->buf;
    p.BV = own->buf + (int64_t)k * own->W;
    p.upd.tout = own->buf + 2 * (int64_t)k * own->W;
    p.upd.tN = own->world;
    p.upd.tstride = own->chunk;
    p.upd.own0 = (int64_t)own->rank * own->W;
    p.upd.own1 = p.upd.own0 + own->W;
  }
  p.upd.dbg = dbg_ptr();
  p.upd.dbg_mode = dev_knob("GEIG_DBG_MODE") ? atoi(dev_knob("GEIG_DBG_MODE")) : 0;
  p.upd.ga_done = 1;       // phase S forms G^A, G^B from z
  p.upd.pre_reduced = 1;   // G^C, ||v''||^2 in F (warps 2-3), reduction in B (warps 2-3)
  p.split = t.splitb;
  p.splitB = t.splitb;   // bf16x2: the backward B operand (z) as hi + lo too
  p.idescB = make_idesc(eb, true, t.BN * (p.splitB ? 2 : 1), TC_BM);
  p.bwd_y_first = dev_knob("GEIG_BWD_X_FIRST") ? 0 : 1;
  p.pair = pair ? 1 : 0;
  // GEIG_OPT_FUSED_PAIRS 1: non-cooperative cluster launch, grid barriers by
  // grid_bar (the profiler can replay it); 2: cooperative cluster launch
  // (grid.sync of cooperative groups)
  const bool pair_coop = pair && t.opt_pairs == 2;
  p.gbar = (pair && !pair_coop) ? reinterpret_cast<unsigned*>(t.dep + 32) : nullptr;   // own 128-byte line; never reset
  if (pair) {
    p.bwd_y_first = 0;   // CTA c <-> columns [128 c, 128 c + 128)
    if (p.tmB != 2) return tc_fail(GEIG_ERR_STATE, "CTA pairs need 2 M tiles per backward item");
  }
  p.l2_keep = dev_knob("GEIG_L2_KEEP") ? 1 : 0;   // measured: evict-last on a whole view thrashes the state arrays (slower)
  p.dbg_nostore = dev_knob("GEIG_DBG_NOSTORE") ? 1 : 0;   // developer: drop GEMM epilogue stores (timing only)
  p.dbg_mode = dev_knob("GEIG_DBG_MODE") ? atoi(dev_knob("GEIG_DBG_MODE")) : 0;   // developer timing knobs (wrong results)
  const size_t stage_bytes = (size_t)std::max(p.tmF, p.tmB) * TC_BM * 128 + (size_t)t.BN * 128 * (t.splitb ? 2 : 1);
  if ((size_t)std::max(p.tmF, p.tmB) * t.BN * (t.splitb ? 2 : 1) > 256)
    return tc_fail(GEIG_ERR_UNSUPPORTED, "fused step: accumulators exceed the TMEM allocation");
  p.stages = (int)std::min<size_t>(TC_MAX_STAGES, (200 * 1024) / stage_bytes);
  p.bar_off = (uint32_t)((std::max((size_t)p.stages * stage_bytes, upd_bytes) + 15) & ~(size_t)15);
  if (pair && (size_t)5 * 64 * (128 + 4) * 4 > p.bar_off)   // 4 update tiles + the staging tile
    return tc_fail(GEIG_ERR_STATE, "CTA pairs: the staging tile does not fit below the barrier region");
  static_assert((2 * TC_MAX_STAGES + 4) * 8 + 64 * 4 + 8 <= 512, "barrier + scratch area + freebar");
  size_t smem = 1024 + p.bar_off + 512 + 4 * 16 * 32 * 4;
  if (smem > 227 * 1024) return tc_fail(GEIG_ERR_UNSUPPORTED, "fused step: shared memory budget exceeded");
  if (p.early_coef) {   // the coefficient region follows the epilogue tiles when it fits
    if (smem + (size_t)GEIG_COEF_FLOATS * 4 <= 227 * 1024) smem += (size_t)GEIG_COEF_FLOATS * 4;
    else p.early_coef = 0;
  }
  static std::atomic<uint64_t> attr_plain{0}, attr_adam{0};
  if (set_smem_attr_once(attr_plain, (const void*)cca_step_kernel<2, false>, 227 * 1024) != cudaSuccess ||
      set_smem_attr_once(attr_adam, (const void*)cca_step_kernel<2, true>, 227 * 1024) != cudaSuccess)
    return tc_fail(GEIG_ERR_CUDA, "cudaFuncSetAttribute(cca_step_kernel) failed");
  void* args[] = {(void*)&maps, (void*)&p};
  void* kfn = p.upd.adam ? (void*)cca_step_kernel<2, true> : (void*)cca_step_kernel<2, false>;
  if (pair && !pair_coop) {
    // the pair launch is not cooperative: every CTA pair of the grid must be
    // co-resident (one CTA per SM) for its grid barriers
    int ncl = 0;
    cudaLaunchConfig_t oc = {};
    oc.gridDim = dim3(grid_ctas);
    oc.blockDim = dim3(FS_THREADS);
    oc.dynamicSmemBytes = smem;
    cudaLaunchAttribute ca;
    ca.id = cudaLaunchAttributeClusterDimension;
    ca.val.clusterDim.x = 2; ca.val.clusterDim.y = 1; ca.val.clusterDim.z = 1;
    oc.attrs = &ca;
    oc.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&ncl, kfn, &oc) != cudaSuccess || 2 * ncl < grid_ctas) {
      // not every pair fits at once (another context holds SMs, MPS limits):
      // this plan falls back to one CTA per item, cooperative launch
      cudaGetLastError();
      t.opt_pairs = 0;
      return fused_cca_step(t, X, Y, nsteps, b, scale, Vbf, AV, BV, upd_in, grid_in, upd_bytes_in, st, products_only,
                            tables, update_only, own, pair_grid);
    }
  }
  cudaError_t e = launch_coop(kfn, dim3(grid_ctas), dim3(FS_THREADS), args, smem, st, t.l2win, pair ? 2 : 0, !pair || pair_coop);
  if (e != cudaSuccess) return tc_fail(GEIG_ERR_CUDA, std::string("cca_step_kernel launch: ") + cudaGetErrorString(e));

  return GEIG_OK;
}

}}  // namespace geig::tc
