/*
 * geig.h — C ABI of the B200-native gamma-EigenGame hot path
 * (arxiv 2206.04993, "The Generalized Eigenvalue Problem as a Nash
 * Equilibrium").  Citations are PAPER.md line numbers with the section /
 * algorithm they fall in.
 *
 * The library solves the top-k generalized eigenvalue problem A v = lambda B v
 * (§1) by running Alg. 2 ("Stochastic gamma-EigenGame",
 * PAPER.md:996-1030): k players hold unit vectors v_i (strategies,
 * PAPER.md:871) and auxiliary vectors [Bv]_i; one step forms the minibatch
 * products A_t v_j and B_t v_j for all players, the k x k inner-product
 * tables, the normalised parents y_j = v_j / sqrt(max(<v_j,[Bv]_j>, rho)),
 * the lower-triangular penalty sums, the v_i ascent + sphere retraction and
 * the [Bv]_i running-average update.
 *
 * Layouts (all row-major, all device memory unless a function says HOST):
 *   d = dx + dy (CCA) or d (dense).
 *   V, AUX ([Bv]), AV, BV : k x d float32, row i = player i (player-major,
 *                           each player's d-vector contiguous).
 *   CCA views X : b x dx, Y : b x dy, one sample per row (fp32 or bf16).
 *   Dense A, B : d x d symmetric, fp32 (or bf16), row-major.
 *   Gram tables : k x k float32, row i, column j.
 *
 * Minibatch estimates (§3, Alg. 2 line 7 "unbiased estimates
 * using independent data batches"), reading R1: the b rows of a
 * step are split into halves; rows [0,h) estimate A, rows [h,2h) estimate B,
 * h = floor(b/2):
 *   A_t v = (1/h) [X1^T (Y1 v_y) ; Y1^T (X1 v_x)]
 *   B_t v = (1/h) [X2^T (X2 v_x) ; Y2^T (Y2 v_y)]      (PAPER.md:831 CCA)
 *
 * L2: the solver's state arena is marked persisting in L2 through an access-
 * policy window attached to the library's own cooperative launches (no
 * stream attribute is changed).  Side effect: geig_create raises the
 * device's persisting-L2 set-aside (cudaLimitPersistingL2CacheSize) to at
 * most the arena size and never lowers it; geig_destroy resets the device's
 * persisting lines (cudaCtxResetPersistingL2Cache).
 *
 * Ownership: the solver owns V, AUX and its scratch (allocated in
 * geig_create, freed in geig_destroy).  Every pointer argument is owned by the
 * caller and only read (or written, for outputs) during the call / the
 * stream-ordered work it enqueues.  All device work is enqueued on the
 * solver's stream (geig_set_stream); calls return without synchronising
 * except the *_host variants and geig_sync.
 *
 * Errors: every function returns GEIG_OK (0) or a nonzero geig_status; the
 * message of the last error of the calling thread is geig_last_error().
 * Invalid sizes/pointers -> GEIG_ERR_ARG; CUDA failures -> GEIG_ERR_CUDA;
 * configurations the compiled kernels do not cover (e.g. k > 128) ->
 * GEIG_ERR_UNSUPPORTED.  Nothing falls back to a CPU path.
 */
#ifndef GEIG_H_
#define GEIG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct geig_solver geig_solver;

typedef enum {
  GEIG_OK = 0,
  GEIG_ERR_ARG = 1,
  GEIG_ERR_CUDA = 2,
  GEIG_ERR_UNSUPPORTED = 3,
  GEIG_ERR_STATE = 4
} geig_status;

/* Problem family (PAPER.md:765 generic GEP; PAPER.md:828 CCA). */
typedef enum { GEIG_DENSE = 0, GEIG_CCA = 1 } geig_problem;

/* Arithmetic of the minibatch products (the GEMMs):
 *  GEIG_MATH_F32   : FFMA fp32 on CUDA cores (exactness-check variant)
 *  GEIG_MATH_BF16  : tcgen05 tensor cores, bf16 operands, fp32 accumulate
 *  GEIG_MATH_TF32  : tcgen05 tensor cores, tf32 operands, fp32 accumulate
 *                    (fp32 data; the CCA backward reads X^T as an MN-major
 *                    tf32 operand in the 128-byte / 32-byte-chunk swizzle)
 *  GEIG_MATH_3XTF32: tcgen05 tf32 with hi/lo split (fp32 data): the
 *                    streamed A tile is split in shared memory into
 *                    tf32_rna(a) + (a - hi), B arrives as hi / lo planes,
 *                    A_hi B_hi + A_hi B_lo + A_lo B_hi per K step
 *                    (~fp32-accurate tensor-core products)
 *  GEIG_MATH_BF16X2: tcgen05 bf16 with the V and Z operands carried as
 *                    hi + lo bf16 halves (one N = 2k MMA per K step): the
 *                    bf16 data is exact, so the products are ~fp32-accurate
 * The Gram tables and the update are always fp32. */
typedef enum {
  GEIG_MATH_F32 = 0,
  GEIG_MATH_BF16 = 1,
  GEIG_MATH_TF32 = 2,
  GEIG_MATH_3XTF32 = 3,
  GEIG_MATH_BF16X2 = 4
} geig_math;

/* Storage dtype of X, Y (CCA) or A, B (dense). */
typedef enum { GEIG_DATA_F32 = 0, GEIG_DATA_BF16 = 1 } geig_dtype;

/* Create a solver for k players (1 <= k <= 128) on CUDA device `device`.
 * dense: dx = d, dy = 0.  cca: dx, dy >= 1.  rho >= 0 is the clipping floor of
 * Alg. 2 line 8 ("scalar rho lower bounding sigma_min(B)").
 * max_rows bounds the batch size b of later geig_products_cca calls (scratch
 * is sized for it; 0 for dense).  V and AUX are zero until geig_init_state /
 * geig_set_state. */
geig_status geig_create(geig_solver** out, int problem, int64_t dx, int64_t dy,
                        int32_t k, int math, int data_dtype, double rho,
                        int64_t max_rows, int device);

/* Destroy the solver and free everything it owns (NULL is a no-op). */
geig_status geig_destroy(geig_solver* s);

/* Stream (a cudaStream_t passed as void*; NULL = legacy default stream).
 * Switching to a different stream first waits for the work already enqueued
 * on the old one (the solver's fused launches must run in call order). */
geig_status geig_set_stream(geig_solver* s, void* stream);

/* Block the host until all work enqueued by this solver has finished. */
geig_status geig_sync(geig_solver* s);

/* Alg. 2 lines 2-3: from the raw draws G (k x d, device,
 * fp32; v_i ~ N(0, I_d) drawn by the caller) set v_i = G_i/||G_i|| and
 * [Bv]_i = v_i.  Also resets the step counter. */
geig_status geig_init_state(geig_solver* s, const float* G);

/* Overwrite / read the state (V, AUX: k x d fp32, device). AUX may be NULL.
 * Internally the retraction v <- v/||v|| of Alg. 2 line 17 is applied when
 * the next update reads the state; geig_get returns the retracted
 * (unit-norm) v_i. */
geig_status geig_set_state(geig_solver* s, const float* V, const float* AUX);
geig_status geig_get(geig_solver* s, float* V, float* AUX);

/* Minibatch products for CCA (stage a1): AV = scale * A_t-sum V, BV likewise,
 * i.e. AV_j = scale * [X1^T (Y1 v_jy) ; Y1^T (X1 v_jx)] and
 * BV_j = scale * [X2^T (X2 v_jx) ; Y2^T (Y2 v_jy)] with halves of b rows
 * (reading R1).  scale = 1/h gives A_t v, B_t v; multi-GPU callers pass
 * 1/(world * h) and all-reduce (Appendix F).  X: b x dx,
 * Y: b x dy (data_dtype), row stride = dx / dy elements.  2 <= b <= max_rows.
 * AV, BV: k x d fp32 outputs (overwritten). */
geig_status geig_products_cca(geig_solver* s, const void* X, const void* Y,
                              int64_t b, float scale, float* AV, float* BV);

/* Dense products (configs 0, 4): AV[:, r0:r1] = A[r0:r1, :] V^T, BV likewise
 * (rows r0..r1 of the symmetric A, B; a row shard for multi-GPU).  A, B:
 * (r1-r0) x d row-major slices (row stride d), data_dtype.  Only columns
 * [r0, r1) of AV, BV are written. */
geig_status geig_products_dense(geig_solver* s, const void* A, const void* B,
                                int64_t r0, int64_t r1, float* AV, float* BV);

/* Stages a2-a4 (Alg. 2 lines 8-19): from the products
 * AV_j = A_t v_j, BV_j = B_t v_j of the CURRENT state, form the Gram tables,
 * y_j / [By]_j normalisation with the rho floor, rewards and lower-triangular
 * penalties, v_i <- (v_i + eta grad_i)/||.||, [Bv]_i += gamma (BV_i - [Bv]_i).
 * All players read the iteration-start snapshot (parfor). */
geig_status geig_update(geig_solver* s, const float* AV, const float* BV,
                        double eta, double gamma);

/* Multi-GPU form of the step (Appendix F) with the Gram
 * tables aggregated beside the products.  geig_products_cca_tables writes,
 * in ONE launch of the fused kernel's phases F, S, B, this rank's scaled
 * partial products AV, BV (like geig_products_cca) and into T the partial
 * sums of the tables that depend on the rank's rows — tri(G^A) and diag(G^B)
 * formed from the forward products (Alg. 2 lines 8-11; reading R3') — while
 * G^C and ||v''||^2, which depend only on the replicated state, stay in the
 * solver.  The caller sums AV, BV and T over the ranks (one all-reduce when
 * the three are adjacent in one buffer) and calls geig_update_tables, which
 * runs the update from the summed products and tables without re-forming
 * the Gram tables.  T: geig_table_floats(s) device floats.  Needs the fused
 * path (bf16 / bf16x2 math, k <= 64, d % 4 == 0): GEIG_ERR_UNSUPPORTED
 * otherwise (use geig_products_cca + geig_update).  The state must not change
 * between the two calls. */
int64_t geig_table_floats(const geig_solver* s);
geig_status geig_products_cca_tables(geig_solver* s, const void* X, const void* Y,
                                     int64_t b, float scale, float* AV, float* BV,
                                     float* T);
geig_status geig_update_tables(geig_solver* s, const float* AV, const float* BV,
                               const float* T, double eta, double gamma);

/* Column-owned multi-GPU step (the products reduce-scattered instead of
 * all-reduced; Appendix F, "parallelized the estimation of the
 * matrix-vector products ... then aggregated this information across
 * machines"; Alg. 2 lines 8-19 are separable over feature columns once the
 * k x k tables are summed).  Rank `rank` of `world` owns the columns
 * [rank W, (rank + 1) W), W = d / world, and keeps V, [Bv] current on them
 * only.  Per step:
 *   geig_products_cca_owned  one launch (forward, split-K sums, backward):
 *                            buf = world chunks of geig_owned_chunk_floats
 *                            floats, chunk r = [AV | BV (k x W each, columns
 *                            of rank r, row stride W) | tables (the rank's
 *                            partial G^A, G^B from its rows and G^C,
 *                            ||v''||^2 from its own columns)];
 *   reduce-scatter (sum) of buf -> the rank's chunk (caller, e.g. NCCL);
 *   geig_update_owned        the update of the own columns from the summed
 *                            chunk; writes the rank's block of the gathered
 *                            bf16 shadow;
 *   all-gather of the shadow blocks (caller): geig_shadow_buffer gives the
 *                            device buffer [world][hi|lo][k][W] bf16 and the
 *                            bytes per rank (rank r's block at r * bytes).
 * geig_set_partition(s, 1, 0) switches back.  Needs CCA, bf16 / bf16x2 math,
 * k <= 64, d % (64 world) == 0 and dx % 64 == 0 (GEIG_ERR_UNSUPPORTED).  While
 * partitioned, geig_get returns the raw (unretracted) v'' — only the own
 * columns are current and the retraction needs every rank's columns; the
 * caller gathers the blocks and divides by the row norms.  Errors:
 * GEIG_ERR_STATE without a partition; GEIG_ERR_ARG for bad sizes, NULL or
 * unaligned (16-byte) buffers. */
geig_status geig_set_partition(geig_solver* s, int world, int rank);
int64_t geig_owned_chunk_floats(const geig_solver* s);
geig_status geig_shadow_buffer(geig_solver* s, void** ptr, int64_t* bytes_per_rank);
geig_status geig_products_cca_owned(geig_solver* s, const void* X, const void* Y,
                                    int64_t b, float scale, float* buf);
geig_status geig_update_owned(geig_solver* s, const float* chunk, double eta,
                              double gamma);

/* Peer-memory form of the column-owned step (one process per GPU over
 * NVLink peer memory; Appendix F, with the reduce-scatter and
 * the all-gather folded into the kernels): instead of NCCL collectives,
 *  - the products launch stores every column's AV | BV and the rank's table
 *    row straight into the OWNER's receive buffer (slot = this rank) from
 *    the backward epilogue, and then raises this rank's receive flag at
 *    every owner;
 *  - the update launch waits for the flags of all senders, sums the slots in
 *    rank order (deterministic: the same sum as a reduce-scatter of rank
 *    order), updates the own columns, writes its bf16 shadow block into
 *    EVERY rank's gathered shadow, and raises its shadow flag at every rank;
 *  - the next products launch waits for every rank's shadow flag.
 * Flags are 32-bit step epochs (monotonic, never reset) at system scope.
 * Setup: after geig_set_partition, geig_peer_buffers gives this rank's
 * receive buffer (world x geig_owned_chunk_floats floats) and flag words
 * (device memory, for CUDA IPC export with geig_ipc_handle); with
 * geig_shadow_buffer's gathered shadow these three are exchanged among the
 * ranks (geig_ipc_open maps another process's buffer) and passed to
 * geig_set_peers as arrays of `world` device pointers (entry `rank` = this
 * rank's own buffers).  geig_step_cca_peer then runs one step (two
 * launches); the ranks must call it in lockstep (the kernels wait on each
 * other's flags: a rank that never calls traps the others' kernels after
 * seconds).  Up to 8 ranks.  Errors: GEIG_ERR_STATE without a partition /
 * peers; GEIG_ERR_ARG for NULL, unaligned or inconsistent pointers. */
geig_status geig_peer_buffers(geig_solver* s, void** recv, int64_t* recv_bytes,
                              void** flags, int64_t* flags_bytes);
geig_status geig_set_peers(geig_solver* s, void* const* recv, void* const* shadow,
                           void* const* flags);
geig_status geig_step_cca_peer(geig_solver* s, const void* X, const void* Y,
                               int64_t b, float scale, double eta, double gamma);
/* The two launches of geig_step_cca_peer separately (e.g. several ranks
 * emulated in one process: every rank's products, then every rank's
 * update); GEIG_ERR_STATE when called out of order. */
geig_status geig_products_cca_peer(geig_solver* s, const void* X, const void* Y,
                                   int64_t b, float scale);
geig_status geig_update_peer(geig_solver* s, double eta, double gamma);

/* CUDA IPC of device allocations between the processes of one node:
 * geig_ipc_handle writes the 64-byte handle of dev_ptr (the base of a
 * device allocation of this process); geig_ipc_open maps another process's
 * handle (peer access enabled lazily); geig_ipc_close unmaps it. */
geig_status geig_ipc_handle(const void* dev_ptr, void* handle64);
geig_status geig_ipc_open(const void* handle64, void** dev_ptr);
geig_status geig_ipc_close(void* dev_ptr);

/* One full step = products + update on the solver's scratch.  On the bf16
 * tensor-core path with k <= 64 the whole step is ONE persistent cooperative
 * kernel (forward GEMM, split-K reduction, backward GEMM, Gram tables and
 * update separated by grid barriers); otherwise products then update. */
geig_status geig_step_cca(geig_solver* s, const void* X, const void* Y,
                          int64_t b, double eta, double gamma);
geig_status geig_step_dense(geig_solver* s, const void* A, const void* B,
                            double eta, double gamma);

/* Alg. 1's loop (deterministic full-batch game): nsteps
 * consecutive dense steps on the same d x d matrices A, B (device, row-major,
 * the solver's data dtype).  Equivalent to nsteps calls of geig_step_dense.
 * With fp32 math, k <= 16 and A, B small enough to sit in one SM's shared
 * memory (d <= ~100 at fp32), the steps run in ONE launch of the one-CTA
 * small-problem kernel with A, B resident (GEIG_OPT_SMALL_STEP); otherwise
 * products + update per step.  Errors: GEIG_ERR_ARG for NULL pointers or
 * nsteps outside [0, 2^30]; GEIG_ERR_STATE for a CCA solver. */
geig_status geig_run_dense(geig_solver* s, const void* A, const void* B,
                           int64_t nsteps, double eta, double gamma);

/* Alg. 2's loop over t ("for t = 1 : T"): nsteps
 * consecutive CCA steps, step i on the minibatch (X[i], Y[i]) — host arrays
 * of nsteps DEVICE pointers, each view b x d_view row-major in the solver's
 * data dtype (batches may repeat).  Equivalent to nsteps calls of
 * geig_step_cca (same kernels and arithmetic, bit-identical state); on the
 * fused tensor-core path (bf16 / bf16x2, k <= 64) the steps run inside ONE
 * persistent cooperative launch (grid barrier between steps), removing the
 * per-step launch gap.  The pointer arrays are read during the call only.
 * Errors: GEIG_ERR_ARG for NULL arrays or nsteps outside [0, 2^20]; the
 * errors of geig_step_cca otherwise. */
geig_status geig_run_cca(geig_solver* s, const void* const* X,
                         const void* const* Y, int64_t b, int64_t nsteps,
                         double eta, double gamma);

/* nsteps CCA steps end to end from HOST buffers (X_host[t], Y_host[t]:
 * pinned host memory, b x d_view rows each): the host->device copy of batch
 * t + 1 (a copy stream, double-buffered device staging) overlaps step t on
 * the solver's stream; after every step its k x k normalised G^A table is
 * copied back into ga_host (nullable; pinned, k*k floats; the last step's
 * table remains).  Synchronises before returning; *h2d / *d2h = bytes
 * moved (nullable).  Same results as nsteps geig_step_cca calls on the
 * device copies.  Errors: those of geig_step_cca; GEIG_ERR_ARG for NULL
 * arrays. */
geig_status geig_run_cca_host(geig_solver* s, const void* const* X_host,
                              const void* const* Y_host, int64_t b, int64_t nsteps,
                              double eta, double gamma, float* ga_host,
                              int64_t* h2d, int64_t* d2h);

/* Variants of the update, applied by every following step (geig_update,
 * geig_step_cca, geig_run_cca, geig_step_dense); resident update only
 * (k <= 64, otherwise GEIG_ERR_UNSUPPORTED).
 *
 * geig_set_smooth: Alg. 3, "Smooth Stochastic gamma-EigenGame"
 * (PAPER.md:1597-1621): the clipped denominators of Alg. 2 l.8 are replaced
 * by [<v,Bv>]_j = exp(log rho + (log nu - log rho) sigma(z_j)) (l.7), and
 * z_i += gamma (<v_i,[Bv]_i> - [<v,Bv>]_i) [<v,Bv>]_i (log nu - log rho)
 * sigma(z_i)(1 - sigma(z_i)) (l.14, l.21; ascent sign as in the box, DESIGN
 * reading R6).  nu (upper bound of lambda_max(B)) must exceed rho > 0;
 * nu <= 0 switches back to Alg. 2.  Resets z to 0 (l.4).  Errors:
 * GEIG_ERR_ARG for rho >= nu or rho == 0.
 *
 * geig_smooth_state: copy the k values of z in (device z_in, may be NULL)
 * and/or out (device z_out, may be NULL), stream-ordered.  GEIG_ERR_STATE
 * when Alg. 3 is off.
 *
 * geig_set_adam: Adam(b1, b2, eps) ascent on v_i (Appendix H)
 * with the Alg. 2 (or 3) direction as the gradient and eta of each step as
 * the learning rate: m = b1 m + (1-b1) g, s = b2 s + (1-b2) g^2,
 * v' = v + eta (m / (1-b1^t)) / (sqrt(s / (1-b2^t)) + eps), then the sphere
 * retraction (l.17).  Zeroes the moments (k x d fp32 each, owned by the
 * solver) and the step count t.  b1 < 0 switches back to plain ascent.
 * Needs d % 4 == 0. */
geig_status geig_set_smooth(geig_solver* s, double nu);
geig_status geig_smooth_state(geig_solver* s, const float* z_in, float* z_out);
geig_status geig_set_adam(geig_solver* s, double b1, double b2, double eps);

/* End-to-end step from HOST buffers (pinned or pageable): copies X, Y host ->
 * device (stream-ordered), runs geig_step_cca and copies the k x k Gram table
 * GA (A-table of the step) back to `ga_host` (may be NULL), then synchronises.
 * Returns the bytes moved in *h2d / *d2h (may be NULL). */
geig_status geig_step_cca_host(geig_solver* s, const void* X_host,
                               const void* Y_host, int64_t b, double eta,
                               double gamma, float* ga_host, int64_t* h2d,
                               int64_t* d2h);

/* Diagnostics of the last geig_update (device outputs, k x k fp32 each, any
 * may be NULL): GA[i][j] = <v_i, AV_j>, GC[i][j] = <v_i, [Bv]_j>,
 * GB[i][j] = <v_i, BV_j> (only the diagonal of GB is computed; the rest is
 * zero; for GA and GC only i >= j is computed, the rest is zero) — the
 * "k x k inner-product tables" of the north star, from the iteration-start
 * state. */
geig_status geig_get_gram(geig_solver* s, float* GA, float* GB, float* GC);

/* Schedule options of a solver (they change which kernels run and how work
 * is tiled, never the arithmetic of Alg. 2; results differ at most by
 * floating-point summation order).  No environment variable is read by the
 * library.
 *  GEIG_OPT_FUSED_M_TILES   : 128-row M tiles per work item of the fused
 *                             step's GEMM phases (0 = auto: backward 2 where
 *                             the 256-column tiles keep the grid busy, else 1;
 *                             forward 2 beside a 2-tile backward or for
 *                             batches of >= 8192 rows, else 1; 1; 2)
 *  GEIG_OPT_SMALL_STEP      : 1 = (default) fp32 (GEIG_MATH_F32) steps of
 *                             small problems — k <= 16, KP d <= 8192 (KP = k rounded up to 8 or 16) and
 *                             the state plus a chunk of rows (CCA) or A and
 *                             B (dense) within one SM's 227 KB of shared
 *                             memory, 16-byte aligned rows — run as ONE
 *                             launch of a one-CTA kernel per call
 *                             (geig_step_cca / geig_run_cca /
 *                             geig_step_dense / geig_run_dense: the whole
 *                             run in one launch, state resident in shared
 *                             memory, each batch byte read once); 0 = the
 *                             staged products + update kernels
 *  GEIG_OPT_FUSED_PAIRS     : 1 = (default) full fused steps (geig_step_cca,
 *                             geig_run_cca; bf16 / bf16x2, views a multiple of
 *                             256 wide) run on CTA pairs (thread-block
 *                             clusters of 2): the two halves of each
 *                             256-column backward tile are one pair's work and
 *                             the backward accumulators move into the update
 *                             through distributed shared memory instead of
 *                             global memory; 0 = one CTA per item
 *  GEIG_OPT_SMALL_CLUSTER   : CTAs (a thread-block cluster) of the small-problem
 *                             CCA step: each takes a contiguous share of every
 *                             batch's rows and owns a block of the update's
 *                             columns; the products, Gram tables and v'' are
 *                             combined through distributed shared memory in
 *                             rank order (deterministic).  0 = (default) auto:
 *                             the largest power of 2 <= 8 leaving >= 64 rows
 *                             and >= 16 columns per CTA; 1, 2, 4, 8 = forced
 *  GEIG_OPT_GRAM_TC         : 1 = (default) the streamed update (k > 64) of a
 *                             tf32 / 3xTF32 solver forms its Gram tables
 *                             G^A, G^C on the tensor cores (one launch of
 *                             split-K partial rows before the update); 0 =
 *                             FFMA in the update kernel
 *  GEIG_OPT_STAGED_PRODUCTS : 1 = geig_products_cca runs the three-launch
 *                             staged tcgen05 products (forward GEMM, z
 *                             reshuffle, backward GEMM) instead of phases
 *                             F, S, B of the fused kernel; 0 = fused (default)
 * Errors: GEIG_ERR_ARG for an unknown option or a value out of range. */
typedef enum { GEIG_OPT_FUSED_M_TILES = 1, GEIG_OPT_STAGED_PRODUCTS = 2, GEIG_OPT_SMALL_STEP = 3,
               GEIG_OPT_FUSED_PAIRS = 4, GEIG_OPT_GRAM_TC = 5,
               GEIG_OPT_SMALL_CLUSTER = 6 } geig_option;
geig_status geig_set_option(geig_solver* s, int option, int64_t value);

/* Phase durations (ns, %globaltimer of CTA 0) of the last update:
 * out[0] Gram partials, out[1] grid reduction, out[2] coefficients + fused
 * update; if the last step ran the fused single-launch kernel
 * (geig_step_cca, bf16, k <= 64) out[3] = forward products phase and
 * out[4] = reshuffle + backward products phases, else 0.  Synchronises the
 * solver's stream. */
geig_status geig_update_phase_ns(geig_solver* s, int64_t* out);

/* Number of kernel launches this solver has enqueued since creation. */
int64_t geig_launch_count(const geig_solver* s);

/* Human-readable message of the last error on this thread ("" if none). */
const char* geig_last_error(void);

/* Library version string. */
const char* geig_version(void);

#ifdef __cplusplus
}
#endif

#endif /* GEIG_H_ */
