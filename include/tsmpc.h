/*
 * tsmpc.h — C ABI of the B200-native scenario-tree APG solver (libtsmpc.so).
 *
 * This is the drop-in boundary for the reference's accelerated dual proximal
 * gradient path.  The reference (`treesmpc`, pure Python) has no FFI layer; the
 * entry points below replace its Python solver functions one for one and are
 * bound from Python with ctypes by `paper_1604_01074_b200/_native.py`
 * (see INTEGRATION.md for the binding a reference maintainer would add):
 *
 *   tsmpc_plan_create     replaces the per-(model, tree) setup that the reference
 *                         does inside SolveContext.__init__
 *                         (pkg/src/treesmpc/factor.py:86-128) plus the upload of
 *                         factor_step outputs (factor.py:67-76) and the dual
 *                         scaling (engine.py:120-143, 239-277).
 *   tsmpc_set_cache       uploads one StageCache (elimination.py:54-65,114-158).
 *   tsmpc_solve           engine.solve (engine.py:485-601): fixed-iteration APG
 *                         loop, ergodic averages, residual, duality gap.
 *   tsmpc_solve_step      factor.solve_step / SolveContext.solve
 *                         (factor.py:174-217).
 *   tsmpc_prox            engine.prox_g (engine.py:157-183).
 *   tsmpc_dual_operator   one application of the scaled dual-gradient operator used
 *                         by engine.compute_lambda (engine.py:286-337).
 *
 * Conventions: every array is host memory, float64, C-contiguous row-major,
 * with the reference's shapes (points.py:17-57): per-node arrays have n_nodes
 * rows, per-edge arrays n_edges = n_nodes-1 rows, row e <-> node e+1.  Device
 * memory is owned by the plan.  A plan is not thread-safe; use one host thread
 * per plan.  Functions return TSMPC_OK (0) or a negative status; the message of
 * the last failure on the calling thread is returned by tsmpc_last_error().
 */
#ifndef TSMPC_H
#define TSMPC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSMPC_OK               0
#define TSMPC_ERR_DIMENSION   -1   /* -> DimensionError  */
#define TSMPC_ERR_VALIDATION  -2   /* -> ValidationError */
#define TSMPC_ERR_CUDA        -3   /* -> DeviceError     */
#define TSMPC_ERR_NCCL        -4   /* -> DeviceError     */
#define TSMPC_ERR_ARGUMENT    -5   /* NULL / out-of-range argument */

typedef struct tsmpc_plan tsmpc_plan;

/* Model, factor matrices, scaling and tree of one plan (all host pointers). */
typedef struct tsmpc_problem {
  int32_t n_x, n_u, n_v, n_d, n_e; /* states, inputs, reduced inputs, demands, junctions */
  int32_t N;                       /* horizon (stages 0..N)                            */
  int32_t n_nodes;
  /* model / factor (factor.py:38-76, elimination.py:34-103) */
  const double* A;        /* n_x*n_x                                   */
  const double* B;        /* n_x*n_u                                   */
  const double* L;        /* n_u*n_v  orthonormal basis of ker(E)      */
  const double* Bbar;     /* n_x*n_v  = B L                            */
  const double* Phi;      /* n_v*n_x  = -Rbar^{-1} Bbar'               */
  const double* Psi;      /* n_v*n_u  = -Rbar^{-1} L'                  */
  const double* Wu;       /* n_u*n_u  control-increment weight         */
  const double* E;        /* n_e*n_u  junction matrix                  */
  const double* E_pinvT;  /* n_e*n_u  = ((E')(E E')^{-1})'  (gap)      */
  const double* u_min; const double* u_max;   /* n_u */
  const double* x_min; const double* x_max;   /* n_x */
  const double* x_s;                          /* n_x */
  double W_alpha, Wx, gamma_d;
  /* dual scaling (engine.py:120-143); NULL -> identity */
  const double* sig_stage;   /* N      */
  const double* zeta_stage;  /* N      */
  const double* psi_stage;   /* N*n_u  */
  /* tree (tree.py:31-94) */
  const int64_t* stage_starts; /* N+2     */
  const int64_t* anc;          /* n_nodes */
  const int64_t* child_start;  /* n_nodes */
  const int64_t* child_stop;   /* n_nodes */
  const double* prob;          /* n_nodes */
  /* optional block-structured kernel basis (precompute.structured_basis):
   * Ls = L M spans ker(E) with Ls' Wu Ls = diag(lam_s).  When present, A is
   * diagonal and every leaf chain fits a tile, tsmpc_solve runs the sparse
   * persistent kernel; NULL -> dense fused-operator kernel only. */
  const double* Ls;            /* n_u*n_v */
  const double* lam_s;         /* n_v     */
  const double* Ms;            /* n_v*n_v */
} tsmpc_problem;

/* Host buffers filled by tsmpc_solve; any pointer may be NULL to skip it. */
typedef struct tsmpc_result {
  double* u0;          /* n_u             = u_avg[0]                          */
  double* x;           /* n_nodes*n_x     last primal iterate                 */
  double* u;           /* n_edges*n_u                                          */
  double* x_avg;       /* n_nodes*n_x     ergodic states                       */
  double* u_avg;       /* n_edges*n_u     ergodic controls                     */
  double* dual_sig;    /* n_edges*n_x     final dual, scaled coordinates       */
  double* dual_zeta;   /* n_edges*n_x                                          */
  double* dual_psi;    /* n_edges*n_u                                          */
  double* resid_trace; /* iters (only with TSMPC_RECORD_RESIDUALS)             */
  double residual_inf; /* out */
  double gap;          /* out (NaN when TSMPC_SKIP_GAP)                        */
  double device_ms;    /* out: CUDA-event time of the on-device iteration loop */
  int32_t iterations;  /* out: iterations actually run                         */
  double device_total_ms;   /* out: CUDA-event time of loop + duality gap        */
  int64_t kernel_launches;  /* out: libtsmpc kernels launched by this call       */
  double* gap_trace;   /* iters (only with TSMPC_GAP_TRACE): duality gap after every
                          iteration, engine.py:577-582                              */
} tsmpc_result;

#define TSMPC_RECORD_RESIDUALS 1   /* residual_inf of every iteration -> resid_trace */
#define TSMPC_SKIP_GAP         2   /* do not evaluate the duality gap               */
#define TSMPC_KEEP_DEVICE      4   /* leave results on the device (no D2H but u0)   */
#define TSMPC_WARM_DEVICE      8   /* warm start from the last solve's final dual (HBM) */
#define TSMPC_GAP_TRACE       16   /* duality gap of every iteration -> gap_trace (implies
                                      RECORD_RESIDUALS; single-GPU structured-basis plans;
                                      one launch per iteration + the gap's kernels)       */

/* Problem / tree geometry and device planning.  Returns NULL on failure. */
tsmpc_plan* tsmpc_plan_create(const tsmpc_problem* prob, int device);
void tsmpc_plan_destroy(tsmpc_plan* plan);

/* Subtree sharding across the GPUs of one node (one process per GPU).  Rank 0
 * creates an NCCL unique id (128 bytes) with tsmpc_nccl_unique_id and shares it
 * (e.g. torch.distributed broadcast); every rank then creates its shard plan.
 * The leaf chains are split by the trunk node they hang from; a trunk position
 * with one rank's chains below is computed by that rank only, the positions with
 * several ranks' chains below ("mixed", the top of the tree) are replicated.
 * tsmpc_solve on a shard plan runs, per iteration, phase 1 (backward, bottom-up
 * sums below the cut) -> ncclAllReduce of the cut exchange rows (per cut
 * position its bottom-up sums, per mixed position its chain-head sums; one
 * contributor per entry: exact) -> phase 2, and returns results for
 * tsmpc_plan_edges(plan, 0, ...) only; the residual is the max over ranks; the
 * duality gap is evaluated on the state assembled across ranks.
 * Replaces the reference's intra-stage thread pool (pkg/src/treesmpc/_parallel.py,
 * factor.py:107-128) at the node level.  Requires the structured-basis kernel. */
int tsmpc_nccl_unique_id(uint8_t* out128);
tsmpc_plan* tsmpc_plan_create_shard(const tsmpc_problem* prob, int device, int32_t rank,
                                    int32_t world, const uint8_t* nccl_id128);
/* Several shard plans of one tree on ONE device, created with nccl_id128 = NULL
 * (local shard plans, ranks 0..n-1 of world n, plans[r] = rank r), solved in
 * lockstep in one process: per iteration, phase 1 of every shard, an in-place
 * device sum of their cut exchange rows (the exchange ncclAllReduce performs
 * across GPUs), phase 2 of every shard; residuals are max-reduced the same way.
 * outs[r] receives rank r's rows, as tsmpc_solve on an NCCL shard plan would.
 * Exercises the multi-rank split on a single GPU (the kernels of different
 * shards never wait on each other).  n <= 8; warm starts from host arrays are
 * not taken (TSMPC_WARM_DEVICE is). */
int tsmpc_solve_group(tsmpc_plan* const* plans, int32_t n, const double* p, int32_t iters,
                      double lam, const double* theta, const double* coef, int32_t flags,
                      tsmpc_result* outs);
/* Single-process multi-GPU (one host thread drives n GPUs): n shard plans of one
 * tree, rank r on devices[r], with communicators from ncclCommInitAll;
 * plans_out[r] receives rank r's plan (destroy each with tsmpc_plan_destroy).
 * tsmpc_solve_multi runs one solve over all of them -- per iteration phase 1 on
 * every GPU, the cut-row all-reduces inside one NCCL group, phase 2 on every
 * GPU -- and fills outs[r] as tsmpc_solve fills a shard plan's result (the
 * duality gap on the assembled state).  This is what engine.solve runs for
 * SolverConfig(devices=(...)): the sharded solve behind the reference API. */
int tsmpc_plans_create_multi(const tsmpc_problem* prob, const int32_t* devices, int32_t n,
                             tsmpc_plan** plans_out);
/* The cut exchange inside the persistent kernel, over peer memory (NVLink /
 * NVSwitch), instead of two launches and an ncclAllReduce per iteration: once
 * both phases of an iteration are in one launch, each rank's CTAs store their
 * slice of the exchange rows into every rank's receive rows, fence at system
 * scope and bump every rank's arrival counter; each rank waits for all arrivals
 * of the iteration, sums the world rows (one non-zero contributor per entry:
 * exact) and continues with phase 2 -- one launch per solve, the last tile's fill
 * kept in shared memory across iterations.  Process per GPU: every rank exports
 * its blob (tsmpc_plan_peer_handles, CUDA IPC handles of its receive rows and
 * counter, TSMPC_PEER_BLOB_BYTES), the ranks all-gather them (rank order), and
 * every rank calls tsmpc_plan_peer_open with the world blobs; all ranks must then
 * use the exchange (or all call tsmpc_plan_peer_close).  tsmpc_plans_create_multi
 * enables it itself when every device pair has peer access (TSMPC_NO_PEER=1
 * keeps the NCCL path).  A rank whose peers do not arrive within ~2 s aborts the
 * launch (TSMPC_ERR_CUDA) instead of hanging.  Wide shard plans only. */
#define TSMPC_PEER_BLOB_BYTES 160
int tsmpc_plan_peer_handles(const tsmpc_plan* plan, uint8_t* blob);
int tsmpc_plan_peer_open(tsmpc_plan* plan, const uint8_t* blobs, int32_t world);
int tsmpc_plan_peer_close(tsmpc_plan* plan);
int tsmpc_solve_multi(tsmpc_plan* const* plans, int32_t n, const double* p, int32_t iters,
                      double lam, const double* theta, const double* coef, int32_t flags,
                      tsmpc_result* outs);
/* Edges whose rows a plan computes (which = 0: all for a single-GPU plan, owned
 * chains + own and mixed trunk positions for a shard plan; which = 1: trunk
 * edges).  Writes up to cap
 * edge ids to out (may be NULL) and returns the count (or a negative status). */
int tsmpc_plan_edges(const tsmpc_plan* plan, int32_t which, int64_t* out, int64_t cap);

/* Per-forecast stage cache (elimination.py:114-158).
 * beta n_edges*n_v, uhat n_edges*n_u, evec n_edges*n_x, q n_u,
 * prices N*n_u (alpha1 + alpha2(k+j) per stage), jrhs n_edges*n_e (= -Ed d per
 * edge) and gdd n_edges*n_x (= Gd d per edge) are only read by the duality gap
 * (engine.py:347-480) and may be NULL when TSMPC_SKIP_GAP is always used. */
int tsmpc_set_cache(tsmpc_plan* plan, const double* beta, const double* uhat,
                    const double* evec, const double* q, const double* prices,
                    const double* jrhs, const double* gdd);

/* Device stage cache (elimination.py:114-158 build_stage_cache, tree.py:319-331
 * node_demands).  Once per plan: part_map n_u*n_d, Gd n_x*n_d, Ed n_e*n_d,
 * Rhat = Wu L n_u*n_v, eps_edge n_edges*n_d (eps of node e+1), pbar n_edges.
 * Per forecast: dhat N*n_d, q n_u, prices N*n_u (alpha1 + alpha2(k+j)) and
 * abar N*n_v (W_alpha L' price(k+j)); beta/uhat/evec and the gap inputs are then
 * built in HBM (replaces tsmpc_set_cache's E*(n_v+n_u+n_x) upload).
 * tsmpc_get_cache downloads beta/uhat/evec (any pointer may be NULL). */
int tsmpc_set_cache_operators(tsmpc_plan* plan, int32_t n_d, const double* part_map,
                              const double* Gd, const double* Ed, const double* Rhat,
                              const double* eps_edge, const double* pbar);
int tsmpc_set_forecast(tsmpc_plan* plan, const double* dhat, const double* q,
                       const double* prices, const double* abar);
int tsmpc_get_cache(tsmpc_plan* plan, double* beta, double* uhat, double* evec);

/* engine.solve: `iters` APG iterations at step size `lam` from y0 = y_-1 = warm
 * (three blocks, scaled coordinates) or zero when warm_sig == NULL.
 * theta / coef: optional momentum tables of length iters (NULL -> computed). */
int tsmpc_solve(tsmpc_plan* plan, const double* p, int32_t iters, double lam,
                const double* warm_sig, const double* warm_zeta, const double* warm_psi,
                const double* theta, const double* coef, int32_t flags,
                tsmpc_result* out);

/* Residual stopping test for later tsmpc_solve calls (extension; the reference
 * loop is fixed-iteration): every check_every iterations the residual_inf of
 * that iteration is reduced on the device and the solve stops as soon as it is
 * <= tol (tol <= 0 disables).  result.iterations reports the iterations run and
 * result.residual_inf the stopping residual.  Honoured by the structured-basis
 * kernel of single-GPU plans; other plans run max_iters. */
int tsmpc_set_stopping(tsmpc_plan* plan, double tol, int32_t check_every);
/* Timing trial (extension, no reference counterpart): `iters` iterations of the
 * plan's persistent kernel on whatever its buffers hold (zero right after
 * creation; the loop's cost does not depend on the data), CUDA-event time in *ms.
 * The Python layer uses it to pick the fastest of a few placements of a large
 * plan's buffers in device memory (plan.tuned_plan).  On a shard plan: this
 * rank's two launches per iteration without the cross-rank exchange, i.e. the
 * per-rank compute time of a multi-GPU solve (bench.py's sharded estimate). */
int tsmpc_plan_trial(tsmpc_plan* plan, int32_t iters, double* ms);

/* factor.solve_step: z = argmin <z, H'w> + f(z) for an unscaled dual w. */
int tsmpc_solve_step(tsmpc_plan* plan, const double* w_sig, const double* w_zeta,
                     const double* w_psi, const double* p, double* x_out, double* u_out);

/* engine.prox_g on n_rows rows with prox parameter `lam`; scaling rows per edge
 * are taken from the plan when use_scaling != 0 (rows must then equal n_edges). */
int tsmpc_prox(tsmpc_plan* plan, int32_t n_rows, const double* t_sig,
               const double* t_zeta, const double* t_psi, double lam, int32_t use_scaling,
               double* o_sig, double* o_zeta, double* o_psi);

/* Power-iteration support for compute_lambda: for the dual vector y resident on
 * the device (set by tsmpc_dual_operator_set), computes Dy = S H (z(0) - z(S y))
 * with a zero-demand cache built from beta0, stores Dy as the next y and returns
 * <y, Dy> and <Dy, Dy>.  Used by `compute_lambda` in engine.py of the package. */
int tsmpc_dual_operator_begin(tsmpc_plan* plan, const double* beta0);
int tsmpc_dual_operator_set_ones(tsmpc_plan* plan);
int tsmpc_dual_operator_step(tsmpc_plan* plan, double* y_dot_dy, double* dy_dot_dy,
                             double* y_dot_y);

/* Introspection (tests / bench): info = {levels, ctas, tiles, segments,
 * smem_bytes, diag_A, threads, tile_rows, sms, collapsed, trunk_edges, sparse,
 * resident_ctas, sharded, rank, world, owned_chain_edges, total_chains,
 * trunk_ctas, wide, exchange_doubles (shard plans: the doubles every rank sums
 * per iteration), fill_rows_hbm (wide plans with multi-tile or sharded CTAs: the
 * epilogue leaves the next backward's fill rows in HBM), peer_exchange (shard
 * plans: the cut exchange runs inside the kernel over peer memory)}. */
int tsmpc_plan_info(const tsmpc_plan* plan, int64_t* info, int32_t n_info);

/* Host-only planning (no device needed): the segment / level / tile / trunk
 * decomposition tsmpc_plan_create would build for this tree with `max_ctas` CTAs.
 * info = {levels, ctas, tiles, segments, rows, trunk_edges, max_rows_per_cta,
 *         max_tiles_per_cta, max_trunk_path}. */
int tsmpc_describe_tree(const tsmpc_problem* prob, int32_t max_ctas, int32_t collapse,
                        int64_t* info, int32_t n_info);
/* Host-only planning of the sparse kernel: info = {ctas, tiles, chains,
 * trunk_edges, resident_ctas, max_rows_per_cta, max_needs, smem_bytes,
 * trunk_ctas (split mode: spare CTAs running the trunk; 0 otherwise)}. */
int tsmpc_describe_sparse(const tsmpc_problem* prob, int32_t max_ctas, int64_t smem_limit,
                          int64_t* info, int32_t n_info);
/* Page-locked host memory for result buffers (cudaHostAlloc, portable across
 * devices): tsmpc_solve's device->host copies into such buffers run at DMA speed
 * (the Python layer returns SolveReport arrays from a pool of these). */
void* tsmpc_host_alloc(int64_t bytes);
void tsmpc_host_free(void* ptr);

/* Host-only planning of one shard: info = {ctas, owned_chains, owned_rows,
 * trunk_edges, total_chains, owned_trunk_nodes (chain-head groups), smem_bytes,
 * own_trunk_positions (only this rank's chains below), mixed_positions (several
 * ranks' chains below: replicated), cut_positions (single-rank subtrees hanging
 * from a mixed position), exchange_rows, exchange_doubles (per iteration, the
 * count every rank sums: SURVEY §8e's cut), result_rows}; the edges whose rows
 * the shard computes (tsmpc_plan_edges(plan, 0)) go to edges[0..cap) when
 * edges != NULL. */
int tsmpc_describe_shard(const tsmpc_problem* prob, int32_t max_ctas, int64_t smem_limit,
                         int32_t rank, int32_t world, int64_t* info, int32_t n_info,
                         int64_t* edges, int64_t cap);
const char* tsmpc_last_error(void);
/* Which persistent kernel tsmpc_solve runs: "sparse" (structured basis,
 * tsmpc_sparse.cu) or "dense: <reason>" (fused-operator DMMA kernel). */
const char* tsmpc_plan_path(const tsmpc_plan* plan);
/* Phase cycle counters of CTA 0 (non-zero only in -DTSMPC_TIMERS builds); reset on read. */
int tsmpc_debug_timers(tsmpc_plan* plan, uint64_t* out, int32_t n);
int tsmpc_device_count(void);

#ifdef __cplusplus
}
#endif
#endif /* TSMPC_H */
