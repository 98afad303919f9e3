// tsmpc_kernels.cuh — device side of the B200 scenario-tree APG solver.
//
// One persistent cooperative kernel runs every APG iteration of a solve
// (reference loop: pkg/src/treesmpc/engine.py:537-585).  The tree is cut into
// *segments* — maximal only-child chains, <= kMaxSeg edges — grouped by segment
// depth ("level").  Each CTA owns a fixed set of segments per level, packed into
// tiles of <= kTileM edge rows.  A tile is processed entirely in shared memory:
//
//   backward (bwd_tile, levels D-1 .. 0)       reference factor.py:142-156
//     s = D_sig w_sig + D_zeta w_zeta, psi^ = D_psi w_psi, w = y + c (y - y_prev)
//     xiq scan   xiq_e = s_e + A' sum_children xiq_c              (elementwise if A diagonal)
//     GEMM 1     h_e = [xiq_e | psi^_e] [Bbar ; L]                 (DMMA m8n8k4, fp64)
//     g scan     g_e = beta_e + h_e + sum_children g_c ;  t_e = g_e / (2 p_e)
//   forward (fwd_tile, levels 0 .. D-1)        reference factor.py:158-170
//     S scan     S_e = t_e + S_parent                   (v = -Rbar^{-1} S, never formed)
//     GEMM 2     [du_e | bv_e] = S_e [Psi | Phi]                   (DMMA m8n8k4, fp64)
//     x scan     x_e = A x_anc + bv_e + e_e ;  u_e = uhat_e + du_e
//     epilogue   prox_g, dual update, ergodic averages, residual  engine.py:546-575
//
// Grid barriers are needed only between levels (2(D-1) per iteration); for the
// paper-shaped trees D = 4.  See DESIGN.md for the derivation (the backward
// sweep's Rbar^{-1} is folded into the forward operator, which removes one of the
// three per-edge contractions of the reference).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>

namespace tsmpc {

constexpr int kThreads = 416;      // 13 warps (128 registers each); GEMM items = (n-tile, m-part)
constexpr int kWarps = kThreads / 32;
constexpr int kTileM = 96;         // edge rows per shared-memory tile (<= 12 m-tiles)
constexpr int kMaxSeg = 32;        // longest segment (longer chains are split into levels)

enum Mode : int { kModeApg = 0, kModeStep = 1 };

struct Params {
  // dimensions
  int nx, nu, nv, N, n_nodes, n_edges;
  int NXP, NUP, NVP;            // global row pitches (multiples of 4 doubles)
  int KS1, NT1;                 // GEMM 1: k-steps (K1 = NXP+NUP), n-tiles (ceil(nv/8))
  int KS2, NT2, NU8;            // GEMM 2: k-steps (ceil(nv/4)), n-tiles, du columns
  int LDA1, LDB1;               // shared-memory leading dims, backward sweep (A | C)
  int LDA2, LDB2;               // shared-memory leading dims, forward sweep (A | C)
  int META_OFF;                 // offset (doubles) of the tile metadata ints
  int diagA;
  double Wx, gamma_d;
  // model
  const double* a_diag;         // NXP (diag A)
  const double* A;              // nx*nx (dense A)
  const double* W1f;            // fragment-ordered [NT1][KS1][32]
  const double* W2f;            // fragment-ordered [NT2][KS2][32]
  const double *x_s, *x_min, *x_max, *u_min, *u_max;
  const double *sig_stage, *zeta_stage, *psi_stage;  // N, N, N*NUP
  const double *sig_rcp, *zeta_rcp, *psi_rcp;        // reciprocals of the above
  double inv_lam;                                    // 1 / lam
  // tree
  const int *anc, *child_start, *child_stop, *edge_stage;
  const double* inv2p;
  // plan
  int n_levels, n_ctas;
  const int* lvl_tiles;         // n_levels*n_ctas + 1
  const int* tile_seg;          // n_tiles + 1
  const int* seg_row;           // n_segs + 1
  const int* row_edge;          // n_rows
  // collapsed trunk (diagonal A): every non-leaf segment edge is a "trunk" edge,
  // handled by one component-sliced sweep + one distributed GEMM per iteration
  int collapsed;                // 1: leaf segments are level 0 tiles, trunk collapsed
  int n_trunk;                  // trunk edges T
  const int* trunk_edge;        // T, ascending edge id (stage-major)
  const int* trunk_stage_ptr;   // N+1 offsets into trunk_edge per edge stage
  const int* trunk_pos;         // E, position in trunk_edge or -1
  const int* trunk_parent;      // T: trunk position of the parent edge, -1 below the root
  int trunk_smem;               // 1: the component sweep fits its slice in shared memory
  const int* trunk_child0;      // T: trunk pos of the first child if all children are trunk,
                                //    -1 if none is (chain heads only), -2 if mixed
  const int* path_ptr;          // T+1 offsets into path_list
  const int* path_list;         // trunk positions root .. t for every trunk edge t
  int KY_LD, KSK, NTT;          // KY pitch (NVP + NXP + NUP), GEMM k-steps, n-tiles
  int OUT_LD, U_OFF, X_OFF;     // OUT pitch and column offsets of u and bv + e
  double* KY;                   // T x KY_LD  [K | Yx | Ypsi]
  double* OUT;                  // T x OUT_LD [S | u | bv + e]
  const double* MTf;            // fragment-ordered [NTT][KSK][32] trunk operator
  // state
  double* ybuf[2];              // slot -> [sig | zeta | psi] blocks
  double *xavg, *uavg, *X, *U, *T, *XIQG, *GG;
  const double *beta, *uhat, *evec;  // uhat/evec may be null (zero)
  const double* p;              // NXP root state (device)
  // loop control
  int mode, iters, scaled, record_all, slot0;
  double lam;
  const double *theta, *coef;
  unsigned long long* resid;    // iters (record_all) or 1 slot, bit pattern of a double >= 0
  // optional residual stopping test (sparse kernel): every check_every iterations
  // the residual is reduced into resid_chk[k] and the solve stops as soon as it is
  // <= tol; iters_done receives the number of iterations run
  double tol;
  int check_every;
  unsigned long long* resid_chk;
  int* iters_done;
  unsigned long long* timers;   // phase cycle counters of CTA timer_cta (TSMPC_TIMERS builds only)
  int timer_cta;
};

// ---------------------------------------------------------------------------
// Structured-basis ("sparse") persistent kernel, tsmpc_sparse.cu.  Used by
// tsmpc_solve when A is diagonal, the plan carries the block-structured kernel
// basis Ls (precompute.structured_basis: Ls' Wu Ls = diag) and every leaf chain
// fits a tile of kTileS rows.  The factor step then needs no dense contraction:
//   h  = Ls' (B' xiq + psi^)          (two sparse products)
//   du = -Ls diag(lam)^-1 S           (one sparse product), bv = B du
// so the loop is bound by memory latency/bandwidth, and each CTA keeps the dual,
// ergodic and t rows of its chains resident in shared memory across iterations
// when they fit (otherwise one tile slot is streamed with cp.async).
// ---------------------------------------------------------------------------
constexpr int kThreadsS = 512;
constexpr int kWarpsS = kThreadsS / 32;
constexpr int kTileS = 24;         // rows per chain tile (a leaf chain never spans tiles)
constexpr int kMinTrunkCtas = 8;   // split mode needs at least this many spare CTAs for the trunk
constexpr int kTileW = 96;         // rows per wide tile (a leaf chain never spans tiles)
// shard plans: role of a trunk position on this rank (trunk schedule pos[8 tp + 7] & 7;
// (pos[8 tp + 7] >> 3) - 1 is its row in the cut exchange buffer XCH, -1 if none).
// Own / foreign: every chain below it belongs to this / another rank; mixed: chains
// of several ranks (replicated: every rank computes it); cut: a single-rank position
// whose parent is mixed (its bottom-up sums cross the cut).
constexpr int kRoleOwn = 0, kRoleForeign = 1, kRoleMixed = 2, kRoleCutOwn = 3, kRoleCutForeign = 4;

struct SParams {
  Params P;                     // dims, model vectors, scaling, tree, state, loop control, KY
  // sparse operators (int pool + double pool, staged in shared memory)
  const int* spi;
  const double* spv;
  int n_spi, n_spv;
  int Bc_ptr, Bc_idx, Br_ptr, Br_idx, Lc_ptr, Lc_idx, Lr_ptr, Lr_idx;  // int-pool offsets
  int Bc_val, Br_val, Lc_val, Lr_val;                                  // double-pool offsets
  // per-CTA plan (ints): see tsmpc_sparse.cu "meta layout"
  const int* meta;
  const int* meta_ptr;          // n_ctas + 1
  int meta_max;
  // trunk schedule (ints, shared by all CTAs): see "trunk schedule layout"
  const int* tsched;
  int n_tsched;
  // shared-memory layout, offsets in doubles from the dynamic base
  int O_BND, O_SCL, O_RED, O_PSI, O_SPV, O_NEED, O_WORK, O_SLOT, O_INT;
  int LA;                       // pitch of work region A: max(NXP, NVP)
  int sweep_in_a;               // trunk sweep buffers start in region A (no CTA keeps t there)
  int sched_smem;               // trunk schedule staged in shared memory during the sweep
  int psi_smem;                 // psi_stage table staged in shared memory (else read via L1)
  int sched_resident, O_SCHED;  // trunk schedule resident in shared memory for the launch
  int n_work;                   // doubles in the work region
  int need_ld;                  // NVP + NXP + NUP  ([S | x | u] of one needed trunk edge)
  int need_max;
  int YW;                       // 2 NXP + NUP      ([sig | zeta | psi] of one dual row)
  int slot_ld;                  // 2 YW + NXP + NUP (+ NVP when some CTA keeps t in its slot rows)
  int slot_rows;                // resident capacity of the slot region (rows)
  const double* beta_s;         // E x NVP  beta in the structured basis (beta M)
  double* TG;                   // E x NVP  t rows of streamed CTAs
  // (the launch window -- iterations and phases -- is a kernel argument, LaunchWin,
  // so that consecutive launches of one plan reuse the uploaded parameters)
  // subtree sharding across GPUs (one process per GPU): the trunk is replicated, the
  // leaf chains are split by the trunk node they hang from; HS holds, per trunk
  // position, [sum of the chain-head g | sum of the chain-head xiq] of the heads
  // hanging from its node (non-zero on the owning rank only) and is summed across
  // ranks between the two phases (ncclAllReduce; exact: one contributor per entry).
  int sharded;
  double* HS;                   // T x HS_LD
  int HS_LD;                    // NVP + NXP
  const unsigned char* towned;  // T: this rank owns the heads of the node below
  // cut exchange (world > 1): instead of HS for every trunk position, the ranks sum
  // only XCH (n_xch x XCH_LD): the head sums of the mixed positions and the bottom-up
  // sums [Z in KY columns | X] of the cut positions, written by their owning rank at
  // the end of phase 1 (zero on the others; exact).  Positions foreign to this rank
  // are skipped by the sweep, the trunk forward and the epilogues.
  // cut == 0 (small trunks): every position is mixed, XCH is HS itself (HS_LD wide)
  // and holds every position's head sums.
  double* XCH;
  int n_xch, XCH_LD;            // XCH_LD = KY_LD + NXP (cut) or HS_LD
  int cut;
  // split mode (single GPU, one tile per chain CTA, spare CTAs): CTAs >= split_c0
  // ("trunk CTAs") run the trunk sweep, then -- after a barrier among themselves --
  // the trunk forward of their trunk rows, exporting per trunk position
  // [du | B du | x] to TR; meanwhile the chain CTAs run their chains' forward with
  // zero trunk input, then add the affine trunk terms from TR after the grid barrier.
  int split, split_c0, split_n;
  int split_local;              // trunk CTAs sweep their own trunk subtrees in shared memory
                                // (all components; no trunk-CTA barrier, KY stays on chip)
  double* TR;                   // T x TR_LD
  int TR_LD;                    // NUP + 2 NXP
  unsigned int* sub_ctr;        // [trunk-CTA barrier, heads published, TR published] (zeroed per launch)
  int split_flags;              // directed signals between chain and trunk CTAs instead of grid barriers
  int a_unit;                   // A = I (a = 1 in every state component): chain recursions are plain sums
  const int* tpi;               // split mode: combined trunk-forward operators (SparseHostPlan::tpi/tpv)
  const double* tpv;
  int M1_ptr, M1_col, M2_ptr, M2_col, M1_val, M2_val;
  int n_tpi, n_tpv;
  int tops;                     // 1: trunk CTAs stage tpv | tpi in their slot region at O_SLOT + O_TOPS
  int O_TOPS;
  int split_heads, O_HSUM;      // chain CTAs publish their head values right after the fill, by
                                // reductions ([sum beta_s | sum psi^ | sum G_d s | sum z] at O_HSUM)
  unsigned int* abort_flag;     // raised by a spin-wait that timed out (plan-owned, zeroed per solve)
  int tile_cap;                 // rows of the work regions A / B (kTileS, or the widest wide tile)
  // wide mode (apg_wide_kernel): a CTA's chains are packed into tiles of up to
  // kTileW rows that are processed as one (the chain scans of all its chains run
  // together), and the dual / ergodic rows stay in HBM (L2-resident), read into
  // registers by the fill and the epilogue -- no shared-memory slot rows.  t rows
  // stay in region A when a CTA has one tile (tmode 0), else they go through TG.
  int wide;
  int wide_prefill;             // the epilogue of the CTA's last tile leaves the next fill
  // fill rows through HBM (multi-tile or sharded wide CTAs): the epilogue of every tile
  // that cannot leave its next fill in shared memory writes it to FG (E x FL,
  // [s (NXP) | psi^ (NUP)]), and the next backward copies it in (cp.async) instead of
  // reading both dual rows and extrapolating
  double* FG;
  int FL;                       // NXP + NUP
  // per-row / per-chain meta windows (CTAs with many tiles whose full meta does not fit
  // in shared memory, e.g. W16k): only the header, tiles, needs, levels and own rows
  // are staged at launch; the rows {edge, stage, inv2p} and chain segments of the
  // tile being processed are copied into a window (O_WIN ints after the staged ints:
  // rows then, 4 tile_cap ints further, segments) before each tile
  int rows_window, O_WIN;
  // cut exchange over peer memory inside the persistent kernel (shard plans whose
  // ranks mapped each other's receive buffers: LaunchWin.phase & 4).  Per iteration
  // every CTA stores its slice of XCH into slot (generation & 1), sender row `rank`,
  // of every rank's RX, fences (system scope) and bumps every rank's arrival counter
  // once; a rank waits until its counter reaches (generation + 1) x xch_expect, then
  // sums the world sender rows of its slice in rank order back into XCH.
  double* const* peer_rx;               // world pointers (this device's view of rank p's RX)
  unsigned long long* const* peer_cnt;  // world pointers (rank p's arrival counter)
  double* RX;                           // 2 x world x n_xch x XCH_LD
  unsigned long long* RXCNT;            // this rank's arrival counter (monotone across solves)
  int rank, world;
  unsigned long long xch_expect;        // arrivals per iteration: world x CTAs per rank
  int hsum_nseg;                // wide split mode: chains per chain CTA the head-sum scratch holds
};

// Launch window of the structured-basis kernels (a kernel argument): iterations
// [nu0, nu1) and phases (1: backward (+ head pre-reduction when sharded), 2: trunk
// sweep, needs, forward + epilogue; 4: shard plans with peer-mapped receive buffers
// run both phases and the cut exchange in one launch).  Single-GPU plans run every
// iteration with both phases in one launch.  wb_end: the window ends with a full write-back (the
// state of iteration nu1 - 1 is left in HBM: per-iteration duality gap).
struct LaunchWin {
  int nu0, nu1, phase, wb_end;
  unsigned long long xgen;  // peer exchange (phase & 4): generation of iteration nu0
};

// Phase timers (profiling builds: -DTSMPC_TIMERS).  Slot k accumulates the cycles
// CTA 0 spends between consecutive marks.
#ifdef TSMPC_TIMERS
#define TSMPC_MARK(P, k, t)                                                   \
  do {                                                                        \
    __syncthreads();                                                          \
    if (blockIdx.x == (P).timer_cta && threadIdx.x == 0 && (P).timers) {      \
      const long long now_ = clock64();                                       \
      atomicAdd((P).timers + (k), (unsigned long long)(now_ - (t)));          \
      (t) = now_;                                                             \
    }                                                                         \
  } while (0)
// Timeline stamps (profiling builds): %globaltimer of point k of every CTA, for the
// iteration the kernel marks traced (slots 16 + 8 CTA + k of the timer buffer;
// tools/trace_probe.py).
#define TSMPC_STAMP(P, k, on)                                                 \
  do {                                                                        \
    if ((on) && threadIdx.x == 0 && (P).timers) {                             \
      unsigned long long g_;                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_));                 \
      (P).timers[16 + 8 * blockIdx.x + (k)] = g_;                             \
    }                                                                         \
  } while (0)
#else
#define TSMPC_MARK(P, k, t) do { } while (0)
#define TSMPC_STAMP(P, k, on) do { } while (0)
#endif

}  // namespace tsmpc
