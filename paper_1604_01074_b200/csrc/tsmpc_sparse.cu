// tsmpc_sparse.cu — structured-basis persistent APG kernel for sm_100a.
//
// One cooperative launch runs every APG iteration of engine.solve
// (reference pkg/src/treesmpc/engine.py:537-585).  The solve step
// (factor.py:142-170) is evaluated in the block-structured kernel basis Ls of
// precompute.structured_basis, where Rbar_s = Ls' Wu Ls is diagonal.  Per edge e
// with t_e = g_e / (2 p_e) and S_e = sum_{a on root..e} t_a:
//
//   backward  xiq_e = s_e + a .* sum_children xiq_c        s = D_sig w_sig + D_zeta w_zeta
//             g_e   = beta_s,e + Ls' (B' xiq_e + psi^_e) + sum_children g_c
//   forward   du_e  = Lt S_e   (Lt = -Ls diag(lam)^-1)      u_e = uhat_e + du_e
//             x_e   = a .* x_anc + (B du_e + e_e)
//
// so every contraction of the reference is a sparse product with a handful of
// non-zeros per row (Barcelona-size network: 165 in Ls, ~150 in B) and the
// iteration is bound by memory traffic and latency, not FP64 throughput.
//
// Work split (host plan, tsmpc_capi.cu:plan_sparse): leaf chains (maximal
// only-child paths ending at a leaf, <= kTileS edges) are packed into tiles; a
// CTA owns a fixed list of tiles for the whole launch.  Every other edge is a
// trunk edge.  Per iteration:
//
//   A  backward over the CTA's tiles -> chain-head sums GG (g), XIQG (xiq)
//      grid barrier
//   B  trunk sweep, component-sliced over all CTAs -> KY = [K | Yx | Ypsi]
//      (the collapsed trunk of DESIGN.md §2, linear in the chain-head sums)
//      grid barrier
//   D  each CTA evaluates S, x, u of the trunk edges on its heads' root paths
//      ("needs") from KY, runs the epilogue of its own trunk rows, then the
//      forward sweep + prox / dual-update epilogue of its tiles.
//
// Residency: if all rows of a CTA fit the slot region, their dual rows (y and
// y_prev), ergodic rows and t rows stay in shared memory for the whole launch
// and HBM is touched only for the static per-edge vectors (beta_s, uhat, e)
// and, on the last iteration, the outputs.  Otherwise one tile slot is streamed
// with cp.async, prefetched one step ahead (see bwd/fwd below).
#include "tsmpc_kernels.cuh"
#include <cstring>
#include <mutex>

namespace cg = cooperative_groups;

namespace tsmpc {

extern __shared__ __align__(16) double s_dyn[];

// The launch parameters live in constant memory (set by sparse_launch on the
// launching stream): every field access is a uniform constant-bank load that
// the compiler may hoist freely, also inside the __noinline__ phase functions.
__constant__ SParams g_sp;
// the launch window of the running kernel (set from the kernel argument at entry)
__shared__ LaunchWin s_win;
__shared__ int s_trace_on;  // timer builds: this iteration is the traced one
// meta windows (SParams::rows_window): first row / segment of the staged tile
__shared__ int s_row_off, s_seg_off;

namespace {

// ---- meta layout (ints, per CTA) -------------------------------------------
//   [0] ntiles [1] nrows [2] nsegs [3] nneed [4] nlev [5] nown [6] resident
//   [7] tmode (where t rows live: 0 region A, 1 slot rows, 2 HBM)
//   tiles : ntiles x {row0, nrows, seg0, nsegs}
//   rows  : nrows  x {edge, stage, inv2p lo, inv2p hi}
//   segs  : nsegs  x {lo, hi, pneed, 0}         (lo/hi relative to the tile)
//   needs : nneed  x {trunk pos, pneed, edge, stage}   (sorted by depth)
//   lev   : nlev + 1 need offsets per depth
//   own   : nown need indices (trunk rows whose epilogue this CTA runs)
struct Meta {
  const int* m;
  int ntiles, nrows, nsegs, nneed, nlev, nown, resident, tmode;
  const int *tiles, *rows, *segs, *needs, *lev, *own;
  // rows_w / segs_w: the meta windows of the current tile (SParams::rows_window), else null
  __device__ void bind(const int* base, const int* rows_w = nullptr, const int* segs_w = nullptr) {
    m = base;
    ntiles = m[0]; nrows = m[1]; nsegs = m[2]; nneed = m[3]; nlev = m[4]; nown = m[5]; resident = m[6];
    tmode = m[7];
    tiles = m + 8;
    rows = rows_w ? rows_w : tiles + 4 * ntiles;
    segs = rows_w ? segs_w : rows + 4 * nrows;
    needs = rows_w ? tiles + 4 * ntiles : segs + 4 * nsegs;
    lev = needs + 4 * nneed;
    own = lev + nlev + 1;
  }
  __device__ int edge(int row) const { return rows[4 * row]; }
  __device__ int stage(int row) const { return rows[4 * row + 1]; }
  __device__ double inv2p(int row) const {
    return __hiloint2double(rows[4 * row + 3], rows[4 * row + 2]);
  }
};

// ---- trunk schedule layout (ints, identical for all CTAs) ------------------
//   [0] T [1] nlev [2] n_tch [3] n_hch
//   lev : nlev + 1 trunk-position offsets per edge stage (ascending)
//   pos : T x {edge, stage, parent pos, tch0, ntch, hch0, nhch, 0}
//   tch : trunk children (positions);  hch : chain-head children (edge ids)

// max / min of the prox projections: a compare and a select (fmax / fmin add NaN
// handling the iterates never need; TSMPC_FMAX=1 restores them)
#ifndef TSMPC_FMAX
#define TSMPC_FMAX 0
#endif
__device__ __forceinline__ double dmax(double a, double b) { return TSMPC_FMAX ? fmax(a, b) : (a > b ? a : b); }
__device__ __forceinline__ double dmin(double a, double b) { return TSMPC_FMAX ? fmin(a, b) : (a < b ? a : b); }
__device__ __forceinline__ double extrap(double y, double yp, double c) {
  return __dadd_rn(y, __dmul_rn(c, __dsub_rn(y, yp)));
}
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ void stcg(double* p, double v) { __stcg(p, v); }

__device__ __forceinline__ void cp16(double* sdst, const double* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
// bulk (TMA engine) row copies global -> shared completing on an mbarrier (wide
// kernel's FG fill rows and TG t rows): 16-byte aligned addresses, sizes multiple of 16
#ifndef TSMPC_BULK
#define TSMPC_BULK 1
#endif
#ifndef TSMPC_UNR
#define TSMPC_UNR 2
#endif
constexpr int kUnr = TSMPC_UNR;  // rows in flight per thread in the wide kernel's sparse row phases
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::
          "r"(smem_u32(bar)), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_row(void* sdst, const void* gsrc, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(sdst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// generic-proxy accesses of this thread ordered before later async-proxy (bulk copy) ones
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__shared__ unsigned long long s_bulk_bar;  // bulk row copies of the wide kernel (FGK)
__shared__ unsigned s_bulk_phase;
// all threads: arm the bulk barrier for `total` bytes and issue copies 0..n-1
// (issue(i) calls bulk_row).  The destination's last readers are behind the block
// barrier that ended the previous phase; the barrier's tx-count may dip below zero
// while copies complete before thread 0's expect_tx, and its phase cannot complete
// before that arrival.
template <class ISSUE>
__device__ __forceinline__ void bulk_issue(int n, unsigned total, ISSUE issue) {
  if (TSMPC_BULK & 2) {  // experiment: proxy fence and barriers before the copies
    fence_proxy_async();
    __syncthreads();
  }
  if (threadIdx.x == 0) mbar_expect_tx(&s_bulk_bar, total);
  if (TSMPC_BULK & 2) __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) issue(i);
}
// all threads: wait for the bytes of the last bulk_issue
__device__ __forceinline__ void bulk_wait() {
  mbar_wait(&s_bulk_bar, s_bulk_phase);
  __syncthreads();
  if (threadIdx.x == 0) s_bulk_phase ^= 1u;
}
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// directed signals of split mode (counters zeroed per launch): a CTA publishes
// its writes (arrive) / waits until `target` arrivals (wait)
__device__ __forceinline__ void signal_arrive(unsigned int* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
  }
}
// Spin-waits give up after ~2 s of clock64 time: the waiting CTA raises the
// plan's abort flag and returns, every other wait returns as soon as it sees the
// flag, so all CTAs run to the end of the launch (no CTA exits early: the grid
// barriers stay consistent) and the host reports TSMPC_ERR_CUDA with a message
// instead of a hung GPU or a sticky trap that would poison the CUDA context.
// A timeout means a plan inconsistency (or a debugger stopping the kernel); the
// results of that launch are discarded.
constexpr long long kSpinLimit = 4000000000LL;

__device__ __forceinline__ void spin_until(const unsigned int* ctr, unsigned int target) {
  const long long t0 = clock64();
  volatile const unsigned int* abort_flag = g_sp.abort_flag;
  while (*((volatile const unsigned int*)ctr) < target) {
    if (*abort_flag) return;
    if (clock64() - t0 > kSpinLimit) {
      atomicExch(const_cast<unsigned int*>(abort_flag), 1u);
      return;
    }
  }
}

__device__ __forceinline__ void spin_until64(const unsigned long long* ctr, unsigned long long target) {
  const long long t0 = clock64();
  volatile const unsigned int* abort_flag = g_sp.abort_flag;
  while (*((volatile const unsigned long long*)ctr) < target) {
    if (*abort_flag) return;
    if (clock64() - t0 > kSpinLimit) {
      atomicExch(const_cast<unsigned int*>(abort_flag), 1u);
      return;
    }
  }
}

__device__ __forceinline__ void signal_wait(unsigned int* ctr, unsigned int target) {
  if (threadIdx.x == 0) {
    spin_until(ctr, target);
    __threadfence();
  }
  __syncthreads();
}

// Element phases map threads component-major: thread = (row group g, component
// k), g = tid / kKW, rows r = g, g + kGroups, ...  The per-component sparse
// column range is read once per phase; no integer divisions.  Phase functions
// are __noinline__ and rebuild their context from the __grid_constant__
// parameters (the whole loop body stays within the instruction cache).
constexpr int kKW = 128;                    // component lanes per row group (n_x, n_u <= 128)
constexpr int kGroups = kThreadsS / kKW;    // 4 row groups
constexpr int kRowsPT = kTileS / kGroups;   // rows per thread in a full tile
constexpr int kCh = 8;                      // rows per register chunk of the chain scans

// ---- tensor memory (TMEM) holding static per-row vectors (see kTmB, kTmRB) ----
// Every thread of a CTA that uses it owns a private 128-column block of one TMEM
// lane: lane = tid mod 128, columns 128 (tid / 128) .. + 127.  The accesses are
// warp-collective (.sync.aligned): every lane of a warp takes part.
__shared__ uint32_t s_tmem;  // TMEM base of this CTA (0 is a valid address)
__shared__ int s_tm_on;      // the static vectors are in TMEM (else read from HBM)
__device__ __forceinline__ uint32_t tm_addr(int col) {
  return s_tmem + ((uint32_t)(((threadIdx.x >> 5) & 3) * 32) << 16) + (uint32_t)((threadIdx.x >> 7) * 128 + col);
}
__device__ __forceinline__ void tm_st1(uint32_t a, double v) {  // warp-collective
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n" ::"r"(a), "r"(__double2loint(v)),
               "r"(__double2hiint(v))
               : "memory");
}
// 8 doubles (16 columns) from a, warp-collective; the caller waits (tm_wait_ld)
__device__ __forceinline__ void tm_ld8(uint32_t a, double* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(a));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __hiloint2double((int)r[2 * i + 1], (int)r[2 * i]);
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
// all 512 columns (one CTA per SM), allocated by warp 0; s_tmem after the barrier
__device__ __forceinline__ void tm_alloc_all() {
  if ((threadIdx.x >> 5) == 0) {
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&s_tmem);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(dst) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
// after this thread's stores: mark the CTA's vectors resident (s_tm_on)
__device__ __forceinline__ void tm_fill_done() {
  tm_wait_st();
  if (threadIdx.x == 0) s_tm_on = 1;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tm_release() {
  if (!s_tm_on) return;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if ((threadIdx.x >> 5) == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(s_tmem) : "memory");
}
// resident one-tile CTAs (apg_sparse_kernel): beta_s, uhat, e of the thread's
// kRowsPT rows (group mapping) in columns 0.., 16.., 32..
constexpr int kTmRB = 0, kTmRU = 16, kTmRE = 32;
static_assert(kRowsPT <= 8, "resident TMEM slots hold 8 rows per thread");

struct Ctx {
  const SParams* S;
  const Params* P;
  Meta mt;
  double* bnd;     // x_s, x_min, x_max (NXP), u_min, u_max (NUP), a_diag (NXP), p (NXP)
  double* scl;     // sig, zeta, 1/sig, 1/zeta per stage (N each)
  double* psi;     // psi_stage (N x NUP) or null (unscaled)
  double* red;     // epilogue row descriptors (5 ints per row)
  const int* spi;  // sparse index pool (shared)
  const double* spv;
  double* need;    // need rows [S | x | u]
  double* work;    // region A (tcap x LA) | region B (tcap x NUP)
  double* slot;
  int NXP, NUP, NVP, YW, SL, N, LA;
  int nx, nu, nv, E;
  int tcap;        // rows of the work regions (kTileS; the largest wide tile in wide mode)
  // region A: xiq -> h -> t (backward), S -> bv + e -> x (forward); region B: z / du -> u
  __device__ double* A() const { return work; }
  __device__ double* B() const { return work + tcap * LA; }
  __device__ const double* adiag() const { return bnd + 3 * NXP + 2 * NUP; }
  __device__ const double* proot() const { return bnd + 4 * NXP + 2 * NUP; }
  __device__ int* rdesc() const { return reinterpret_cast<int*>(red); }
  const double* psi_g;  // psi_stage in HBM when the table does not fit shared memory
  int psi_o;            // offset of the psi_stage table in shared memory, -1 if not there
  // (indexing s_dyn directly keeps the access an LDS; a possibly-null pointer
  // would compile to a generic load)
  __device__ double dpsi(int st, int k) const {
    return psi_o >= 0 ? s_dyn[psi_o + st * NUP + k] : (psi_g ? __ldg(psi_g + (size_t)st * NUP + k) : 1.0);
  }
  __device__ bool scaled() const { return psi_o >= 0 || psi_g; }
};

__device__ __forceinline__ Ctx ctx_of() {
  const SParams& S = g_sp;
  const Params& P = S.P;
  Ctx c;
  c.S = &S;
  c.P = &P;
  c.NXP = P.NXP; c.NUP = P.NUP; c.NVP = P.NVP;
  c.YW = S.YW; c.SL = S.slot_ld; c.N = P.N;
  c.nx = P.nx; c.nu = P.nu; c.nv = P.nv; c.E = P.n_edges;
  c.bnd = s_dyn + S.O_BND;
  c.scl = s_dyn + S.O_SCL;
  c.red = s_dyn + S.O_RED;
  c.psi = P.scaled && S.psi_smem ? s_dyn + S.O_PSI : nullptr;
  c.psi_o = P.scaled && S.psi_smem ? S.O_PSI : -1;
  c.psi_g = P.scaled && !S.psi_smem ? P.psi_stage : nullptr;
  c.LA = S.LA;
  c.tcap = S.tile_cap;
  c.need = s_dyn + S.O_NEED;
  c.work = s_dyn + S.O_WORK;
  c.slot = s_dyn + S.O_SLOT;
  const int* ints = reinterpret_cast<const int*>(s_dyn + S.O_INT);
  if (S.rows_window)
    c.mt.bind(ints, ints + S.O_WIN - 4 * s_row_off, ints + S.O_WIN + 4 * S.tile_cap - 4 * s_seg_off);
  else
    c.mt.bind(ints);
  c.spi = ints + S.meta_max;
  c.spv = s_dyn + S.O_SPV;
  return c;
}

// One compressed column (or row) of an operator; its first kNZ entries are
// row-invariant and held in registers for the whole phase.
constexpr int kNZ = 4;
struct SpCol {
  int q0, q1;
  int idx[kNZ];
  double val[kNZ];
};
__device__ __forceinline__ SpCol sp_col(const Ctx& c, int ptr_off, int idx_off, int val_off, int k) {
  SpCol s;
  s.q0 = c.spi[ptr_off + k];
  s.q1 = c.spi[ptr_off + k + 1];
#pragma unroll
  for (int m = 0; m < kNZ; ++m) {
    const bool v = s.q0 + m < s.q1;
    s.idx[m] = v ? c.spi[idx_off + s.q0 + m] : 0;
    s.val[m] = v ? c.spv[val_off + s.q0 + m] : 0.0;
  }
  return s;
}
// acc + sum_q val_q * row[idx_q], q ascending (fixed order)
__device__ __forceinline__ double sp_dot(const Ctx& c, const SpCol& s, int idx_off, int val_off,
                                         const double* row, double acc) {
#pragma unroll
  for (int m = 0; m < kNZ; ++m)
    if (s.q0 + m < s.q1) acc = fma(s.val[m], row[s.idx[m]], acc);
#pragma unroll 1
  for (int q = s.q0 + kNZ; q < s.q1; ++q) acc = fma(c.spv[val_off + q], row[c.spi[idx_off + q]], acc);
  return acc;
}

// slot row pointers: Y0 | Y1 | XA | UA | T
__device__ __forceinline__ double* slot_row(const Ctx& c, int srow) { return c.slot + (size_t)srow * c.SL; }

// Issue cp.async copies of rows into slot-format smem rows.  Row r of the batch
// is edge edge_of(r) -> smem row dst + r * SL.  parts: 1 = both dual rows,
// 2 = ergodic rows.  ysm = smem dual index that receives HBM slot `cur`.
__device__ __noinline__ void load_rows(const int* edges, int estride, int nrows, double* dst,
                                       int parts, int cur, int ysm) {
  // one (row, contiguous part) pair per warp pass; lanes stream 16-byte chunks
  const SParams& S = g_sp;
  const Params& P = S.P;
  const int NXP = P.NXP, NUP = P.NUP, YW = S.YW, SL = S.slot_ld;
  const size_t E = (size_t)P.n_edges;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int p0 = (parts & 1) ? 0 : 6, p1 = (parts & 2) ? 8 : 6;
  const int np = p1 - p0;
#pragma unroll 1
  for (int w = warp; w < nrows * np; w += kWarpsS) {
    const int r = w / np, part = p0 + (w - r * np);
    const int e = edges[r * estride];
    double* srow = dst + (size_t)r * SL;
    const double* src;
    double* d;
    int len;
    if (part < 6) {  // dual rows: parts 0-2 from HBM slot cur, 3-5 from cur ^ 1
      const int which = part / 3, blk = part - 3 * which;
      const double* Y = P.ybuf[cur ^ which];
      d = srow + (size_t)(ysm ^ which) * YW + blk * NXP;
      src = blk < 2 ? Y + (size_t)blk * E * NXP + (size_t)e * NXP : Y + 2 * E * NXP + (size_t)e * NUP;
      len = blk < 2 ? NXP : NUP;
    } else if (part == 6) {
      d = srow + 2 * YW;
      src = P.xavg + (size_t)(e + 1) * NXP;
      len = NXP;
    } else {
      d = srow + 2 * YW + NXP;
      src = P.uavg + (size_t)e * NUP;
      len = NUP;
    }
    for (int q = lane; q < len / 2; q += 32) cp16(d + 2 * q, src + 2 * q);
  }
}

// ----------------------------------------------------------------------------
// epilogue: prox_g (engine.py:146-183), dual update, ergodic averages, residual
// (engine.py:546-575) for rows described by c.rdesc(): {edge, stage, x offset,
// u offset, slot-row offset} (offsets in doubles from the dynamic shared-memory
// base).  Dual rows: y at index ysm, y_prev at ysm ^ 1; y+ replaces y_prev in
// place.  wt: also write y+ and the ergodic rows to HBM (slot `ncur` gets y+).
//
// psi block (box projection, elementwise): thread (g, k) for its rows, given u.
// state blocks (two weighted-distance proxes): one warp per row — the row norm
// is a warp reduction and the prox factor a warp-uniform scalar, so the block
// needs no shared-memory exchange and no barrier.
// ----------------------------------------------------------------------------
// iteration whose residual feeds the stopping test (its state is written back)
__device__ __forceinline__ bool is_check(const Params& P, int nu) {
  return P.tol > 0.0 && (nu + 1) % P.check_every == 0 && nu + 1 < P.iters;
}

// iteration whose state is written back to HBM in full (last iteration, stopping
// checks, the end of a write-back window)
__device__ __forceinline__ bool is_last(const Params& P, int nu) {
  return nu == P.iters - 1 || is_check(P, nu) || (s_win.wb_end && nu == s_win.nu1 - 1);
}

struct EpiConst {
  double cf, th, om, lam, ilam, lam_p;
  bool last, want, wt;
  double* Yn;
  bool pre;      // also leave the next iteration's fill (s -> x slot, psi^ -> u slot)
  double cfn;    // momentum coefficient of the next iteration
};

__device__ __forceinline__ EpiConst epi_const(const Params& P, int nu_it, double cf, double th, bool wt, int ncur,
                                              bool pre = false, double cfn = 0.0) {
  EpiConst k;
  k.pre = pre;
  k.cfn = cfn;
  k.cf = cf;
  k.th = th;
  k.om = __dsub_rn(1.0, th);
  k.lam = P.lam;
  k.ilam = P.inv_lam;
  k.lam_p = 1.0 / P.lam;
  k.last = is_last(P, nu_it);
  k.want = k.last || P.record_all;
  k.wt = wt;
  k.Yn = P.ybuf[ncur];
  return k;
}

#ifndef TSMPC_WANT_T
#define TSMPC_WANT_T 1
#endif
// psi block of row r, component k (k < n_u); u = the row's control component
template <bool WANT>
__device__ __forceinline__ void epi_psi_elem(const Ctx& c, const Params& P, const EpiConst& q, const int* d,
                                             int ysm, int k, double u, double& rmax, double ulo, double uhi) {
  const int e = d[0], st = d[1];
  double* row = s_dyn + d[4];
  const double* yc = row + (size_t)ysm * c.YW + 2 * c.NXP;
  double* yp = row + (size_t)(ysm ^ 1) * c.YW + 2 * c.NXP;
  const double dp = c.dpsi(st, k);
  const double w = extrap(yc[k], yp[k], q.cf);
  const double hp = __dmul_rn(u, dp);
  const double a = __dadd_rn(__dmul_rn(w, q.ilam), hp);
  const double t = dmin(dmax(a, __dmul_rn(dp, ulo)), __dmul_rn(dp, uhi));
  const double ny = __dadd_rn(w, __dmul_rn(q.lam, __dsub_rn(hp, t)));
  yp[k] = ny;
  if (q.pre) {  // the next backward's fill of this element (bwd_tile step 1)
    const double wn = extrap(ny, yc[k], q.cfn);
    s_dyn[d[3] + k] = c.scaled() ? __dmul_rn(wn, dp) : wn;
  }
  if (WANT && q.want) rmax = fmax(rmax, fabs(__dsub_rn(u, __ddiv_rn(t, dp))));
  double* ua = row + 2 * c.YW + c.NXP;
  const double na = __dadd_rn(__dmul_rn(ua[k], q.om), __dmul_rn(q.th, u));
  ua[k] = na;
  if (q.wt) {
    stcg(q.Yn + 2 * (size_t)c.E * c.NXP + (size_t)e * c.NUP + k, ny);
    stcg(P.uavg + (size_t)e * c.NUP + k, na);
  }
  if (q.last) stcg(P.U + (size_t)e * c.NUP + k, u);
}

// state blocks of rows described by rdesc, one warp per row.  WANT: the residual
// may be needed (compiled apart: otherwise ptxas if-converts its divisions into
// every element)
template <bool WANT>
__device__ __noinline__ void epi_state_t(int nu_it, double cf, double th, int nrows, int ysm, bool wt, int ncur,
                                         double* rmax_io, bool pre, double cfn) {
  const SParams& S = g_sp;
  const Ctx c = ctx_of();
  const Params& P = S.P;
  const EpiConst q = epi_const(P, nu_it, cf, th, wt, ncur, pre, cfn);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t E = (size_t)c.E;
  const double* xs_s = c.bnd;
  const double* xmn_s = c.bnd + c.NXP;
  const double* xmx_s = c.bnd + 2 * c.NXP;
  const int N = c.N;
  double rmax = *rmax_io;
  // the lane's bounds, hoisted (the row stores could alias them for the compiler)
  double bxs[4], bmn[4], bmx[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int i = lane + 32 * m;
    bxs[m] = i < c.nx ? xs_s[i] : 0.0;
    bmn[m] = i < c.nx ? xmn_s[i] : 0.0;
    bmx[m] = i < c.nx ? xmx_s[i] : 0.0;
  }
  // rows from the last warp down: the first warps carry the extra psi rows
  // (epi_psi_rows: row group g = warp / 4), so the warps with a second state row
  // are the ones with one psi row fewer
#pragma unroll 1
  for (int r = kWarpsS - 1 - warp; r < nrows; r += kWarpsS) {
    const int* d = c.rdesc() + 5 * r;
    const int e = d[0], st = d[1];
    double* row = s_dyn + d[4];
    const double* yc = row + (size_t)ysm * c.YW;
    double* yp = row + (size_t)(ysm ^ 1) * c.YW;
    double* xa = row + 2 * c.YW;
    const double* x = s_dyn + d[2];
    const double ds = c.scl[st], dz = c.scl[N + st];
    double ws[4], wz[4], ts[4], tz[4];
    double ss = 0.0, sz = 0.0;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int i = lane + 32 * m;
      ws[m] = wz[m] = ts[m] = tz[m] = 0.0;
      if (i < c.nx) {
        ws[m] = extrap(yc[i], yp[i], q.cf);
        wz[m] = extrap(yc[c.NXP + i], yp[c.NXP + i], q.cf);
        const double xi = x[i];
        ts[m] = __dadd_rn(__dmul_rn(ws[m], q.ilam), __dmul_rn(xi, ds));
        tz[m] = __dadd_rn(__dmul_rn(wz[m], q.ilam), __dmul_rn(xi, dz));
        const double gs_ = __dsub_rn(dmax(ts[m], __dmul_rn(ds, bxs[m])), ts[m]);
        const double gz = __dsub_rn(dmin(dmax(tz[m], __dmul_rn(dz, bmn[m])), __dmul_rn(dz, bmx[m])), tz[m]);
        ss = fma(gs_, gs_, ss);
        sz = fma(gz, gz, sz);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      ss += __shfl_xor_sync(0xffffffffu, ss, off);
      sz += __shfl_xor_sync(0xffffffffu, sz, off);
    }
    // factor min(1, weight / distance) (engine.py:146-155), as weight * rsqrt(distance^2):
    // the full IEEE sqrt + division sequences cost more than the rest of the row,
    // and the factor differs from weight / sqrt(.) by about one ulp
    const double wgt_s = __dmul_rn(__dmul_rn(q.lam_p, P.Wx), c.scl[2 * N + st]);
    const double wgt_z = __dmul_rn(__dmul_rn(q.lam_p, P.gamma_d), c.scl[3 * N + st]);
    const double fs = ss > __dmul_rn(wgt_s, wgt_s) ? __dmul_rn(wgt_s, rsqrt(ss)) : 1.0;
    const double fz = sz > __dmul_rn(wgt_z, wgt_z) ? __dmul_rn(wgt_z, rsqrt(sz)) : 1.0;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int i = lane + 32 * m;
      if (i < c.nx) {
        const double xi = x[i];
        const double hs = __dmul_rn(xi, ds), hz = __dmul_rn(xi, dz);
        const double ps = dmax(ts[m], __dmul_rn(ds, bxs[m]));
        const double pz = dmin(dmax(tz[m], __dmul_rn(dz, bmn[m])), __dmul_rn(dz, bmx[m]));
        const double t_s = __dadd_rn(ts[m], __dmul_rn(fs, __dsub_rn(ps, ts[m])));
        const double t_z = __dadd_rn(tz[m], __dmul_rn(fz, __dsub_rn(pz, tz[m])));
        const double ns = __dadd_rn(ws[m], __dmul_rn(q.lam, __dsub_rn(hs, t_s)));
        const double nz = __dadd_rn(wz[m], __dmul_rn(q.lam, __dsub_rn(hz, t_z)));
        yp[i] = ns;
        yp[c.NXP + i] = nz;
        if (WANT && q.want) {
          rmax = fmax(rmax, fabs(__dsub_rn(xi, __ddiv_rn(t_s, ds))));
          rmax = fmax(rmax, fabs(__dsub_rn(xi, __ddiv_rn(t_z, dz))));
        }
        const double na = __dadd_rn(__dmul_rn(xa[i], q.om), __dmul_rn(q.th, xi));
        xa[i] = na;
        if (q.wt) {
          stcg(q.Yn + (size_t)e * c.NXP + i, ns);
          stcg(q.Yn + E * c.NXP + (size_t)e * c.NXP + i, nz);
          stcg(P.xavg + (size_t)(e + 1) * c.NXP + i, na);
        }
        if (q.last) stcg(P.X + (size_t)(e + 1) * c.NXP + i, xi);
        if (q.pre) {  // the next backward's fill of this element (bwd_tile step 1)
          const double wsn = extrap(ns, yc[i], q.cfn), wzn = extrap(nz, yc[c.NXP + i], q.cfn);
          const_cast<double*>(x)[i] = __dadd_rn(__dmul_rn(wsn, ds), __dmul_rn(wzn, dz));
        }
      }
    }
  }
  *rmax_io = rmax;
}

// psi block of rows described by rdesc (component-major), u read from the rows
template <bool WANT>
__device__ __noinline__ void epi_psi_rows_t(int nu_it, double cf, double th, int nrows, int ysm, bool wt, int ncur,
                                            double* rmax_io, bool pre, double cfn) {
  const SParams& S = g_sp;
  const Ctx c = ctx_of();
  const Params& P = S.P;
  const EpiConst q = epi_const(P, nu_it, cf, th, wt, ncur, pre, cfn);
  const int k = threadIdx.x & (kKW - 1), g = threadIdx.x / kKW;
  double rmax = *rmax_io;
  if (k < c.nu) {
    // the component's bounds, hoisted (the row stores could alias them for the compiler)
    const double ulo = c.bnd[3 * c.NXP + k], uhi = c.bnd[3 * c.NXP + c.NUP + k];
#pragma unroll 1
    for (int r = g; r < nrows; r += kGroups) {
      const int* d = c.rdesc() + 5 * r;
      epi_psi_elem<WANT>(c, P, q, d, ysm, k, s_dyn[d[3] + k], rmax, ulo, uhi);
    }
  }
  *rmax_io = rmax;
}

__device__ __forceinline__ bool want_resid(const Params& P, int nu) { return is_last(P, nu) || P.record_all; }
__device__ __forceinline__ void epi_state(int nu_it, double cf, double th, int nrows, int ysm, bool wt, int ncur,
                                          double* rmax_io, bool pre = false, double cfn = 0.0) {
  if (!TSMPC_WANT_T || want_resid(g_sp.P, nu_it)) epi_state_t<true>(nu_it, cf, th, nrows, ysm, wt, ncur, rmax_io, pre, cfn);
  else epi_state_t<false>(nu_it, cf, th, nrows, ysm, wt, ncur, rmax_io, pre, cfn);
}
__device__ __forceinline__ void epi_psi_rows(int nu_it, double cf, double th, int nrows, int ysm, bool wt, int ncur,
                                             double* rmax_io, bool pre = false, double cfn = 0.0) {
  if (!TSMPC_WANT_T || want_resid(g_sp.P, nu_it)) epi_psi_rows_t<true>(nu_it, cf, th, nrows, ysm, wt, ncur, rmax_io, pre, cfn);
  else epi_psi_rows_t<false>(nu_it, cf, th, nrows, ysm, wt, ncur, rmax_io, pre, cfn);
}

// ----------------------------------------------------------------------------
// backward sweep of tile ti (reference factor.py:142-156).  t rows go to region
// A in place (tmode 0: the CTA's only tile stays in shared memory), to the
// tile's slot rows (tmode 1) or to HBM (tmode 2, streamed CTAs).
// ----------------------------------------------------------------------------
// the resident one-tile CTA's static vectors -> TMEM (apg_sparse_kernel)
__device__ __noinline__ void tm_static_fill_res() {
  tm_alloc_all();
  const SParams& S = g_sp;
  const Ctx c = ctx_of();
  const Params& P = S.P;
  const int row0 = c.mt.tiles[0], nrows = c.mt.tiles[1];
  const int k = threadIdx.x & (kKW - 1), g = threadIdx.x / kKW;
#pragma unroll 1
  for (int m = 0; m < 8; ++m) {
    const int r = g + kGroups * m;
    const bool ok = m < kRowsPT && r < nrows;
    const size_t e = ok ? (size_t)c.mt.edge(row0 + r) : 0;
    tm_st1(tm_addr(kTmRB + 2 * m), ok && k < c.nv ? ldcg(S.beta_s + e * c.NVP + k) : 0.0);
    tm_st1(tm_addr(kTmRU + 2 * m), ok && k < c.nu ? ldcg(P.uhat + e * c.NUP + k) : 0.0);
    tm_st1(tm_addr(kTmRE + 2 * m), ok && k < c.nx ? ldcg(P.evec + e * c.NXP + k) : 0.0);
  }
  tm_fill_done();
}

// TMS: the tile's static vectors are resident in TMEM (s_tm_on; compiled apart)
template <bool TMS>
__device__ __noinline__ void bwd_tile(int ti, double cf, int ysm, int srow0, bool resident, int cur,
                                      bool prefilled = false) {
  const SParams& S = g_sp;
  const Ctx c = ctx_of();
  const Params& P = S.P;
  const int* td = c.mt.tiles + 4 * ti;
  const int row0 = td[0], nrows = td[1], seg0 = td[2], nsegs = td[3];
  const int tid = threadIdx.x, k = tid & (kKW - 1), g = tid / kKW;
  const int nx = c.nx, nu = c.nu, nv = c.nv, N = c.N, LA = c.LA;
  const int tmode = c.mt.tmode;
  double* RA = c.A();
  double* RB = c.B();
  long long tm_ = clock64();
  (void)tm_;
  // prefetch beta_s (the bias of h) for this thread's rows
  double bpre[kRowsPT];
  if (TMS) {
    double b8[8];
    tm_ld8(tm_addr(kTmRB), b8);
    tm_wait_ld();
#pragma unroll
    for (int m = 0; m < kRowsPT; ++m) bpre[m] = b8[m];
  } else {
#pragma unroll
    for (int m = 0; m < kRowsPT; ++m) {
      const int r = g + kGroups * m;
      bpre[m] = 0.0;
      if (r < nrows && k < nv) bpre[m] = ldcg(S.beta_s + (size_t)c.mt.edge(row0 + r) * c.NVP + k);
    }
  }
  if (!resident) {
    cp_wait<0>();
    __syncthreads();
  }
  // (1) fill: s = D_sig w_sig + D_zeta w_zeta -> A ; psi^ = D_psi w_psi -> B
  // (prefilled: the previous iteration's epilogue left exactly these values)
#pragma unroll 1
  for (int m = 0; m < (prefilled ? 0 : kRowsPT); ++m) {
    const int r = g + kGroups * m;
    if (r >= nrows) break;
    const double* yc = slot_row(c, srow0 + r) + (size_t)ysm * c.YW;
    const double* yp = slot_row(c, srow0 + r) + (size_t)(ysm ^ 1) * c.YW;
    const int st = c.mt.stage(row0 + r);
    if (k < nx) {
      const double ws = extrap(yc[k], yp[k], cf);
      const double wz = extrap(yc[c.NXP + k], yp[c.NXP + k], cf);
      RA[r * LA + k] = __dadd_rn(__dmul_rn(ws, c.scl[st]), __dmul_rn(wz, c.scl[N + st]));
    }
    if (k < nu) {
      const double wp = extrap(yc[2 * c.NXP + k], yp[2 * c.NXP + k], cf);
      RB[r * c.NUP + k] = c.scaled() ? __dmul_rn(wp, c.dpsi(st, k)) : wp;
    }
  }
  __syncthreads();
  TSMPC_MARK(P, 0, tm_);
  if (S.split_heads && S.split_flags) {
    // split mode: the trunk needs only this chain's head values, which are linear in
    // the fill:  xiq_head = sum_d a^d s_d,  g_head = sum beta_s + Ls'(sum psi^ + B' sum_d G_d s_d)
    // (d = depth below the head, G_d = 1 + a + ... + a^d).  Publish them now; the
    // scans below produce the per-row t for this CTA's own forward.
    double* hb = s_dyn + S.O_HSUM;  // sum beta_s (NVP), set at launch start
    double* hp = hb + c.NVP;        // sum psi^ (NUP)
    double* hx = hp + c.NUP;        // sum_d G_d s_d (NXP)
    double* hz = hx + c.NXP;        // sum z (NUP)
    const int* sg = c.mt.segs + 4 * seg0;  // one chain per tile in split mode
    const int lo = sg[0], n = sg[1] - lo, head = c.mt.edge(row0 + lo);
    const bool pub = sg[2] >= 0;
    const double* adiag = c.adiag();
    if (pub) {
#pragma unroll 1
      for (int idx = tid; idx < nx + nu; idx += kThreadsS) {
        if (idx < nx) {
          const int i = idx;
          const double a = adiag[i];
          double xh = 0.0, xs = 0.0, pw = 1.0, gw = 1.0;
#pragma unroll 4
          for (int d = 0; d < n; ++d) {
            const double sv = RA[(lo + d) * LA + i];
            xh = fma(pw, sv, xh);
            xs = fma(gw, sv, xs);
            pw = __dmul_rn(pw, a);
            gw = __dadd_rn(gw, pw);
          }
          stcg(P.XIQG + (size_t)head * c.NXP + i, xh);
          hx[i] = xs;
        } else {
          const int j = idx - nx;
          double ps = 0.0;
#pragma unroll 4
          for (int d = 0; d < n; ++d) ps = __dadd_rn(ps, RB[(lo + d) * c.NUP + j]);
          hp[j] = ps;
        }
      }
      __syncthreads();
      if (tid < nu) {
        const int* cp = c.spi + S.Bc_ptr;
        const int* ci = c.spi + S.Bc_idx;
        const double* cv = c.spv + S.Bc_val;
        double z = hp[tid];
#pragma unroll 1
        for (int q = cp[tid]; q < cp[tid + 1]; ++q) z = fma(cv[q], hx[ci[q]], z);
        hz[tid] = z;
      }
      __syncthreads();
      if (tid < nv) {
        const int* cp = c.spi + S.Lc_ptr;
        const int* ci = c.spi + S.Lc_idx;
        const double* cv = c.spv + S.Lc_val;
        double h = 0.0;
#pragma unroll 1
        for (int q = cp[tid]; q < cp[tid + 1]; ++q) h = fma(cv[q], hz[ci[q]], h);
        stcg(P.GG + (size_t)head * c.NVP + tid, __dadd_rn(hb[tid], h));
      }
    }
    signal_arrive(S.sub_ctr + 1);
  }
  // streamed CTAs: the slot is free again -> prefetch the next tile's dual rows
  // (or, after the last backward tile, the ergodic rows the forward sweep needs)
  if (!resident) {
    const int* tn = c.mt.tiles + 4 * (ti > 0 ? ti - 1 : 0);
    load_rows(c.mt.rows + 4 * tn[0], 4, tn[1], c.slot, ti > 0 ? 1 : 2, cur, ysm);
    cp_commit();
  }
  // (2) xiq scan, tail -> head (leaf tails have no children: s + a .* 0 = s)
  const double* adiag = c.adiag();
#pragma unroll 1
  for (int idx = tid; idx < nsegs * nx; idx += kThreadsS) {
    const int s = idx / nx, i = idx - s * nx;
    const int* sg = c.mt.segs + 4 * (seg0 + s);
    const int lo = sg[0], n = sg[1] - lo;
    const double a = adiag[i];
    double* col = RA + lo * LA + i;
    double x = 0.0;
    // chunks of kCh rows: the loads of a chunk are in flight together, then the
    // dependent recursion runs from registers
#pragma unroll 1
    for (int j1 = n; j1 > 0; j1 -= kCh) {
      double v[kCh];
#pragma unroll
      for (int u = 0; u < kCh; ++u) v[u] = j1 - 1 - u >= 0 ? col[(j1 - 1 - u) * LA] : 0.0;
#pragma unroll
      for (int u = 0; u < kCh; ++u)
        if (j1 - 1 - u >= 0) {
          x = __dadd_rn(v[u], __dmul_rn(x, a));
          col[(j1 - 1 - u) * LA] = x;
        }
    }
    if (sg[2] >= 0 && !(S.split_heads && S.split_flags)) stcg(P.XIQG + (size_t)c.mt.edge(row0 + lo) * c.NXP + i, x);
  }
  __syncthreads();
  TSMPC_MARK(P, 1, tm_);
  // (3) z = psi^ + B' xiq   (column k of B)  B <- B + B' A
  if (k < nu) {
    const SpCol col = sp_col(c, S.Bc_ptr, S.Bc_idx, S.Bc_val, k);
#pragma unroll
    for (int m = 0; m < kRowsPT; ++m) {
      const int r = g + kGroups * m;
      if (r < nrows) RB[r * c.NUP + k] = sp_dot(c, col, S.Bc_idx, S.Bc_val, RA + r * LA, RB[r * c.NUP + k]);
    }
  }
  __syncthreads();
  TSMPC_MARK(P, 5, tm_);
  // (4) h = beta_s + Ls' z   (column k of Ls)  A <- beta_s + Ls' B
  if (k < nv) {
    const SpCol col = sp_col(c, S.Lc_ptr, S.Lc_idx, S.Lc_val, k);
#pragma unroll
    for (int m = 0; m < kRowsPT; ++m) {
      const int r = g + kGroups * m;
      if (r < nrows) RA[r * LA + k] = __dadd_rn(bpre[m], sp_dot(c, col, S.Lc_idx, S.Lc_val, RB + r * c.NUP, 0.0));
    }
  }
  __syncthreads();
  TSMPC_MARK(P, 2, tm_);
  // (5) g scan, tail -> head: g_e = h_e + g_child ; t_e = g_e / (2 p_e)
#pragma unroll 1
  for (int idx = tid; idx < nsegs * nv; idx += kThreadsS) {
    const int s = idx / nv, kk = idx - s * nv;
    const int* sg = c.mt.segs + 4 * (seg0 + s);
    const int lo = sg[0], n = sg[1] - lo;
    double* col = RA + lo * LA + kk;
    double gv = 0.0;
    double* tcol = tmode == 0 ? col : slot_row(c, srow0 + lo) + 2 * c.YW + c.NXP + c.NUP + kk;
    const int tld = tmode == 0 ? LA : c.SL;
#pragma unroll 1
    for (int j1 = n; j1 > 0; j1 -= kCh) {
      double v[kCh], ip[kCh];
#pragma unroll
      for (int u = 0; u < kCh; ++u) {
        const int j = j1 - 1 - u;
        v[u] = j >= 0 ? col[j * LA] : 0.0;
        ip[u] = j >= 0 ? c.mt.inv2p(row0 + lo + j) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kCh; ++u) {
        const int j = j1 - 1 - u;
        if (j >= 0) {
          gv = __dadd_rn(v[u], gv);
          const double t = __dmul_rn(gv, ip[u]);
          if (tmode == 2) stcg(S.TG + (size_t)c.mt.edge(row0 + lo + j) * c.NVP + kk, t);
          else tcol[j * tld] = t;
        }
      }
    }
    if (sg[2] >= 0 && !(S.split_heads && S.split_flags)) stcg(P.GG + (size_t)c.mt.edge(row0 + lo) * c.NVP + kk, gv);
  }
  __syncthreads();
  TSMPC_MARK(P, 3, tm_);
}

// ----------------------------------------------------------------------------
// forward sweep of tile ti (factor.py:158-170) + epilogue
// ----------------------------------------------------------------------------
template <bool TMS>
__device__ __noinline__ void fwd_tile(int ti, int nu_it, double cf, double th, int ysm,
                                      int srow0, bool resident, int cur, double* rmax) {
  const SParams& S = g_sp;
  const Ctx c = ctx_of();
  const Params& P = S.P;
  const int* td = c.mt.tiles + 4 * ti;
  const int row0 = td[0], nrows = td[1], seg0 = td[2], nsegs = td[3];
  const int tid = threadIdx.x, k = tid & (kKW - 1), g = tid / kKW;
  const int nx = c.nx, nu = c.nu, nv = c.nv, LA = c.LA;
  const int tmode = c.mt.tmode;
  double* RA = c.A();
  double* RB = c.B();
  long long tm_ = clock64();
  (void)tm_;
  if (!resident) {
    // t rows of this tile -> region A; then (after the previous epilogue) the slot
    {
      const int lane = tid & 31;
#pragma unroll 1
      for (int r = tid >> 5; r < nrows; r += kWarpsS) {
        const double* src = S.TG + (size_t)c.mt.edge(row0 + r) * c.NVP;
        for (int q = lane; q < c.NVP / 2; q += 32) cp16(RA + r * LA + 2 * q, src + 2 * q);
      }
    }
    cp_commit();
    if (ti > 0) load_rows(c.mt.rows + 4 * row0, 4, nrows, c.slot, 3, cur, ysm);
    cp_commit();
  }
  if (tid < nrows) {  // row descriptors of the epilogue
    int* d = c.rdesc() + 5 * tid;
    d[0] = c.mt.edge(row0 + tid);
    d[1] = c.mt.stage(row0 + tid);
    d[2] = (int)(RA + tid * LA - s_dyn);
    d[3] = (int)(RB + tid * c.NUP - s_dyn);
    d[4] = (int)(slot_row(c, srow0 + tid) - s_dyn);
  }
  // prefetch the static biases: uhat (u = uhat + du) and e (x recursion)
  double upre[kRowsPT], epre[kRowsPT];
  if (TMS) {
    double u8[8], e8[8];
    tm_ld8(tm_addr(kTmRU), u8);
    tm_ld8(tm_addr(kTmRE), e8);
    tm_wait_ld();
#pragma unroll
    for (int m = 0; m < kRowsPT; ++m) {
      upre[m] = u8[m];
      epre[m] = e8[m];
    }
  } else {
#pragma unroll
    for (int m = 0; m < kRowsPT; ++m) {
      const int r = g + kGroups * m;
      upre[m] = epre[m] = 0.0;
      if (r < nrows) {
        const int e = c.mt.edge(row0 + r);
        if (k < nu) upre[m] = ldcg(P.uhat + (size_t)e * c.NUP + k);
        if (k < nx) epre[m] = ldcg(P.evec + (size_t)e * c.NXP + k);
      }
    }
  }
  if (!resident) {
    cp_wait<1>();
    __syncthreads();
  }
  // (1) S scan, head -> tail: S_e = t_e + S_parent  (A, in place unless tmode 1)
#pragma unroll 1
  for (int idx = tid; idx < nsegs * nv; idx += kThreadsS) {
    const int s = idx / nv, kk = idx - s * nv;
    const int* sg = c.mt.segs + 4 * (seg0 + s);
    const int lo = sg[0], n = sg[1] - lo, pn = sg[2];
    double* scol = RA + lo * LA + kk;
    const double* tcol = tmode == 1 ? slot_row(c, srow0 + lo) + 2 * c.YW + c.NXP + c.NUP + kk : scol;
    const int tld = tmode == 1 ? c.SL : LA;
    double Sv = pn >= 0 && !S.split ? c.need[(size_t)pn * S.need_ld + kk] : 0.0;  // split: added later
#pragma unroll 1
    for (int j0 = 0; j0 < n; j0 += kCh) {
      double v[kCh];
#pragma unroll
      for (int u = 0; u < kCh; ++u) v[u] = j0 + u < n ? tcol[(j0 + u) * tld] : 0.0;
#pragma unroll
      for (int u = 0; u < kCh; ++u)
        if (j0 + u < n) {
          Sv = __dadd_rn(v[u], Sv);
          scol[(j0 + u) * LA] = Sv;
        }
    }
  }
  __syncthreads();
  TSMPC_MARK(P, 4, tm_);
  // (2) du = Lt S   (row k of Lt)  B <- Lt A
  if (k < nu) {
    const SpCol col = sp_col(c, S.Lr_ptr, S.Lr_idx, S.Lr_val, k);
#pragma unroll
    for (int m = 0; m < kRowsPT; ++m) {
      const int r = g + kGroups * m;
      if (r < nrows) RB[r * c.NUP + k] = sp_dot(c, col, S.Lr_idx, S.Lr_val, RA + r * LA, 0.0);
    }
  }
  __syncthreads();
  TSMPC_MARK(P, 11, tm_);
  // (3) bv + e = B du + e   (row k of B)  A <- B B + e
  if (k < nx) {
    const SpCol col = sp_col(c, S.Br_ptr, S.Br_idx, S.Br_val, k);
#pragma unroll
    for (int m = 0; m < kRowsPT; ++m) {
      const int r = g + kGroups * m;
      if (r < nrows) RA[r * LA + k] = __dadd_rn(sp_dot(c, col, S.Br_idx, S.Br_val, RB + r * c.NUP, 0.0), epre[m]);
    }
  }
  __syncthreads();
  TSMPC_MARK(P, 6, tm_);
  // (4) u = uhat + du (B) and the psi block of the epilogue (elementwise, u in a
  // register) ; x scan, head -> tail: x = a .* x_anc + (bv + e) (A)
  if (!resident) cp_wait<0>();  // the slot rows of a streamed tile
  __syncthreads();
  if (k < nu) {
#pragma unroll
    for (int m = 0; m < kRowsPT; ++m) {
      const int r = g + kGroups * m;
      if (r < nrows) RB[r * c.NUP + k] = __dadd_rn(RB[r * c.NUP + k], upre[m]);
    }
  }
  // the thread reads back only its own u entries: no barrier needed
  if (!S.split)
    epi_psi_rows(nu_it, cf, th, nrows, ysm, !resident || is_last(P, nu_it), cur ^ 1, rmax);
  {
    const double* adiag = c.adiag();
    const double* pr = c.proot();
#pragma unroll 1
    for (int idx = tid; idx < nsegs * nx; idx += kThreadsS) {
      const int s = idx / nx, i = idx - s * nx;
      const int* sg = c.mt.segs + 4 * (seg0 + s);
      const int lo = sg[0], n = sg[1] - lo, pn = sg[2];
      double* col = RA + lo * LA + i;
      double x = pn >= 0 ? (S.split ? 0.0 : c.need[(size_t)pn * S.need_ld + c.NVP + i]) : pr[i];
      const double a = adiag[i];
#pragma unroll 1
      for (int j0 = 0; j0 < n; j0 += kCh) {
        double v[kCh];
#pragma unroll
        for (int u = 0; u < kCh; ++u) v[u] = j0 + u < n ? col[(j0 + u) * LA] : 0.0;
#pragma unroll
        for (int u = 0; u < kCh; ++u)
          if (j0 + u < n) {
            x = __dadd_rn(__dmul_rn(x, a), v[u]);
            col[(j0 + u) * LA] = x;
          }
      }
    }
  }
  __syncthreads();
  TSMPC_MARK(P, 7, tm_);
  if (S.split) return;  // trunk terms and epilogue: fwd_finish, after the grid barrier
  // (5) epilogue, state blocks (warp per row)
  epi_state(nu_it, cf, th, nrows, ysm, !resident || is_last(P, nu_it), cur ^ 1, rmax);
  __syncthreads();
  TSMPC_MARK(P, 8, tm_);
}

// ----------------------------------------------------------------------------
// ----------------------------------------------------------------------------
// split mode, after the grid barrier: the chain's forward ran with zero trunk
// input; S, du, bv, x are affine in the trunk parent's values, so
//   u_e += du_tp                                   (du = Lt S, S_e = S_tp + local)
//   x_e += G_d .* (B du_tp) + a^(d+1) .* x_tp       (d = depth below the head,
//                                                    G_d = 1 + a + ... + a^d)
// with [du_tp | B du_tp | x_tp] read from TR.  Then the prox / dual epilogue.
// ----------------------------------------------------------------------------
__device__ __noinline__ void fwd_finish(int ti, int nu_it, double cf, double th, int ysm, bool resident, int cur,
                                        double* rmax) {
  const SParams& S = g_sp;
  const Ctx c = ctx_of();
  const Params& P = S.P;
  const int* td = c.mt.tiles + 4 * ti;
  const int nrows = td[1], seg0 = td[2], nsegs = td[3];
  const int tid = threadIdx.x, k = tid & (kKW - 1), g = tid / kKW;
  const int nx = c.nx, nu = c.nu, LA = c.LA;
  double* RA = c.A();
  double* RB = c.B();
  long long tm_ = clock64();
  (void)tm_;
  const bool last = is_last(P, nu_it);
  // one chain per tile in split mode
  const int pn = c.mt.segs[4 * seg0 + 2];
  // the parent's [du | B du | x] row, staged once (split_heads: in the head-sum
  // scratch after sum beta_s; else read through L2 where used)
  const double* tr = pn >= 0 ? S.TR + (size_t)pn * S.TR_LD : nullptr;
  if (pn >= 0 && S.split_heads) {
    double* st = s_dyn + S.O_HSUM + c.NVP;
    for (int q = tid; q < S.TR_LD; q += kThreadsS) st[q] = ldcg(tr + q);
    __syncthreads();
    tr = st;
  }
  if (pn >= 0 && k < nu) {
    const double d = tr[k];
#pragma unroll
    for (int m = 0; m < kRowsPT; ++m) {
      const int r = g + kGroups * m;
      if (r < nrows) RB[r * c.NUP + k] = __dadd_rn(RB[r * c.NUP + k], d);
    }
  }
  TSMPC_MARK(P, 13, tm_);
  if (pn >= 0 && S.a_unit) {
    // a = 1: G_d = d + 1 and a^(d+1) = 1 exactly, so every row is independent
    // (same values as the recurrence below)
    const int lo = c.mt.segs[4 * seg0];
#pragma unroll 1
    for (int idx = tid; idx < nrows * nx; idx += kThreadsS) {
      const int r = idx / nx, i = idx - r * nx;
      const double bt = tr[c.NUP + i], xt = tr[c.NUP + c.NXP + i];
      double* x = RA + r * LA + i;
      *x = __dadd_rn(*x, __dadd_rn(__dmul_rn((double)(r - lo + 1), bt), __dmul_rn(1.0, xt)));
    }
  } else if (pn >= 0) {
    const double* adiag = c.adiag();
#pragma unroll 1
    for (int idx = tid; idx < nsegs * nx; idx += kThreadsS) {
      const int s = idx / nx, i = idx - s * nx;
      const int* sg = c.mt.segs + 4 * (seg0 + s);
      const int lo = sg[0], n = sg[1] - lo;
      const double bt = tr[c.NUP + i], xt = tr[c.NUP + c.NXP + i];
      const double a = adiag[i];
      double* col = RA + lo * LA + i;
      double gs = 1.0, pw = a;
#pragma unroll 4
      for (int j = 0; j < n; ++j) {
        col[j * LA] = __dadd_rn(col[j * LA], __dadd_rn(__dmul_rn(gs, bt), __dmul_rn(pw, xt)));
        gs = __dadd_rn(__dmul_rn(gs, a), 1.0);
        pw = __dmul_rn(pw, a);
      }
    }
  }
  __syncthreads();
  TSMPC_MARK(P, 14, tm_);
  // psi and state blocks back to back: they write disjoint columns of the rows
  // prefill: the next iteration of this launch starts its backward without the fill
  const bool pre = S.split_heads && S.split_flags && nu_it + 1 < s_win.nu1;
  const double cfn = pre ? P.coef[nu_it + 1] : 0.0;
  epi_psi_rows(nu_it, cf, th, nrows, ysm, !resident || last, cur ^ 1, rmax, pre, cfn);
  TSMPC_MARK(P, 15, tm_);
  epi_state(nu_it, cf, th, nrows, ysm, !resident || last, cur ^ 1, rmax, pre, cfn);
  __syncthreads();
  TSMPC_MARK(P, 8, tm_);
}

// barrier among the trunk CTAs of split mode (arrival counter zeroed per launch)
__device__ __forceinline__ void trunk_barrier(unsigned int* ctr, unsigned int n, unsigned int& target) {
  __syncthreads();
  target += n;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    spin_until(ctr, target);
    __threadfence();
  }
  __syncthreads();
}

// phase B: component-sliced trunk sweep -> KY (see tsmpc_apg.cu trunk_sweep_smem
// for the recursion; here the schedule is staged in shared memory first)
// ----------------------------------------------------------------------------
__device__ __noinline__ void trunk_sweep(double cf, int cur, int part) {
  // part 1: own terms (no chain heads needed: run while waiting for them);
  // part 2: chain-head sums, levels, KY; part 3: both.  Each (edge, component)
  // element stays with the same thread across the parts.
  // Shard plans with a cut (S.n_xch > 0): part 5 (end of phase 1) runs the bottom-up
  // sums of the positions below the cut that this rank owns and exports the cut
  // positions' sums and the mixed positions' head sums to XCH; part 3 (phase 2, after
  // the cross-rank sum of XCH) imports the other ranks' cut sums instead of
  // computing them.  Positions foreign to this rank are skipped throughout.
  const SParams& S = g_sp;
  const Ctx c = ctx_of();
  const Params& P = S.P;
  const int ncomp = c.nv + c.nx + c.nu;
  // component slice of this CTA (split mode: among the trunk CTAs)
  const int si = S.split ? (int)blockIdx.x - S.split_c0 : (int)blockIdx.x;
  const int ns = S.split ? S.split_n : (int)gridDim.x;
  const int c_lo = (int)((long long)ncomp * si / ns);
  const int c_hi = (int)((long long)ncomp * (si + 1) / ns);
  const int nc = c_hi - c_lo;
  if (nc <= 0) return;
  const int* g = S.tsched;
  const int T = __ldg(g), nlev = __ldg(g + 1);
  double* Zs = S.sweep_in_a ? c.A() : c.B();
  double* Xs = Zs + (size_t)T * nc;
  double* Ip = Xs + (size_t)T * nc;  // 1 / (2 p) of each trunk edge
  long long ts_ = clock64();
  (void)ts_;
  const int* sch = g;  // schedule: resident / staged in shared memory when it fits, else via L1
  if (S.sched_resident) {
    sch = reinterpret_cast<const int*>(s_dyn + S.O_SCHED);
  } else if (S.sched_smem) {
    int* ss = reinterpret_cast<int*>(Ip + T);
    if (part & 1) {
#pragma unroll 1
      for (int i = threadIdx.x; i < S.n_tsched; i += kThreadsS) ss[i] = __ldg(g + i);
      __syncthreads();
    }
    sch = ss;
  }
  const int* lev = sch + 4;
  const int* pos = lev + nlev + 1;
  const int* tch = pos + 8 * T;
  const int* hch = tch + sch[2];
  const size_t E = (size_t)c.E;
  const double* Y = P.ybuf[cur];
  const double* Yp = P.ybuf[cur ^ 1];
  const double* adiag = c.adiag();
  TSMPC_MARK(P, 13, ts_);
  if (part & 1) {
    // (1a) own terms: beta (v), s = D_sig w_sig + D_zeta w_zeta (x), D_psi w_psi (u)
#pragma unroll 1
    for (int tp = threadIdx.x; tp < T; tp += kThreadsS) Ip[tp] = __ldg(P.inv2p + pos[8 * tp]);
#pragma unroll 1
    for (int idx = threadIdx.x; idx < T * nc; idx += kThreadsS) {
      const int tp = idx / nc, k = idx - tp * nc, q = c_lo + k;
      const int* ps = pos + 8 * tp;
      const int a = ps[0], st = ps[1], rl = ps[7] & 7;
      double z = 0.0, x = 0.0;
      if (rl == kRoleForeign || rl == kRoleCutForeign) {
        // another rank's subtree
      } else if (q < c.nv) {
        z = ldcg(S.beta_s + (size_t)a * c.NVP + q);
      } else if (q < c.nv + c.nx) {
        const int i = q - c.nv;
        const size_t o = (size_t)a * c.NXP + i;
        const double ws = extrap(ldcg(Y + o), ldcg(Yp + o), cf);
        const double wz = extrap(ldcg(Y + E * c.NXP + o), ldcg(Yp + E * c.NXP + o), cf);
        const double ds = c.scl[st], dz = c.scl[c.N + st];
        x = __dadd_rn(__dmul_rn(ws, ds), __dmul_rn(wz, dz));
      } else {
        const int j = q - c.nv - c.nx;
        const size_t o = 2 * E * c.NXP + (size_t)a * c.NUP + j;
        const double wp = extrap(ldcg(Y + o), ldcg(Yp + o), cf);
        z = c.scaled() ? __dmul_rn(wp, c.dpsi(st, j)) : wp;
      }
      Zs[idx] = z;
      Xs[idx] = x;
    }
  }
  if (!(part & 6)) return;
  if (part & 1) __syncthreads();  // the steps below map elements to threads differently
  const bool exporting = part & 4;
  auto kycol = [&](int q) {
    return q < c.nv ? q : (q < c.nv + c.nx ? c.NVP + (q - c.nv) : c.NVP + c.NXP + (q - c.nv - c.nx));
  };
  // per (trunk position, component) steps of the recursion
  auto heads = [&](int tp, int k) {  // (1b) chain-head children, childless fold
    const int q = c_lo + k, idx = tp * nc + k;
    const int* ps = pos + 8 * tp;
    const int h0 = ps[5], nh = ps[6], rl = ps[7] & 7;
    if (rl == kRoleForeign || (rl == kRoleMixed && exporting)) return;
    if (rl == kRoleCutForeign) {  // another rank's bottom-up sums (phase 2)
      if (!exporting) {
        const double* xr = S.XCH + (size_t)((ps[7] >> 3) - 1) * S.XCH_LD;
        Zs[idx] = ldcg(xr + kycol(q));
        Xs[idx] = q >= c.nv && q < c.nv + c.nx ? ldcg(xr + P.KY_LD + (q - c.nv)) : 0.0;
      }
      return;
    }
    // chain-head sums: this rank's (HS), or all ranks' for a mixed position (XCH)
    const double* hs = rl == kRoleMixed ? S.XCH + (size_t)((ps[7] >> 3) - 1) * S.XCH_LD : S.HS + (size_t)tp * S.HS_LD;
    double z = Zs[idx], x = Xs[idx];
    if (q < c.nv) {
      if (S.sharded) {
        if (nh > 0) z = __dadd_rn(z, ldcg(hs + q));
      } else {
#pragma unroll 1
        for (int m0 = 0; m0 < nh; m0 += kCh) {  // loads of a chunk in flight together
          double v[kCh];
#pragma unroll
          for (int u = 0; u < kCh; ++u) v[u] = m0 + u < nh ? ldcg(P.GG + (size_t)hch[h0 + m0 + u] * c.NVP + q) : 0.0;
#pragma unroll
          for (int u = 0; u < kCh; ++u)
            if (m0 + u < nh) z = __dadd_rn(z, v[u]);
        }
      }
    } else if (q < c.nv + c.nx) {
      const int i = q - c.nv;
      double h = 0.0;
      if (S.sharded) {
        if (nh > 0) h = ldcg(hs + c.NVP + i);
      } else {
#pragma unroll 1
        for (int m0 = 0; m0 < nh; m0 += kCh) {
          double v[kCh];
#pragma unroll
          for (int u = 0; u < kCh; ++u) v[u] = m0 + u < nh ? ldcg(P.XIQG + (size_t)hch[h0 + m0 + u] * c.NXP + i) : 0.0;
#pragma unroll
          for (int u = 0; u < kCh; ++u)
            if (m0 + u < nh) h = __dadd_rn(h, v[u]);
        }
      }
      x = __dadd_rn(x, __dmul_rn(h, adiag[i]));
    }
    if (ps[4] == 0) {  // no trunk children: the bottom-up step (children sums 0) here
      if (q >= c.nv && q < c.nv + c.nx) {
        x = __dadd_rn(x, __dmul_rn(0.0, adiag[q - c.nv]));
        z = __dadd_rn(x, 0.0);
      } else {
        z = __dadd_rn(z, 0.0);
      }
    }
    Zs[idx] = z;
    Xs[idx] = x;
  };
  auto up = [&](int tp, int k, int l) {  // (2) add trunk children; level 0 also scales
    const int q = c_lo + k, idx = tp * nc + k;
    const int* ps = pos + 8 * tp;
    const int c0 = ps[3], n = ps[4], rl = ps[7] & 7;
    if (rl == kRoleForeign || rl == kRoleCutForeign || (rl == kRoleMixed && exporting)) return;
    double zs = 0.0, xs = 0.0;
#pragma unroll 1
    for (int m = 0; m < n; ++m) {
      const int cp = tch[c0 + m];
      zs = __dadd_rn(zs, Zs[cp * nc + k]);
      xs = __dadd_rn(xs, Xs[cp * nc + k]);
    }
    double zn;
    if (q >= c.nv && q < c.nv + c.nx) {
      const double xiq = __dadd_rn(Xs[idx], __dmul_rn(xs, adiag[q - c.nv]));
      Xs[idx] = xiq;
      zn = __dadd_rn(xiq, zs);
    } else {
      zn = __dadd_rn(Zs[idx], zs);
    }
    Zs[idx] = l == 0 ? __dmul_rn(zn, Ip[tp]) : zn;
  };
  auto foreign = [&](int tp) {
    const int rl = pos[8 * tp + 7] & 7;
    return rl == kRoleForeign || rl == kRoleCutForeign;
  };
  auto down = [&](int tp, int k) {  // (3) K_a, Y_a = own * inv2p_a + parent's
    if (foreign(tp)) return;
    const int idx = tp * nc + k;
    const int pp = pos[8 * tp + 2];
    double v = __dmul_rn(Zs[idx], Ip[tp]);
    if (pp >= 0) v = __dadd_rn(v, Zs[pp * nc + k]);
    Zs[idx] = v;
  };
  auto store = [&](int tp, int k) {  // (4) KY column
    if (foreign(tp)) return;
    stcg(P.KY + (size_t)tp * P.KY_LD + kycol(c_lo + k), Zs[tp * nc + k]);
  };
#pragma unroll 1
  for (int idx = threadIdx.x; idx < T * nc; idx += kThreadsS) heads(idx / nc, idx % nc);
  __syncthreads();
  TSMPC_MARK(P, 14, ts_);
  if (S.split) {
    // levels: a warp per component (lanes over trunk positions), so every level
    // step of one component's recursion stays inside the warp (no block barriers)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll 1
    for (int k = warp; k < nc; k += kWarpsS) {
#pragma unroll 1
      for (int l = nlev - 2; l >= 0; --l) {
#pragma unroll 1
        for (int tp = lev[l] + lane; tp < lev[l + 1]; tp += 32) up(tp, k, l);
        __syncwarp();
      }
#pragma unroll 1
      for (int l = nlev >= 2 ? 1 : 0; l < nlev; ++l) {
#pragma unroll 1
        for (int tp = lev[l] + lane; tp < lev[l + 1]; tp += 32) down(tp, k);
        __syncwarp();
      }
#pragma unroll 1
      for (int tp = lane; tp < T; tp += 32) store(tp, k);
    }
    return;
  }
  // bottom-up over edge-stage levels (the deepest level has no trunk children:
  // done above); level 0 also takes its top-down step (no parent)
#pragma unroll 1
  for (int l = nlev - 2; l >= 0; --l) {
#pragma unroll 1
    for (int idx = lev[l] * nc + threadIdx.x; idx < lev[l + 1] * nc; idx += kThreadsS) up(idx / nc, idx % nc, l);
    __syncthreads();
  }
  if (exporting) {
    // every exchange row of this CTA's components: this rank's cut sums [Z | X] and
    // mixed-position head sums, zero where another rank contributes
#pragma unroll 1
    for (int idx = threadIdx.x; idx < T * nc; idx += kThreadsS) {
      const int tp = idx / nc, k = idx - tp * nc, q = c_lo + k;
      const int code = pos[8 * tp + 7], rl = code & 7;
      if ((code >> 3) == 0) continue;
      double* xr = S.XCH + (size_t)((code >> 3) - 1) * S.XCH_LD;
      double z = 0.0, x = 0.0;
      if (rl == kRoleCutOwn) {
        z = Zs[idx];
        x = Xs[idx];
      } else if (rl == kRoleMixed && q < c.nv + c.nx && S.towned[tp]) {
        z = ldcg(S.HS + (size_t)tp * S.HS_LD + (q < c.nv ? q : c.NVP + (q - c.nv)));
      }
      if (rl != kRoleMixed || q < c.nv + c.nx) stcg(xr + kycol(q), z);
      if (rl != kRoleMixed && q >= c.nv && q < c.nv + c.nx) stcg(xr + P.KY_LD + (q - c.nv), x);
    }
    return;
  }
#pragma unroll 1
  for (int l = nlev >= 2 ? 1 : 0; l < nlev; ++l) {
#pragma unroll 1
    for (int idx = lev[l] * nc + threadIdx.x; idx < lev[l + 1] * nc; idx += kThreadsS) down(idx / nc, idx % nc);
    __syncthreads();
  }
  TSMPC_MARK(P, 15, ts_);
#pragma unroll 1
  for (int idx = threadIdx.x; idx < T * nc; idx += kThreadsS) store(idx / nc, idx % nc);
}

// ----------------------------------------------------------------------------
// split mode, trunk CTA: the sweep of trunk_sweep restricted to the trunk
// subtrees holding this CTA's rows, for ALL components, in shared memory (the
// slot region is unused on trunk CTAs).  Every trunk CTA of a subtree repeats
// it, which replaces a barrier among the trunk CTAs and the KY round trip
// through L2; the KY rows of the CTA's needs go straight to the staging rows of
// trunk_needs (region B, pitch KY_LD + NUP + NXP).
// Meta section after `own`: {nsub, nslev, slev[nslev+1], sub tp[nsub], local index[T]}.
// ----------------------------------------------------------------------------
__device__ __noinline__ void trunk_sweep_local(double cf, int cur) {
  const SParams& S = g_sp;
  const Ctx c = ctx_of();
  const Params& P = S.P;
  const int* sb = c.mt.own + c.mt.nown;
  const int nsub = sb[0], nsl = sb[1];
  const int* slev = sb + 2;
  const int* stp = slev + nsl + 1;
  const int* lio = stp + nsub;
  const int ncomp = c.nv + c.nx + c.nu;
  double* Zs = s_dyn + S.O_SLOT;
  double* Xs = Zs + (size_t)nsub * ncomp;
  double* Ip = Xs + (size_t)nsub * ncomp;
  const int* g = S.tsched;
  const int T = __ldg(g), nlev = __ldg(g + 1);
  const int* sch = S.sched_resident ? reinterpret_cast<const int*>(s_dyn + S.O_SCHED) : g;
  const int* pos = sch + 4 + nlev + 1;
  const int* tch = pos + 8 * T;
  const int* hch = tch + sch[2];
  const size_t E = (size_t)c.E;
  const double* Y = P.ybuf[cur];
  const double* Yp = P.ybuf[cur ^ 1];
  const double* adiag = c.adiag();
#pragma unroll 1
  for (int li = threadIdx.x; li < nsub; li += kThreadsS) Ip[li] = __ldg(P.inv2p + pos[8 * stp[li]]);
  // (1) own terms + chain-head children
#pragma unroll 1
  for (int idx = threadIdx.x; idx < nsub * ncomp; idx += kThreadsS) {
    const int li = idx / ncomp, q = idx - li * ncomp;
    const int* ps = pos + 8 * stp[li];
    const int a = ps[0], st = ps[1], h0 = ps[5], nh = ps[6];
    double z = 0.0, x = 0.0;
    if (q < c.nv) {
      z = ldcg(S.beta_s + (size_t)a * c.NVP + q);
#pragma unroll 1
      for (int m0 = 0; m0 < nh; m0 += kCh) {
        double v[kCh];
#pragma unroll
        for (int u = 0; u < kCh; ++u) v[u] = m0 + u < nh ? ldcg(P.GG + (size_t)hch[h0 + m0 + u] * c.NVP + q) : 0.0;
#pragma unroll
        for (int u = 0; u < kCh; ++u)
          if (m0 + u < nh) z = __dadd_rn(z, v[u]);
      }
    } else if (q < c.nv + c.nx) {
      const int i = q - c.nv;
      const size_t o = (size_t)a * c.NXP + i;
      const double ws = extrap(ldcg(Y + o), ldcg(Yp + o), cf);
      const double wz = extrap(ldcg(Y + E * c.NXP + o), ldcg(Yp + E * c.NXP + o), cf);
      const double s = __dadd_rn(__dmul_rn(ws, c.scl[st]), __dmul_rn(wz, c.scl[c.N + st]));
      double h = 0.0;
#pragma unroll 1
      for (int m0 = 0; m0 < nh; m0 += kCh) {
        double v[kCh];
#pragma unroll
        for (int u = 0; u < kCh; ++u) v[u] = m0 + u < nh ? ldcg(P.XIQG + (size_t)hch[h0 + m0 + u] * c.NXP + i) : 0.0;
#pragma unroll
        for (int u = 0; u < kCh; ++u)
          if (m0 + u < nh) h = __dadd_rn(h, v[u]);
      }
      x = __dadd_rn(s, __dmul_rn(h, adiag[i]));
    } else {
      const int j = q - c.nv - c.nx;
      const size_t o = 2 * E * c.NXP + (size_t)a * c.NUP + j;
      const double wp = extrap(ldcg(Y + o), ldcg(Yp + o), cf);
      z = c.scaled() ? __dmul_rn(wp, c.dpsi(st, j)) : wp;
    }
    if (ps[4] == 0) {  // no trunk children: the bottom-up step (children sums 0) here
      if (q >= c.nv && q < c.nv + c.nx) {
        x = __dadd_rn(x, __dmul_rn(0.0, adiag[q - c.nv]));
        z = __dadd_rn(x, 0.0);
      } else {
        z = __dadd_rn(z, 0.0);
      }
    }
    Zs[idx] = z;
    Xs[idx] = x;
  }
  __syncthreads();
  // (2) bottom-up over the subtree levels: add trunk children (the deepest level
  // has none: done above); level 0 also takes its top-down step (no parent)
#pragma unroll 1
  for (int l = nsl - 2; l >= 0; --l) {
#pragma unroll 1
    for (int idx = slev[l] * ncomp + threadIdx.x; idx < slev[l + 1] * ncomp; idx += kThreadsS) {
      const int li = idx / ncomp, q = idx - li * ncomp;
      const int* ps = pos + 8 * stp[li];
      const int c0 = ps[3], n = ps[4];
      double zs = 0.0, xs = 0.0;
#pragma unroll 1
      for (int m = 0; m < n; ++m) {
        const int lc = lio[tch[c0 + m]];
        zs = __dadd_rn(zs, Zs[lc * ncomp + q]);
        xs = __dadd_rn(xs, Xs[lc * ncomp + q]);
      }
      double zn;
      if (q >= c.nv && q < c.nv + c.nx) {
        const double xiq = __dadd_rn(Xs[idx], __dmul_rn(xs, adiag[q - c.nv]));
        Xs[idx] = xiq;
        zn = __dadd_rn(xiq, zs);
      } else {
        zn = __dadd_rn(Zs[idx], zs);
      }
      Zs[idx] = l == 0 ? __dmul_rn(zn, Ip[li]) : zn;
    }
    __syncthreads();
  }
  // (3) top-down: K_a, Y_a = own * inv2p_a + parent's
#pragma unroll 1
  for (int l = nsl >= 2 ? 1 : 0; l < nsl; ++l) {
#pragma unroll 1
    for (int idx = slev[l] * ncomp + threadIdx.x; idx < slev[l + 1] * ncomp; idx += kThreadsS) {
      const int li = idx / ncomp, q = idx - li * ncomp;
      const int pp = pos[8 * stp[li] + 2];
      double v = __dmul_rn(Zs[idx], Ip[li]);
      if (pp >= 0) v = __dadd_rn(v, Zs[lio[pp] * ncomp + q]);
      Zs[idx] = v;
    }
    __syncthreads();
  }
  // (4) KY rows of the needs -> staging rows of trunk_needs
  const int SLD = P.KY_LD + c.NUP + c.NXP;
  const int* nd = c.mt.needs;
#pragma unroll 1
  for (int idx = threadIdx.x; idx < c.mt.nneed * ncomp; idx += kThreadsS) {
    const int n = idx / ncomp, q = idx - n * ncomp;
    const int col = q < c.nv ? q : (q < c.nv + c.nx ? c.NVP + (q - c.nv) : c.NVP + c.NXP + (q - c.nv - c.nx));
    c.B()[(size_t)n * SLD + col] = Zs[lio[nd[4 * n]] * ncomp + q];
  }
  // (trunk_needs starts with a barrier-protected staging round)
}

// ----------------------------------------------------------------------------
// sharded plans, end of phase 1: per trunk position, the sums over the chain heads
// hanging from its node (same order as the single-GPU sweep: children in node
// order) -> HS; zero where another rank owns those heads.  Grid-strided.
// ----------------------------------------------------------------------------
__device__ __noinline__ void head_prereduce() {
  const SParams& S = g_sp;
  const Ctx c = ctx_of();
  const Params& P = S.P;
  const int* g = S.tsched;
  const int T = __ldg(g), nlev = __ldg(g + 1);
  const int* pos = g + 4 + nlev + 1;
  const int* hch = pos + 8 * T + __ldg(g + 2);
  const int ncomp = c.nv + c.nx;
#pragma unroll 1
  for (int idx = blockIdx.x * kThreadsS + threadIdx.x; idx < T * ncomp; idx += gridDim.x * kThreadsS) {
    const int tp = idx / ncomp, q = idx - tp * ncomp;
    const int h0 = __ldg(pos + 8 * tp + 5), nh = __ldg(pos + 8 * tp + 6);
    double v = 0.0;
    if (S.towned[tp]) {
      if (q < c.nv) {
#pragma unroll 1
        for (int m = 0; m < nh; ++m) v = __dadd_rn(v, ldcg(P.GG + (size_t)__ldg(hch + h0 + m) * c.NVP + q));
      } else {
#pragma unroll 1
        for (int m = 0; m < nh; ++m)
          v = __dadd_rn(v, ldcg(P.XIQG + (size_t)__ldg(hch + h0 + m) * c.NXP + (q - c.nv)));
      }
    }
    stcg(S.HS + (size_t)tp * S.HS_LD + (q < c.nv ? q : c.NVP + (q - c.nv)), v);
  }
}

// ----------------------------------------------------------------------------
// phase D (trunk part): S, x, u of the needed trunk edges from KY
//   S = K + Ls'(B' Yx + Ypsi),  du = Lt S,  u = uhat + du,  x = a .* x_par + (B du + e)
// ----------------------------------------------------------------------------
__device__ __noinline__ void trunk_needs() {
  const SParams& S = g_sp;
  const Ctx c = ctx_of();
  const Params& P = S.P;
  const int nn = c.mt.nneed;
  if (nn == 0) return;
  long long tn_ = clock64();
  (void)tn_;
  const int nx = c.nx, nu = c.nu, nv = c.nv;
  const int LD = S.need_ld;
  const int* nd = c.mt.needs;
  // the u column of each need row holds Yz, then du, then u (no other scratch)
  double* const ND = c.need;
  const int UO = c.NVP + c.NXP;
  // KY, uhat and e rows of the needs, staged in region B in one round of loads
  // (else read through L2 where used)
  const int SLD = P.KY_LD + c.NUP + c.NXP;
  const bool staged = nn * SLD <= c.tcap * c.NUP;
  const double* KYs = c.B();
  if (staged) {
    const int hk = P.KY_LD / 2, hu = c.NUP / 2, hx = c.NXP / 2, per = hk + hu + hx;
#pragma unroll 1
    for (int idx = threadIdx.x; idx < nn * per; idx += kThreadsS) {
      const int n = idx / per, q = idx - n * per;
      double* dst = c.B() + (size_t)n * SLD;
      if (q < hk) {
        if (!S.split_local) cp16(dst + 2 * q, P.KY + (size_t)nd[4 * n] * P.KY_LD + 2 * q);
      }
      else if (q < hk + hu) cp16(dst + P.KY_LD + 2 * (q - hk), P.uhat + (size_t)nd[4 * n + 2] * c.NUP + 2 * (q - hk));
      else cp16(dst + P.KY_LD + c.NUP + 2 * (q - hk - hu), P.evec + (size_t)nd[4 * n + 2] * c.NXP + 2 * (q - hk - hu));
    }
    cp_commit();
    cp_wait<0>();
    __syncthreads();
  }
  TSMPC_MARK(P, 4, tn_);
  auto ky = [&](int n, int col) -> double {
    return staged ? KYs[(size_t)n * SLD + col] : ldcg(P.KY + (size_t)nd[4 * n] * P.KY_LD + col);
  };
  auto uhat_n = [&](int n, int j) -> double {
    return staged ? KYs[(size_t)n * SLD + P.KY_LD + j] : ldcg(P.uhat + (size_t)nd[4 * n + 2] * c.NUP + j);
  };
  auto evec_n = [&](int n, int i) -> double {
    return staged ? KYs[(size_t)n * SLD + P.KY_LD + c.NUP + i] : ldcg(P.evec + (size_t)nd[4 * n + 2] * c.NXP + i);
  };
  if (S.split && staged && S.tops) {
    // split mode: S is only an intermediate (the chains get du / B du / x from TR).
    // du = M1 KY and B du = M2 KY with the combined operators of the planner
    // (staged in this trunk CTA's slot region at launch), one pass; bv + e goes to
    // the (free) S columns for the x walk below
    const double* tv = s_dyn + S.O_SLOT + S.O_TOPS;
    const int* ti = reinterpret_cast<const int*>(tv + S.n_tpv);
    const int* m1p = ti + S.M1_ptr;
    const int* m1c = ti + S.M1_col;
    const double* m1v = tv + S.M1_val;
    const int* m2p = ti + S.M2_ptr;
    const int* m2c = ti + S.M2_col;
    const double* m2v = tv + S.M2_val;
#pragma unroll 1
    for (int idx = threadIdx.x; idx < nn * (nu + nx); idx += kThreadsS) {
      const int n = idx / (nu + nx), r = idx - n * (nu + nx);
      const double* kyr = KYs + (size_t)n * SLD;
      double acc = 0.0;
      if (r < nu) {
#pragma unroll 4
        for (int q = m1p[r]; q < m1p[r + 1]; ++q) acc = fma(m1v[q], kyr[m1c[q]], acc);
        ND[(size_t)n * LD + UO + r] = acc;
        stcg(S.TR + (size_t)nd[4 * n] * S.TR_LD + r, acc);  // du of the trunk row
      } else {
        const int i = r - nu;
#pragma unroll 4
        for (int q = m2p[i]; q < m2p[i + 1]; ++q) acc = fma(m2v[q], kyr[m2c[q]], acc);
        stcg(S.TR + (size_t)nd[4 * n] * S.TR_LD + c.NUP + i, acc);  // B du of the trunk row
        ND[(size_t)n * LD + i] = __dadd_rn(acc, evec_n(n, i));
      }
    }
    __syncthreads();
  } else {
  // (1) Yz = Ypsi + B' Yx
    {
      const int* cp = c.spi + S.Bc_ptr;
      const int* ci = c.spi + S.Bc_idx;
      const double* cv = c.spv + S.Bc_val;
  #pragma unroll 1
      for (int idx = threadIdx.x; idx < nn * nu; idx += kThreadsS) {
        const int n = idx / nu, j = idx - n * nu;
        double z = ky(n, c.NVP + c.NXP + j);
  #pragma unroll 1
        for (int q = cp[j]; q < cp[j + 1]; ++q) z = fma(cv[q], ky(n, c.NVP + ci[q]), z);
        ND[(size_t)n * LD + UO + j] = z;
      }
    }
    __syncthreads();
    TSMPC_MARK(P, 5, tn_);
    // (2) S = K + Ls' Yz
    {
      const int* cp = c.spi + S.Lc_ptr;
      const int* ci = c.spi + S.Lc_idx;
      const double* cv = c.spv + S.Lc_val;
  #pragma unroll 1
      for (int idx = threadIdx.x; idx < nn * nv; idx += kThreadsS) {
        const int n = idx / nv, k = idx - n * nv;
        double h = 0.0;
  #pragma unroll 1
        for (int q = cp[k]; q < cp[k + 1]; ++q) h = fma(cv[q], ND[(size_t)n * LD + UO + ci[q]], h);
        ND[(size_t)n * LD + k] = __dadd_rn(ky(n, k), h);
      }
    }
    __syncthreads();
    TSMPC_MARK(P, 6, tn_);
    // (3) du = Lt S
    {
      const int* rp = c.spi + S.Lr_ptr;
      const int* ri = c.spi + S.Lr_idx;
      const double* rv = c.spv + S.Lr_val;
  #pragma unroll 1
      for (int idx = threadIdx.x; idx < nn * nu; idx += kThreadsS) {
        const int n = idx / nu, j = idx - n * nu;
        double d = 0.0;
  #pragma unroll 1
        for (int q = rp[j]; q < rp[j + 1]; ++q) d = fma(rv[q], ND[(size_t)n * LD + ri[q]], d);
        ND[(size_t)n * LD + UO + j] = d;
        if (S.split) stcg(S.TR + (size_t)nd[4 * n] * S.TR_LD + j, d);  // du of the trunk row
      }
    }
    __syncthreads();
    TSMPC_MARK(P, 7, tn_);
  }
  // (4) bv + e ; then u = uhat + du ; then x level by level (parents first)
  {
    const int* rp = c.spi + S.Br_ptr;
    const int* ri = c.spi + S.Br_idx;
    const double* rv = c.spv + S.Br_val;
#pragma unroll 1
    for (int idx = threadIdx.x; idx < (S.split && staged && S.tops ? 0 : nn * nx); idx += kThreadsS) {
      const int n = idx / nx, i = idx - n * nx;
      double b = 0.0;
#pragma unroll 1
      for (int q = rp[i]; q < rp[i + 1]; ++q) b = fma(rv[q], ND[(size_t)n * LD + UO + ri[q]], b);
      if (S.split) stcg(S.TR + (size_t)nd[4 * n] * S.TR_LD + c.NUP + i, b);  // B du of the trunk row
      // split + staged: bv + e in the (free) S columns, so the x walk below can
      // write x in place without a copy-back pass
      ND[(size_t)n * LD + (S.split && staged ? 0 : c.NVP) + i] = __dadd_rn(b, evec_n(n, i));
    }
    if (!(S.split && staged && S.tops)) __syncthreads();
    TSMPC_MARK(P, 13, tn_);
    // u = uhat + du (independent of the x pass below: no barrier in between)
#pragma unroll 1
    for (int idx = threadIdx.x; idx < nn * nu; idx += kThreadsS) {
      const int n = idx / nu, j = idx - n * nu;
      double* u = ND + (size_t)n * LD + UO + j;
      *u = __dadd_rn(*u, uhat_n(n, j));
    }
    if (!staged) __syncthreads();
    // x of each need: a .* x_parent + (bv + e), down its root path
    const double* adiag = c.adiag();
    if (staged) {
      // one pass: each (need, component) walks its path upwards, weighting the
      // ancestors' (bv + e) by powers of a; the result goes to the staged KY
      // columns (no longer read) and is copied back after a barrier
      double* xo = c.B();
      const int bo = S.split ? 0 : c.NVP;  // where bv + e is
#pragma unroll 1
      for (int idx = threadIdx.x; idx < nn * nx; idx += kThreadsS) {
        const int n = idx / nx, i = idx - n * nx;
        const double a = adiag[i];
        double xv = ND[(size_t)n * LD + bo + i], m = a;
#pragma unroll 1
        for (int anc = nd[4 * n + 1]; anc >= 0; anc = nd[4 * anc + 1]) {
          xv = __dadd_rn(xv, __dmul_rn(m, ND[(size_t)anc * LD + bo + i]));
          m = __dmul_rn(m, a);
        }
        xv = __dadd_rn(xv, __dmul_rn(m, c.proot()[i]));
        if (S.split) {
          ND[(size_t)n * LD + c.NVP + i] = xv;
          stcg(S.TR + (size_t)nd[4 * n] * S.TR_LD + c.NUP + c.NXP + i, xv);
        } else {
          xo[(size_t)n * SLD + i] = xv;
        }
      }
      __syncthreads();
      if (!S.split) {
#pragma unroll 1
        for (int idx = threadIdx.x; idx < nn * nx; idx += kThreadsS) {
          const int n = idx / nx, i = idx - n * nx;
          ND[(size_t)n * LD + c.NVP + i] = xo[(size_t)n * SLD + i];
        }
        __syncthreads();
      }
    } else {
#pragma unroll 1
      for (int l = 0; l < c.mt.nlev; ++l) {
        const int n0 = c.mt.lev[l], n1 = c.mt.lev[l + 1];
#pragma unroll 1
        for (int idx = n0 * nx + threadIdx.x; idx < n1 * nx; idx += kThreadsS) {
          const int n = idx / nx, i = idx - n * nx;
          const int pn = nd[4 * n + 1];
          const double xp = pn >= 0 ? ND[(size_t)pn * LD + c.NVP + i] : c.proot()[i];
          double* xv = ND + (size_t)n * LD + c.NVP + i;
          *xv = __dadd_rn(__dmul_rn(xp, adiag[i]), *xv);
          if (S.split) stcg(S.TR + (size_t)nd[4 * n] * S.TR_LD + c.NUP + c.NXP + i, *xv);
        }
        __syncthreads();
      }
    }
  }
}


// epilogue of the CTA's own trunk rows (dual / ergodic rows live in HBM)
__device__ __noinline__ void trunk_own_rows(int nu_it, double cf, double th, int cur,
                                            double* rmax) {
  const SParams& S = g_sp;
  const Ctx c = ctx_of();
  const int no = c.mt.nown;
  if (no == 0) return;
  const int cap = max(1, min(kTileS, (kTileS * c.NUP) / c.SL));
  const int LD = S.need_ld;
  for (int b0 = 0; b0 < no; b0 += cap) {
    const int nb = min(cap, no - b0);
    const int* own = c.mt.own + b0;
    if (threadIdx.x < nb) {
      const int n = own[threadIdx.x];
      int* d = c.rdesc() + 5 * threadIdx.x;
      d[0] = c.mt.needs[4 * n + 2];
      d[1] = c.mt.needs[4 * n + 3];
      d[2] = (int)(c.need + (size_t)n * LD + c.NVP - s_dyn);
      d[3] = (int)(c.need + (size_t)n * LD + c.NVP + c.NXP - s_dyn);
      d[4] = (int)(c.B() + (size_t)threadIdx.x * c.SL - s_dyn);
    }
    __syncthreads();
    // stage the rows into the work region in slot format (dual at index 0 = HBM cur)
    load_rows(c.rdesc(), 5, nb, c.B(), 3, cur, 0);
    cp_commit();
    cp_wait<0>();
    __syncthreads();
    epi_psi_rows(nu_it, cf, th, nb, 0, true, cur ^ 1, rmax);
    epi_state(nu_it, cf, th, nb, 0, true, cur ^ 1, rmax);
    __syncthreads();
  }
}


// ============================================================================
// wide mode (SParams::wide, apg_wide_kernel): all chains of a CTA form one tile
// of up to kTileW rows (W4k: several such tiles), so every chain scan runs over
// nsegs x components threads at once; the dual (y, y_prev) and ergodic rows are
// never staged in shared memory but read from HBM / L2 into registers by the
// fill and the epilogue, in chunks of rows whose loads are issued together.
// XS: state components per lane in the warp-per-row state epilogue (n_x <= 32 XS).
// ============================================================================
#ifndef TSMPC_CHUNKW
#define TSMPC_CHUNKW 8
#endif
#ifndef TSMPC_R2
#define TSMPC_R2 2
#endif
#ifndef TSMPC_PREF
#define TSMPC_PREF 1
#endif
#ifndef TSMPC_WEAK
#define TSMPC_WEAK 0
#endif
#ifndef TSMPC_FASTEPI
#define TSMPC_FASTEPI 1
#endif
// state loads / stores of the wide epilogues: the rows are this CTA's own (or, for
// trunk rows, read by other CTAs only after a fenced barrier through L2)
__device__ __forceinline__ double epi_ld(const double* p) {
  if (TSMPC_WEAK & 1) return *p;
  return __ldcg(p);
}
__device__ __forceinline__ void epi_st(double* p, double v) {
  if (TSMPC_WEAK & 2) *p = v;
  else __stcg(p, v);
}
constexpr int kChunkW = TSMPC_CHUNKW;  // rows whose loads a thread issues before using them (epilogue)
constexpr int kChunkF = 4;   // the same for the (first-iteration) fill
constexpr int kRW = kTileW / kGroups;   // rows per thread of a wide tile, (group, component) mapping
constexpr int kG8 = kThreadsS / 64;     // row groups of the 64-lane mapping (components < 64)
constexpr int kRX = kTileW / kG8;       // rows per thread of a wide tile in that mapping

// ---- static per-row vectors in tensor memory (TMEM) ---------------------------
// A single-tile wide CTA (SMPC8's chain CTAs: 84 rows) reads, every iteration,
// beta_s (h phase), uhat and e (forward) of its rows: 84 x 280 doubles that do not
// change during the launch.  They are loaded once into TMEM (188 kB of the SM's
// 256 kB, unused otherwise: no MMA here) in the layout of the per-thread register
// prefetches of bwd_wide / fwd_wide, and each iteration reads them back with a
// few wide tcgen05.ld instead of 60 global loads per thread.  Every thread owns
// a private 128-column block of one TMEM lane (lane = tid % 128, columns
// 128 (tid / 128) ...):  beta_s of its kRW rows -> columns 0..47, uhat -> 48..95,
// e (64-lane mapping, kRX rows) -> 96..119.
#ifndef TSMPC_TMLATE
#define TSMPC_TMLATE 1
#endif
#ifndef TSMPC_TMSTATIC
#define TSMPC_TMSTATIC 1
#endif
constexpr int kTmB = 0, kTmU = 2 * kRW, kTmE = 4 * kRW;
static_assert(kTmE + 2 * kRX <= 128, "static TMEM block exceeds a thread's 128 columns");


// psi block of the rows in rdesc (component-major, as epi_psi_rows), state in HBM.
// WANT: this iteration's residual is needed (compiled apart: otherwise ptxas
// if-converts the residual's IEEE divisions into every element).  MODE 0: general
// (every condition tested at run time); MODE 1 / 2: the steady-state iteration
// (prefill, no output write-back, psi table in shared memory), without / with the
// split-mode trunk term folded in -- straight-line code over a full chunk of rows,
// so the elements' dependency chains interleave.
// trb_o (split mode): shared-memory offset of the tile's staged parent rows
// [du | B du | x] (stride trl), -1 if none; u += du_tp is folded in here.
template <bool WANT, int MODE>
__device__ __noinline__ void epi_psi_wide_t(int nu_it, double cf, double th, int nrows, int cur, double* rmax_io,
                                            int pre, double cfn, int trb_o, int trl, int seg0) {
  const SParams& S = g_sp;
  const Ctx c = ctx_of();
  const Params& P = S.P;
  const EpiConst q = epi_const(P, nu_it, cf, th, true, cur ^ 1, pre != 0, cfn);
  constexpr bool FAST = MODE != 0;
  const bool do_pre = FAST || q.pre, do_last = !FAST && q.last;
  const bool fgw = pre == 2;  // the next fill goes to FG (HBM), not to shared memory
  const bool fold = MODE == 2 || (MODE == 0 && trb_o >= 0);
  const int k = threadIdx.x & (kKW - 1), g = threadIdx.x / kKW;
  double rmax = *rmax_io;
  if (k < c.nu) {
    const double ulo = c.bnd[3 * c.NXP + k], uhi = c.bnd[3 * c.NXP + c.NUP + k];
    const size_t E = (size_t)c.E;
    const double* Yc = P.ybuf[cur] + 2 * E * c.NXP + k;
    double* Yn = P.ybuf[cur ^ 1] + 2 * E * c.NXP + k;
    double* UA = P.uavg + k;
    const int* rd = c.rdesc();
    const int psio = c.psi_o + k;
#pragma unroll 1
    for (int r0 = g; r0 < nrows; r0 += kChunkW * kGroups) {
      double yc[kChunkW], yp[kChunkW], ua[kChunkW];
      int eo[kChunkW];
#pragma unroll
      for (int u = 0; u < kChunkW; ++u) {
        const int r = r0 + u * kGroups;
        eo[u] = 0;
        yc[u] = yp[u] = ua[u] = 0.0;
        if (r < nrows) {
          eo[u] = rd[5 * r] * c.NUP;
          yc[u] = epi_ld(Yc + eo[u]);
          yp[u] = epi_ld(Yn + eo[u]);
          ua[u] = epi_ld(UA + eo[u]);
        }
      }
      auto elem = [&](int u, int r) {
        const int* d = rd + 5 * r;
        const int st = d[1];
        double* us = s_dyn + d[3] + k;
        double uu = *us;
        if (fold) {
          const int sg = d[4];
          const double du = s_dyn[trb_o + sg * trl + k];
          uu = c.mt.segs[4 * (seg0 + sg) + 2] >= 0 ? __dadd_rn(uu, du) : uu;
        }
        const double dp = FAST ? s_dyn[psio + st * c.NUP] : c.dpsi(st, k);
        const double w = extrap(yc[u], yp[u], q.cf);
        const double hp = __dmul_rn(uu, dp);
        const double a = __dadd_rn(__dmul_rn(w, q.ilam), hp);
        const double t = dmin(dmax(a, __dmul_rn(dp, ulo)), __dmul_rn(dp, uhi));
        const double ny = __dadd_rn(w, __dmul_rn(q.lam, __dsub_rn(hp, t)));
        epi_st(Yn + eo[u], ny);
        if (WANT && q.want) rmax = fmax(rmax, fabs(__dsub_rn(uu, __ddiv_rn(t, dp))));
        epi_st(UA + eo[u], __dadd_rn(__dmul_rn(ua[u], q.om), __dmul_rn(q.th, uu)));
        if (do_last) epi_st(P.U + eo[u] + k, uu);
        if (do_pre) {  // the next backward's fill of this element
          const double wn = extrap(ny, yc[u], q.cfn);
          const double fv = (FAST || c.scaled()) ? __dmul_rn(wn, dp) : wn;
          if (fgw) stcg(S.FG + (size_t)d[0] * S.FL + c.NXP + k, fv);
          else *us = fv;
        }
      };
      if (FAST && r0 + (kChunkW - 1) * kGroups < nrows) {
#pragma unroll
        for (int u = 0; u < kChunkW; ++u) elem(u, r0 + u * kGroups);
      } else {
#pragma unroll
        for (int u = 0; u < kChunkW; ++u)
          if (r0 + u * kGroups < nrows) elem(u, r0 + u * kGroups);
      }
    }
  }
  *rmax_io = rmax;
}

// state blocks of the rows in rdesc, one warp per row (R2 rows in flight), state in
// HBM.  WANT / MODE as for epi_psi_wide_t; the fold (split mode, A = I) adds
// x += (d + 1) B du_tp + x_tp.
template <int XS, bool WANT, int MODE, bool FGW>
__device__ __noinline__ void epi_state_wide_t(int nu_it, double cf, double th, int nrows, int cur, double* rmax_io,
                                              bool pre, double cfn, int trb_o, int trl, int seg0) {
  const SParams& S = g_sp;
  const Ctx c = ctx_of();
  const Params& P = S.P;
  const EpiConst q = epi_const(P, nu_it, cf, th, true, cur ^ 1, pre, cfn);
  constexpr bool FAST = MODE != 0;
  const bool do_pre = FAST || q.pre, do_last = !FAST && q.last;
  const bool fold = MODE == 2 || (MODE == 0 && trb_o >= 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t E = (size_t)c.E;
  const int N = c.N;
  double rmax = *rmax_io;
  double bxs[XS], bmn[XS], bmx[XS];
#pragma unroll
  for (int m = 0; m < XS; ++m) {
    const int i = lane + 32 * m;
    bxs[m] = i < c.nx ? c.bnd[i] : 0.0;
    bmn[m] = i < c.nx ? c.bnd[c.NXP + i] : 0.0;
    bmx[m] = i < c.nx ? c.bnd[2 * c.NXP + i] : 0.0;
  }
  const double* Ys = P.ybuf[cur];
  const double* Yz = Ys + E * c.NXP;
  double* Ns = P.ybuf[cur ^ 1];
  double* Nz = Ns + E * c.NXP;
  const int* rd = c.rdesc();
  constexpr int R2 = TSMPC_R2;
#pragma unroll 1
  for (int r0 = kWarpsS - 1 - warp; r0 < nrows; r0 += R2 * kWarpsS) {
    double ycs[R2][XS], yps[R2][XS], ycz[R2][XS], ypz[R2][XS], xav[R2][XS];
    int eo[R2];
#pragma unroll
    for (int h = 0; h < R2; ++h) {
      const int r = r0 + h * kWarpsS;
      eo[h] = r < nrows ? rd[5 * r] * c.NXP : 0;
#pragma unroll
      for (int m = 0; m < XS; ++m) {
        const int i = lane + 32 * m;
        const bool ok = r < nrows && i < c.nx;
        ycs[h][m] = ok ? epi_ld(Ys + eo[h] + i) : 0.0;
        yps[h][m] = ok ? epi_ld(Ns + eo[h] + i) : 0.0;
        ycz[h][m] = ok ? epi_ld(Yz + eo[h] + i) : 0.0;
        ypz[h][m] = ok ? epi_ld(Nz + eo[h] + i) : 0.0;
        xav[h][m] = ok ? epi_ld(P.xavg + eo[h] + c.NXP + i) : 0.0;
      }
    }
    auto row = [&](int h, int r) {
      const int* d = rd + 5 * r;
      const int st = d[1];
      double* x = s_dyn + d[2];
      const double ds = c.scl[st], dz = c.scl[N + st];
      double ws[XS], wz[XS], ts[XS], tz[XS], xv[XS];
      double ss = 0.0, sz = 0.0;
      int tpo = -1;        // the parent's [du | B du | x] row (split mode)
      double dep1 = 0.0;   // depth below the chain head + 1
      if (fold) {
        const int* sg = c.mt.segs + 4 * (seg0 + d[4]);
        tpo = sg[2] >= 0 ? trb_o + d[4] * trl : -1;
        dep1 = (double)(r - sg[0] + 1);
      }
#pragma unroll
      for (int m = 0; m < XS; ++m) {
        const int i = lane + 32 * m;
        ws[m] = wz[m] = ts[m] = tz[m] = xv[m] = 0.0;
        if (i < c.nx) {
          ws[m] = extrap(ycs[h][m], yps[h][m], q.cf);
          wz[m] = extrap(ycz[h][m], ypz[h][m], q.cf);
          xv[m] = x[i];
          if (fold && tpo >= 0)
            xv[m] = __dadd_rn(xv[m], __dadd_rn(__dmul_rn(dep1, s_dyn[tpo + c.NUP + i]),
                                               __dmul_rn(1.0, s_dyn[tpo + c.NUP + c.NXP + i])));
          ts[m] = __dadd_rn(__dmul_rn(ws[m], q.ilam), __dmul_rn(xv[m], ds));
          tz[m] = __dadd_rn(__dmul_rn(wz[m], q.ilam), __dmul_rn(xv[m], dz));
          const double ps = dmax(ts[m], __dmul_rn(ds, bxs[m]));
          const double pz = dmin(dmax(tz[m], __dmul_rn(dz, bmn[m])), __dmul_rn(dz, bmx[m]));
          const double gs_ = __dsub_rn(ps, ts[m]);
          const double gz = __dsub_rn(pz, tz[m]);
          ss = fma(gs_, gs_, ss);
          sz = fma(gz, gz, sz);
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        ss += __shfl_xor_sync(0xffffffffu, ss, off);
        sz += __shfl_xor_sync(0xffffffffu, sz, off);
      }
      // prox factor min(1, weight / distance) as weight * rsqrt(distance^2) (see epi_state)
      const double wgt_s = __dmul_rn(__dmul_rn(q.lam_p, P.Wx), c.scl[2 * N + st]);
      const double wgt_z = __dmul_rn(__dmul_rn(q.lam_p, P.gamma_d), c.scl[3 * N + st]);
      const double fs = ss > __dmul_rn(wgt_s, wgt_s) ? __dmul_rn(wgt_s, rsqrt(ss)) : 1.0;
      const double fz = sz > __dmul_rn(wgt_z, wgt_z) ? __dmul_rn(wgt_z, rsqrt(sz)) : 1.0;
#pragma unroll
      for (int m = 0; m < XS; ++m) {
        const int i = lane + 32 * m;
        if (i < c.nx) {
          const double xi = xv[m];
          const double hs = __dmul_rn(xi, ds), hz = __dmul_rn(xi, dz);
          const double ps = dmax(ts[m], __dmul_rn(ds, bxs[m]));
          const double pz = dmin(dmax(tz[m], __dmul_rn(dz, bmn[m])), __dmul_rn(dz, bmx[m]));
          const double t_s = __dadd_rn(ts[m], __dmul_rn(fs, __dsub_rn(ps, ts[m])));
          const double t_z = __dadd_rn(tz[m], __dmul_rn(fz, __dsub_rn(pz, tz[m])));
          const double ns = __dadd_rn(ws[m], __dmul_rn(q.lam, __dsub_rn(hs, t_s)));
          const double nz = __dadd_rn(wz[m], __dmul_rn(q.lam, __dsub_rn(hz, t_z)));
          epi_st(Ns + eo[h] + i, ns);
          epi_st(Nz + eo[h] + i, nz);
          if (WANT && q.want) {
            rmax = fmax(rmax, fabs(__dsub_rn(xi, __ddiv_rn(t_s, ds))));
            rmax = fmax(rmax, fabs(__dsub_rn(xi, __ddiv_rn(t_z, dz))));
          }
          epi_st(P.xavg + eo[h] + c.NXP + i, __dadd_rn(__dmul_rn(xav[h][m], q.om), __dmul_rn(q.th, xi)));
          if (do_last) epi_st(P.X + eo[h] + c.NXP + i, xi);
          if (do_pre) {  // the next backward's fill of this element
            const double wsn = extrap(ns, ycs[h][m], q.cfn), wzn = extrap(nz, ycz[h][m], q.cfn);
            const double fv = __dadd_rn(__dmul_rn(wsn, ds), __dmul_rn(wzn, dz));
            if (FGW) stcg(S.FG + (size_t)d[0] * S.FL + i, fv);
            else x[i] = fv;
          }
        }
      }
    };
    if (FAST && r0 + (R2 - 1) * kWarpsS < nrows) {
#pragma unroll
      for (int h = 0; h < R2; ++h) row(h, r0 + h * kWarpsS);
    } else {
#pragma unroll
      for (int h = 0; h < R2; ++h)
        if (r0 + h * kWarpsS < nrows) row(h, r0 + h * kWarpsS);  // warp-uniform
    }
  }
  *rmax_io = rmax;
}

__device__ __forceinline__ bool epi_fast(const Params& P, int nu_it, int pre) {
  return pre != 0 && !is_last(P, nu_it) && !P.record_all && P.scaled && g_sp.psi_smem;
}

#ifndef TSMPC_PSI2
#define TSMPC_PSI2 1
#endif
// The steady-state psi epilogue (MODE 1 / 2 of epi_psi_wide_t) on component pairs:
// 64-lane groups, 16-byte loads and stores of every array (half the memory
// instructions and row look-ups), the same operations per element in the same
// order (bitwise equal).  Needs even n_u and even shared-memory offsets.
template <int MODE, bool FGW>
__device__ __noinline__ void epi_psi_wide_v2(int nu_it, double cf, double th, int nrows, int cur, bool pre,
                                             double cfn, int trb_o, int trl, int seg0) {
  const SParams& S = g_sp;
  const Ctx c = ctx_of();
  const Params& P = S.P;
  const EpiConst q = epi_const(P, nu_it, cf, th, true, cur ^ 1, pre, cfn);
  constexpr int CH = 4, NG = kThreadsS / 64;
  const int k = 2 * (threadIdx.x & 63), g = threadIdx.x >> 6;
  if (k >= c.nu) return;
  const double2 ulo = *reinterpret_cast<const double2*>(c.bnd + 3 * c.NXP + k);
  const double2 uhi = *reinterpret_cast<const double2*>(c.bnd + 3 * c.NXP + c.NUP + k);
  const size_t E = (size_t)c.E;
  const double* Yc = P.ybuf[cur] + 2 * E * c.NXP + k;
  double* Yn = P.ybuf[cur ^ 1] + 2 * E * c.NXP + k;
  double* UA = P.uavg + k;
  const int* rd = c.rdesc();
  const int psio = c.psi_o + k;
  auto one = [&](double yc, double yp, double ua, double uu, double dp, double lo, double hi, double& ny, double& na,
                 double& fill) {
    const double w = extrap(yc, yp, q.cf);
    const double hp = __dmul_rn(uu, dp);
    const double a = __dadd_rn(__dmul_rn(w, q.ilam), hp);
    const double t = dmin(dmax(a, __dmul_rn(dp, lo)), __dmul_rn(dp, hi));
    ny = __dadd_rn(w, __dmul_rn(q.lam, __dsub_rn(hp, t)));
    na = __dadd_rn(__dmul_rn(ua, q.om), __dmul_rn(q.th, uu));
    fill = __dmul_rn(extrap(ny, yc, q.cfn), dp);
  };
#pragma unroll 1
  for (int r0 = g; r0 < nrows; r0 += CH * NG) {
    double2 yc[CH], yp[CH], ua[CH];
    int eo[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int r = r0 + u * NG;
      eo[u] = 0;
      yc[u] = yp[u] = ua[u] = make_double2(0.0, 0.0);
      if (r < nrows) {
        eo[u] = rd[5 * r] * c.NUP;
        yc[u] = __ldcg(reinterpret_cast<const double2*>(Yc + eo[u]));
        yp[u] = __ldcg(reinterpret_cast<const double2*>(Yn + eo[u]));
        ua[u] = __ldcg(reinterpret_cast<const double2*>(UA + eo[u]));
      }
    }
    auto elem = [&](int u, int r) {
      const int* d = rd + 5 * r;
      double2* us = reinterpret_cast<double2*>(s_dyn + d[3] + k);
      double2 uu = *us;
      if (MODE == 2) {
        const int sg = d[4];
        const double2 du = *reinterpret_cast<const double2*>(s_dyn + trb_o + sg * trl + k);
        if (c.mt.segs[4 * (seg0 + sg) + 2] >= 0) {
          uu.x = __dadd_rn(uu.x, du.x);
          uu.y = __dadd_rn(uu.y, du.y);
        }
      }
      const double2 dp = *reinterpret_cast<const double2*>(s_dyn + psio + d[1] * c.NUP);
      double2 ny, na, fl;
      one(yc[u].x, yp[u].x, ua[u].x, uu.x, dp.x, ulo.x, uhi.x, ny.x, na.x, fl.x);
      one(yc[u].y, yp[u].y, ua[u].y, uu.y, dp.y, ulo.y, uhi.y, ny.y, na.y, fl.y);
      __stcg(reinterpret_cast<double2*>(Yn + eo[u]), ny);
      __stcg(reinterpret_cast<double2*>(UA + eo[u]), na);
      if (FGW)  // the next backward's fill of this element pair
        __stcg(reinterpret_cast<double2*>(S.FG + (size_t)d[0] * S.FL + c.NXP + k), fl);
      else
        *us = fl;
    };
    if (r0 + (CH - 1) * NG < nrows) {
#pragma unroll
      for (int u = 0; u < CH; ++u) elem(u, r0 + u * NG);
    } else {
#pragma unroll
      for (int u = 0; u < CH; ++u)
        if (r0 + u * NG < nrows) elem(u, r0 + u * NG);
    }
  }
}
// epi_psi_wide_v2 applies: even n_u, 16-byte aligned rows in HBM and shared memory
__device__ __forceinline__ bool psi_pairs(int cur, int trb_o, int trl) {
  const Ctx c = ctx_of();
  const Params& P = g_sp.P;
  const size_t a = reinterpret_cast<size_t>(P.ybuf[cur]) | reinterpret_cast<size_t>(P.ybuf[cur ^ 1]) |
                   reinterpret_cast<size_t>(P.uavg) | reinterpret_cast<size_t>(s_dyn);
  const int o = c.nu | c.psi_o | (int)(c.B() - s_dyn) | (trb_o >= 0 ? (trb_o | trl) : 0) | (c.NXP * 2 * c.E);
  return (a & 15) == 0 && (o & 1) == 0;
}
// pre: 0 no next fill, 1 next fill into shared memory, 2 next fill into FG (HBM).
// FGD: the caller may ask for 2 (compiled apart: the one-tile CTAs, which never
// do, keep the dispatch -- and the register allocation -- without the FG variants)
template <bool FGD>
__device__ __forceinline__ void epi_psi_wide(int nu_it, double cf, double th, int nrows, int cur, double* rmax,
                                             int pre, double cfn, int trb_o = -1, int trl = 0, int seg0 = 0) {
  const Params& P = g_sp.P;
#ifdef TSMPC_KO
  if (TSMPC_KO & 1) return;  // timing experiment only: results are wrong
#endif
  if (!FGD) pre = pre != 0;
  if (!TSMPC_WANT_T || is_last(P, nu_it) || P.record_all)
    epi_psi_wide_t<true, 0>(nu_it, cf, th, nrows, cur, rmax, pre, cfn, trb_o, trl, seg0);
  else if (TSMPC_FASTEPI && epi_fast(P, nu_it, pre) && TSMPC_PSI2 && psi_pairs(cur, trb_o, trl))
    FGD && pre == 2
        ? (trb_o >= 0 ? epi_psi_wide_t<false, 0>(nu_it, cf, th, nrows, cur, rmax, pre, cfn, trb_o, trl, seg0)
                      : epi_psi_wide_v2<1, FGD>(nu_it, cf, th, nrows, cur, true, cfn, trb_o, trl, seg0))
        : trb_o >= 0 ? epi_psi_wide_v2<2, false>(nu_it, cf, th, nrows, cur, true, cfn, trb_o, trl, seg0)
                     : epi_psi_wide_v2<1, false>(nu_it, cf, th, nrows, cur, true, cfn, trb_o, trl, seg0);
  else if (TSMPC_FASTEPI && epi_fast(P, nu_it, pre))
    trb_o >= 0 ? epi_psi_wide_t<false, 2>(nu_it, cf, th, nrows, cur, rmax, pre, cfn, trb_o, trl, seg0)
               : epi_psi_wide_t<false, 1>(nu_it, cf, th, nrows, cur, rmax, pre, cfn, trb_o, trl, seg0);
  else
    epi_psi_wide_t<false, 0>(nu_it, cf, th, nrows, cur, rmax, pre, cfn, trb_o, trl, seg0);
}
template <int XS, bool FGD>
__device__ __forceinline__ void epi_state_wide(int nu_it, double cf, double th, int nrows, int cur, double* rmax,
                                               int pre, double cfn, int trb_o = -1, int trl = 0, int seg0 = 0) {
  const Params& P = g_sp.P;
#ifdef TSMPC_KO
  if (TSMPC_KO & 2) return;  // timing experiment only: results are wrong
#endif
  const bool pb = pre != 0;
  if (FGD && pre == 2) {  // next fill into FG
    if (!TSMPC_WANT_T || is_last(P, nu_it) || P.record_all)
      epi_state_wide_t<XS, true, 0, true>(nu_it, cf, th, nrows, cur, rmax, pb, cfn, trb_o, trl, seg0);
    else if (TSMPC_FASTEPI && epi_fast(P, nu_it, pre) && trb_o < 0)
      epi_state_wide_t<XS, false, 1, true>(nu_it, cf, th, nrows, cur, rmax, pb, cfn, trb_o, trl, seg0);
    else
      epi_state_wide_t<XS, false, 0, true>(nu_it, cf, th, nrows, cur, rmax, pb, cfn, trb_o, trl, seg0);
  } else if (!TSMPC_WANT_T || is_last(P, nu_it) || P.record_all)
    epi_state_wide_t<XS, true, 0, false>(nu_it, cf, th, nrows, cur, rmax, pb, cfn, trb_o, trl, seg0);
  else if (TSMPC_FASTEPI && epi_fast(P, nu_it, pre))
    trb_o >= 0 ? epi_state_wide_t<XS, false, 2, false>(nu_it, cf, th, nrows, cur, rmax, pb, cfn, trb_o, trl, seg0)
               : epi_state_wide_t<XS, false, 1, false>(nu_it, cf, th, nrows, cur, rmax, pb, cfn, trb_o, trl, seg0);
  else
    epi_state_wide_t<XS, false, 0, false>(nu_it, cf, th, nrows, cur, rmax, pb, cfn, trb_o, trl, seg0);
}

// backward sweep of wide tile ti (factor.py:142-156): fill from HBM (unless the
// previous epilogue left it), xiq scan, z = psi^ + B' xiq, h = beta_s + Ls' z,
// g scan -> t (region A in place for tmode 0, TG for tmode 2), chain heads -> GG / XIQG
// TMS: the CTA's static vectors are resident in TMEM (s_tm_on; compiled apart, so
// the multi-tile CTAs keep the plain prefetch code and its register allocation)
template <bool TMS, bool FGK>
__device__ __noinline__ void bwd_wide(int ti, double cf, int cur, int pf) {
  const SParams& S = g_sp;
  const Ctx c = ctx_of();
  const Params& P = S.P;
  const int* td = c.mt.tiles + 4 * ti;
  const int row0 = td[0], nrows = td[1], seg0 = td[2], nsegs = td[3];
  const int tid = threadIdx.x, k = tid & (kKW - 1), g = tid / kKW;
  const int nx = c.nx, nu = c.nu, nv = c.nv, N = c.N, LA = c.LA;
  const int tmode = c.mt.tmode;
  const size_t E = (size_t)c.E;
  double* RA = c.A();
  double* RB = c.B();
  long long tm_ = clock64();
  (void)tm_;
  // beta_s of this thread's rows for the h phase, loaded now (the loads are in
  // flight during the fill / head sums / xiq scan / z phases)
  double bpre[kRW];
  if (TMS) {  // resident in TMEM for the launch (read where used with TSMPC_TMLATE)
    static_assert(kRW % 8 == 0, "");
    if (!TSMPC_TMLATE) {
#pragma unroll
      for (int m = 0; m < kRW; m += 8) tm_ld8(tm_addr(kTmB + 2 * m), bpre + m);
      tm_wait_ld();
    }
  } else {
#pragma unroll
    for (int m = 0; m < kRW; ++m) {
      const int r = g + kGroups * m;
      bpre[m] = TSMPC_PREF && r < nrows && k < nv ? ldcg(S.beta_s + (size_t)c.mt.edge(row0 + r) * c.NVP + k) : 0.0;
    }
  }
  if (FGK && pf == 2 && TSMPC_BULK) {
    // (1) fill rows left in FG by the previous iteration's epilogue: [s | psi^] -> A | B,
    // two bulk copies per row
    const double* FG = S.FG;
    const int FL = S.FL, NXP = c.NXP, NUP = c.NUP;
    bulk_issue(2 * nrows, 8u * (unsigned)(nrows * FL), [&](int i) {
      const int r = i >> 1;
      const double* src = FG + (size_t)c.mt.edge(row0 + r) * FL;
      if (i & 1) bulk_row(RB + r * NUP, src + NXP, 8u * NUP, &s_bulk_bar);
      else bulk_row(RA + r * LA, src, 8u * NXP, &s_bulk_bar);
    });
    bulk_wait();
  } else if (FGK && pf == 2) {
    // (1) fill rows left in FG by the previous iteration's epilogue: [s | psi^] -> A | B
    const int hx = c.NXP / 2, per = hx + c.NUP / 2;
#pragma unroll 1
    for (int idx = tid; idx < nrows * per; idx += kThreadsS) {
      const int r = idx / per, q = idx - r * per;
      const double* src = S.FG + (size_t)c.mt.edge(row0 + r) * S.FL;
      if (q < hx) cp16(RA + r * LA + 2 * q, src + 2 * q);
      else cp16(RB + r * c.NUP + 2 * (q - hx), src + c.NXP + 2 * (q - hx));
    }
    cp_commit();
    cp_wait<0>();
    __syncthreads();
  } else if (pf == 0) {
    // (1) fill: s = D_sig w_sig + D_zeta w_zeta -> A ; psi^ = D_psi w_psi -> B
    const double* Y = P.ybuf[cur];
    const double* Yp = P.ybuf[cur ^ 1];
#pragma unroll 1
    for (int r0 = g; r0 < nrows; r0 += kChunkF * kGroups) {
      double a0[kChunkF], a1[kChunkF], a2[kChunkF], a3[kChunkF], b0[kChunkF], b1[kChunkF];
#pragma unroll
      for (int u = 0; u < kChunkF; ++u) {
        const int r = r0 + u * kGroups;
        a0[u] = a1[u] = a2[u] = a3[u] = b0[u] = b1[u] = 0.0;
        if (r < nrows) {
          const size_t e = (size_t)c.mt.edge(row0 + r);
          if (k < nx) {
            const size_t o = e * c.NXP + k;
            a0[u] = ldcg(Y + o);
            a1[u] = ldcg(Yp + o);
            a2[u] = ldcg(Y + E * c.NXP + o);
            a3[u] = ldcg(Yp + E * c.NXP + o);
          }
          if (k < nu) {
            const size_t o = 2 * E * c.NXP + e * c.NUP + k;
            b0[u] = ldcg(Y + o);
            b1[u] = ldcg(Yp + o);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kChunkF; ++u) {
        const int r = r0 + u * kGroups;
        if (r < nrows) {
          const int st = c.mt.stage(row0 + r);
          if (k < nx)
            RA[r * LA + k] = __dadd_rn(__dmul_rn(extrap(a0[u], a1[u], cf), c.scl[st]),
                                       __dmul_rn(extrap(a2[u], a3[u], cf), c.scl[N + st]));
          if (k < nu) {
            const double wp = extrap(b0[u], b1[u], cf);
            RB[r * c.NUP + k] = c.scaled() ? __dmul_rn(wp, c.dpsi(st, k)) : wp;
          }
        }
      }
    }
    __syncthreads();
  }
  TSMPC_MARK(P, 0, tm_);
  const double* adiag = c.adiag();
  TSMPC_STAMP(P, 6, s_trace_on);
  if (S.split) {
    // split mode: the trunk needs only each chain's head values, linear in the fill
    // (see bwd_tile):  xiq_head = sum_d a^d s_d,  g_head = sum beta_s + Ls'(sum psi^ + B' sum_d G_d s_d).
    // Per chain s of the tile: [sum beta_s] at hb + s NVP (launch constant), scratch
    // row [hx (NXP) | hp (NUP) | hz (NUP)] at hs + s HL.
    const double* hb = s_dyn + S.O_HSUM;
    double* hs = s_dyn + S.O_HSUM + S.hsum_nseg * c.NVP;
    const int HL = max(c.NXP + 2 * c.NUP, S.TR_LD);
#pragma unroll 1
    for (int idx = tid; idx < nsegs * (nx + nu); idx += kThreadsS) {
      const int s = idx / (nx + nu), q = idx - s * (nx + nu);
      const int* sg = c.mt.segs + 4 * (seg0 + s);
      if (sg[2] < 0) continue;
      const int lo = sg[0], n = sg[1] - lo;
      if (q < nx) {
        const double a = adiag[q];
        double xh = 0.0, xs = 0.0, pw = 1.0, gw = 1.0;
#pragma unroll 4
        for (int d = 0; d < n; ++d) {
          const double sv = RA[(lo + d) * LA + q];
          xh = fma(pw, sv, xh);
          xs = fma(gw, sv, xs);
          pw = __dmul_rn(pw, a);
          gw = __dadd_rn(gw, pw);
        }
        stcg(P.XIQG + (size_t)c.mt.edge(row0 + lo) * c.NXP + q, xh);
        hs[s * HL + q] = xs;
      } else {
        const int j = q - nx;
        double ps = 0.0;
#pragma unroll 4
        for (int d = 0; d < n; ++d) ps = __dadd_rn(ps, RB[(lo + d) * c.NUP + j]);
        hs[s * HL + c.NXP + j] = ps;
      }
    }
    __syncthreads();
    TSMPC_STAMP(P, 7, s_trace_on);
    {
      const int* cp = c.spi + S.Bc_ptr;
      const int* ci = c.spi + S.Bc_idx;
      const double* cv = c.spv + S.Bc_val;
#pragma unroll 1
      for (int idx = tid; idx < nsegs * nu; idx += kThreadsS) {
        const int s = idx / nu, j = idx - s * nu;
        if (c.mt.segs[4 * (seg0 + s) + 2] < 0) continue;
        const double* h = hs + s * HL;
        double z = h[c.NXP + j];
#pragma unroll 1
        for (int q = cp[j]; q < cp[j + 1]; ++q) z = fma(cv[q], h[ci[q]], z);
        hs[s * HL + c.NXP + c.NUP + j] = z;
      }
    }
    __syncthreads();
    {
      const int* cp = c.spi + S.Lc_ptr;
      const int* ci = c.spi + S.Lc_idx;
      const double* cv = c.spv + S.Lc_val;
#pragma unroll 1
      for (int idx = tid; idx < nsegs * nv; idx += kThreadsS) {
        const int s = idx / nv, k2 = idx - s * nv;
        const int* sg = c.mt.segs + 4 * (seg0 + s);
        if (sg[2] < 0) continue;
        const double* hz = hs + s * HL + c.NXP + c.NUP;
        double h = 0.0;
#pragma unroll 1
        for (int q = cp[k2]; q < cp[k2 + 1]; ++q) h = fma(cv[q], hz[ci[q]], h);
        stcg(P.GG + (size_t)c.mt.edge(row0 + sg[0]) * c.NVP + k2, __dadd_rn(hb[s * c.NVP + k2], h));
      }
    }
    signal_arrive(S.sub_ctr + 1);
    TSMPC_STAMP(P, 5, s_trace_on);
  }
  // (2) xiq scan, tail -> head, every chain of the tile at once
#pragma unroll 1
  for (int idx = tid; idx < nsegs * nx; idx += kThreadsS) {
    const int s = idx / nx, i = idx - s * nx;
    const int* sg = c.mt.segs + 4 * (seg0 + s);
    const int lo = sg[0], n = sg[1] - lo;
    const double a = adiag[i];
    double* col = RA + lo * LA + i;
    double x = 0.0;
#pragma unroll 1
    for (int j1 = n; j1 > 0; j1 -= kCh) {
      double v[kCh];
#pragma unroll
      for (int u = 0; u < kCh; ++u) v[u] = j1 - 1 - u >= 0 ? col[(j1 - 1 - u) * LA] : 0.0;
#pragma unroll
      for (int u = 0; u < kCh; ++u)
        if (j1 - 1 - u >= 0) {
          x = __dadd_rn(v[u], __dmul_rn(x, a));
          col[(j1 - 1 - u) * LA] = x;
        }
    }
    if (sg[2] >= 0 && !S.split) stcg(P.XIQG + (size_t)c.mt.edge(row0 + lo) * c.NXP + i, x);
  }
  __syncthreads();
  TSMPC_MARK(P, 1, tm_);
  // (3) z = psi^ + B' xiq (column k of B), B <- B + B' A
  if (k < nu) {
    const SpCol col = sp_col(c, S.Bc_ptr, S.Bc_idx, S.Bc_val, k);
#pragma unroll (kUnr)
    for (int r = g; r < nrows; r += kGroups)
      RB[r * c.NUP + k] = sp_dot(c, col, S.Bc_idx, S.Bc_val, RA + r * LA, RB[r * c.NUP + k]);
  }
  __syncthreads();
  TSMPC_MARK(P, 5, tm_);
  // (4) h = beta_s + Ls' z (column k of Ls), A <- beta_s + Ls' B
  if (TMS && TSMPC_TMLATE) {
#pragma unroll
    for (int m = 0; m < kRW; m += 8) tm_ld8(tm_addr(kTmB + 2 * m), bpre + m);
    tm_wait_ld();
  }
  if (k < nv) {
    const SpCol col = sp_col(c, S.Lc_ptr, S.Lc_idx, S.Lc_val, k);
#pragma unroll
    for (int m = 0; m < kRW; ++m) {
      const int r = g + kGroups * m;
      if (r < nrows)
        RA[r * LA + k] = __dadd_rn(TSMPC_PREF ? bpre[m] : ldcg(S.beta_s + (size_t)c.mt.edge(row0 + r) * c.NVP + k),
                                   sp_dot(c, col, S.Lc_idx, S.Lc_val, RB + r * c.NUP, 0.0));
    }
  }
  __syncthreads();
  TSMPC_MARK(P, 2, tm_);
  // (5) g scan, tail -> head: g_e = h_e + g_child ; t_e = g_e / (2 p_e)
#pragma unroll 1
  for (int idx = tid; idx < nsegs * nv; idx += kThreadsS) {
    const int s = idx / nv, kk = idx - s * nv;
    const int* sg = c.mt.segs + 4 * (seg0 + s);
    const int lo = sg[0], n = sg[1] - lo;
    double* col = RA + lo * LA + kk;
    double gv = 0.0;
#pragma unroll 1
    for (int j1 = n; j1 > 0; j1 -= kCh) {
      double v[kCh], ip[kCh];
#pragma unroll
      for (int u = 0; u < kCh; ++u) {
        const int j = j1 - 1 - u;
        v[u] = j >= 0 ? col[j * LA] : 0.0;
        ip[u] = j >= 0 ? c.mt.inv2p(row0 + lo + j) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kCh; ++u) {
        const int j = j1 - 1 - u;
        if (j >= 0) {
          gv = __dadd_rn(v[u], gv);
          const double t = __dmul_rn(gv, ip[u]);
          if (tmode == 2) stcg(S.TG + (size_t)c.mt.edge(row0 + lo + j) * c.NVP + kk, t);
          else col[j * LA] = t;
        }
      }
    }
    if (sg[2] >= 0 && !S.split) stcg(P.GG + (size_t)c.mt.edge(row0 + lo) * c.NVP + kk, gv);
  }
  __syncthreads();
  TSMPC_MARK(P, 3, tm_);
}

// forward sweep of wide tile ti (factor.py:158-170) + epilogue; in split mode the
// chains run with zero trunk input and the trunk terms and the epilogue follow in
// fwd_finish_wide
template <int XS, bool TMS, bool FGK>
__device__ __noinline__ void fwd_wide(int ti, int nu_it, double cf, double th, int cur, double* rmax, int pre,
                                      double cfn) {
  const SParams& S = g_sp;
  const Ctx c = ctx_of();
  const Params& P = S.P;
  const int* td = c.mt.tiles + 4 * ti;
  const int row0 = td[0], nrows = td[1], seg0 = td[2], nsegs = td[3];
  const int tid = threadIdx.x, k = tid & (kKW - 1), g = tid / kKW;
  const int nx = c.nx, nu = c.nu, nv = c.nv, LA = c.LA;
  double* RA = c.A();
  double* RB = c.B();
  long long tm_ = clock64();
  (void)tm_;
  // e (64-lane mapping, components < 64) and uhat of this thread's rows, loaded now
  // (in flight during the S scan and du phases)
  const int k8 = tid & 63, g8 = tid >> 6;
  const bool x64 = nx <= 64;
  double epre[kRX], upre[kRW];
  auto tm_ld_e = [&]() {
    double e8[(kRX + 7) / 8 * 8];
#pragma unroll
    for (int m = 0; m < kRX; m += 8) tm_ld8(tm_addr(kTmE + 2 * m), e8 + m);
    tm_wait_ld();
#pragma unroll
    for (int m = 0; m < kRX; ++m) epre[m] = e8[m];
  };
  auto tm_ld_u = [&]() {
#pragma unroll
    for (int m = 0; m < kRW; m += 8) tm_ld8(tm_addr(kTmU + 2 * m), upre + m);
    tm_wait_ld();
  };
  if (TMS) {  // resident in TMEM for the launch (read where used with TSMPC_TMLATE)
    static_assert(kRX % 4 == 0 && kRW % 8 == 0, "");
    if (!TSMPC_TMLATE) {
      tm_ld_u();
      tm_ld_e();
    }
  } else {
#pragma unroll
    for (int m = 0; m < kRX; ++m) {
      const int r = g8 + kG8 * m;
      epre[m] = TSMPC_PREF && x64 && r < nrows && k8 < nx ? ldcg(P.evec + (size_t)c.mt.edge(row0 + r) * c.NXP + k8) : 0.0;
    }
#pragma unroll
    for (int m = 0; m < kRW; ++m) {
      const int r = g + kGroups * m;
      upre[m] = TSMPC_PREF && r < nrows && k < nu ? ldcg(P.uhat + (size_t)c.mt.edge(row0 + r) * c.NUP + k) : 0.0;
    }
  }
  const bool tg_bulk = FGK && TSMPC_BULK && c.mt.tmode == 2;
  if (tg_bulk) {  // t rows of this tile -> region A, a bulk copy per row (waited for below)
    bulk_issue(nrows, 8u * (unsigned)(nrows * c.NVP), [&](int r) {
      bulk_row(RA + r * LA, S.TG + (size_t)c.mt.edge(row0 + r) * c.NVP, 8u * c.NVP, &s_bulk_bar);
    });
  } else if (c.mt.tmode == 2) {  // t rows of this tile -> region A
    const int lane = tid & 31;
#pragma unroll 1
    for (int r = tid >> 5; r < nrows; r += kWarpsS) {
      const double* src = S.TG + (size_t)c.mt.edge(row0 + r) * c.NVP;
      for (int q = lane; q < c.NVP / 2; q += 32) cp16(RA + r * LA + 2 * q, src + 2 * q);
    }
    cp_commit();
  }
#pragma unroll 1
  for (int r = tid; r < nrows; r += kThreadsS) {  // row descriptors of the epilogue
    int* d = c.rdesc() + 5 * r;
    d[0] = c.mt.edge(row0 + r);
    d[1] = c.mt.stage(row0 + r);
    d[2] = (int)(RA + r * LA - s_dyn);
    d[3] = (int)(RB + r * c.NUP - s_dyn);
    if (!S.split) d[4] = 0;
  }
  if (S.split && tid < nsegs) {  // segment of every row (trunk terms of fwd_finish_wide)
    const int* sg = c.mt.segs + 4 * (seg0 + tid);
    for (int r = sg[0]; r < sg[1]; ++r) c.rdesc()[5 * r + 4] = tid;
  }
  if (tg_bulk) bulk_wait();
  else if (c.mt.tmode == 2) cp_wait<0>();
  __syncthreads();
  // (1) S scan, head -> tail: S_e = t_e + S_parent (A, in place)
#pragma unroll 1
  for (int idx = tid; idx < nsegs * nv; idx += kThreadsS) {
    const int s = idx / nv, kk = idx - s * nv;
    const int* sg = c.mt.segs + 4 * (seg0 + s);
    const int lo = sg[0], n = sg[1] - lo, pn = sg[2];
    double* scol = RA + lo * LA + kk;
    double Sv = pn >= 0 && !S.split ? c.need[(size_t)pn * S.need_ld + kk] : 0.0;  // split: added later
#pragma unroll 1
    for (int j0 = 0; j0 < n; j0 += kCh) {
      double v[kCh];
#pragma unroll
      for (int u = 0; u < kCh; ++u) v[u] = j0 + u < n ? scol[(j0 + u) * LA] : 0.0;
#pragma unroll
      for (int u = 0; u < kCh; ++u)
        if (j0 + u < n) {
          Sv = __dadd_rn(v[u], Sv);
          scol[(j0 + u) * LA] = Sv;
        }
    }
  }
  __syncthreads();
  TSMPC_MARK(P, 4, tm_);
  // (2) du = Lt S (row k of Lt), B <- Lt A
  if (k < nu) {
    const SpCol col = sp_col(c, S.Lr_ptr, S.Lr_idx, S.Lr_val, k);
#pragma unroll (kUnr)
    for (int r = g; r < nrows; r += kGroups) RB[r * c.NUP + k] = sp_dot(c, col, S.Lr_idx, S.Lr_val, RA + r * LA, 0.0);
  }
  __syncthreads();
  TSMPC_MARK(P, 11, tm_);
  // (3) bv + e = B du + e (row k of B), A <- B B + e; 64 lanes x 8 row groups
  // when n_x <= 64 (every thread busy), else the (group, component) mapping
  if (TMS && TSMPC_TMLATE) tm_ld_e();
  if (x64) {
    if (k8 < nx) {
      const SpCol col = sp_col(c, S.Br_ptr, S.Br_idx, S.Br_val, k8);
#pragma unroll
      for (int m = 0; m < kRX; ++m) {
        const int r = g8 + kG8 * m;
        if (r < nrows)
          RA[r * LA + k8] = __dadd_rn(sp_dot(c, col, S.Br_idx, S.Br_val, RB + r * c.NUP, 0.0),
                                      TSMPC_PREF ? epre[m] : ldcg(P.evec + (size_t)c.mt.edge(row0 + r) * c.NXP + k8));
      }
    }
  } else if (k < nx) {
    const SpCol col = sp_col(c, S.Br_ptr, S.Br_idx, S.Br_val, k);
#pragma unroll (kUnr)
    for (int r = g; r < nrows; r += kGroups)
      RA[r * LA + k] = __dadd_rn(sp_dot(c, col, S.Br_idx, S.Br_val, RB + r * c.NUP, 0.0),
                                 ldcg(P.evec + (size_t)c.mt.edge(row0 + r) * c.NXP + k));
  }
  __syncthreads();
  TSMPC_MARK(P, 6, tm_);
  // (4) u = uhat + du (B; the psi epilogue below reads back only this thread's
  // entries: no barrier), then the x scan, head -> tail: x = a .* x_anc + (bv + e)
  if (TMS && TSMPC_TMLATE) tm_ld_u();
  if (k < nu) {
#pragma unroll
    for (int m = 0; m < kRW; ++m) {
      const int r = g + kGroups * m;
      if (r < nrows)
        RB[r * c.NUP + k] = __dadd_rn(RB[r * c.NUP + k],
                                      TSMPC_PREF ? upre[m] : ldcg(P.uhat + (size_t)c.mt.edge(row0 + r) * c.NUP + k));
    }
  }
  if (!S.split) epi_psi_wide<FGK && !TMS>(nu_it, cf, th, nrows, cur, rmax, pre, cfn);
  {
    const double* adiag = c.adiag();
    const double* pr = c.proot();
#pragma unroll 1
    for (int idx = tid; idx < nsegs * nx; idx += kThreadsS) {
      const int s = idx / nx, i = idx - s * nx;
      const int* sg = c.mt.segs + 4 * (seg0 + s);
      const int lo = sg[0], n = sg[1] - lo, pn = sg[2];
      double* col = RA + lo * LA + i;
      double x = pn >= 0 ? (S.split ? 0.0 : c.need[(size_t)pn * S.need_ld + c.NVP + i]) : pr[i];
      const double a = adiag[i];
#pragma unroll 1
      for (int j0 = 0; j0 < n; j0 += kCh) {
        double v[kCh];
#pragma unroll
        for (int u = 0; u < kCh; ++u) v[u] = j0 + u < n ? col[(j0 + u) * LA] : 0.0;
#pragma unroll
        for (int u = 0; u < kCh; ++u)
          if (j0 + u < n) {
            x = __dadd_rn(__dmul_rn(x, a), v[u]);
            col[(j0 + u) * LA] = x;
          }
      }
    }
  }
  __syncthreads();
  TSMPC_MARK(P, 7, tm_);
  if (S.split) return;  // trunk terms and epilogue: fwd_finish_wide
  // (5) epilogue, state blocks (warp per row)
  epi_state_wide<XS, FGK && !TMS>(nu_it, cf, th, nrows, cur, rmax, pre, cfn);
  __syncthreads();
  TSMPC_MARK(P, 8, tm_);
}

// split mode, after the chains' trunk parents are published (TR): the forward ran
// with zero trunk input, and S, du, bv, x are affine in the parent's values, so
//   u_e += du_tp,   x_e += G_d .* (B du_tp) + a^(d+1) .* x_tp   (d = depth below the head)
// (see fwd_finish), for every chain of the wide tile; then the prox / dual epilogue.
template <int XS>
__device__ __noinline__ void fwd_finish_wide(int ti, int nu_it, double cf, double th, int cur, double* rmax, bool pre,
                                             double cfn) {
  const SParams& S = g_sp;
  const Ctx c = ctx_of();
  const Params& P = S.P;
  (void)P;
  const int* td = c.mt.tiles + 4 * ti;
  const int nrows = td[1], seg0 = td[2], nsegs = td[3];
  const int tid = threadIdx.x;
  const int nx = c.nx, LA = c.LA;
  double* RA = c.A();
  long long tm_ = clock64();
  (void)tm_;
  // the parents' [du | B du | x] rows, staged once per chain
  double* tr = s_dyn + S.O_HSUM + S.hsum_nseg * c.NVP;
  const int HL = max(c.NXP + 2 * c.NUP, S.TR_LD);
  {
    constexpr int U = 4;  // loads in flight per thread (a 4-chain tile in one round)
    double v[U];
    int dst[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = tid + u * kThreadsS;
      const int s = idx / S.TR_LD, q = idx - s * S.TR_LD;
      const int pn = s < nsegs ? c.mt.segs[4 * (seg0 + s) + 2] : -1;
      dst[u] = pn >= 0 ? s * HL + q : -1;
      v[u] = pn >= 0 ? ldcg(S.TR + (size_t)pn * S.TR_LD + q) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (dst[u] >= 0) tr[dst[u]] = v[u];
#pragma unroll 1
    for (int idx = tid + U * kThreadsS; idx < nsegs * S.TR_LD; idx += kThreadsS) {
      const int s = idx / S.TR_LD, q = idx - s * S.TR_LD;
      const int pn = c.mt.segs[4 * (seg0 + s) + 2];
      if (pn >= 0) tr[s * HL + q] = ldcg(S.TR + (size_t)pn * S.TR_LD + q);
    }
  }
  __syncthreads();
  TSMPC_MARK(P, 13, tm_);
  if (!S.a_unit) {
    // general diagonal A: x_e += G_d .* (B du_tp) + a^(d+1) .* x_tp by the recursion over
    // each chain (A = I: folded into the state epilogue below)
    const double* adiag = c.adiag();
#pragma unroll 1
    for (int idx = tid; idx < nsegs * nx; idx += kThreadsS) {
      const int s = idx / nx, i = idx - s * nx;
      const int* sg = c.mt.segs + 4 * (seg0 + s);
      if (sg[2] < 0) continue;
      const int lo = sg[0], n = sg[1] - lo;
      const double bt = tr[s * HL + c.NUP + i], xt = tr[s * HL + c.NUP + c.NXP + i];
      const double a = adiag[i];
      double* col = RA + lo * LA + i;
      double gs = 1.0, pw = a;
#pragma unroll 4
      for (int j = 0; j < n; ++j) {
        col[j * LA] = __dadd_rn(col[j * LA], __dadd_rn(__dmul_rn(gs, bt), __dmul_rn(pw, xt)));
        gs = __dadd_rn(__dmul_rn(gs, a), 1.0);
        pw = __dmul_rn(pw, a);
      }
    }
    __syncthreads();
  }
  TSMPC_MARK(P, 14, tm_);
  // u += du_tp folded into the psi epilogue, x += (d+1) B du_tp + x_tp (A = I) into the state one
  const int tro = (int)(tr - s_dyn);
  epi_psi_wide<false>(nu_it, cf, th, nrows, cur, rmax, pre, cfn, tro, HL, seg0);
  TSMPC_MARK(P, 15, tm_);
  epi_state_wide<XS, false>(nu_it, cf, th, nrows, cur, rmax, pre, cfn, S.a_unit ? tro : -1, HL, seg0);
  __syncthreads();
  TSMPC_MARK(P, 8, tm_);
}

// epilogue of the CTA's own trunk rows (their dual / ergodic rows live in HBM;
// x and u are the need rows)
template <int XS>
__device__ __noinline__ void trunk_own_rows_wide(int nu_it, double cf, double th, int cur, double* rmax) {
  const SParams& S = g_sp;
  const Ctx c = ctx_of();
  const int no = c.mt.nown;
  if (no == 0) return;
  const int LD = S.need_ld;
  for (int b0 = 0; b0 < no; b0 += c.tcap) {
    const int nb = min(c.tcap, no - b0);
    for (int i = threadIdx.x; i < nb; i += kThreadsS) {
      const int n = c.mt.own[b0 + i];
      int* d = c.rdesc() + 5 * i;
      d[0] = c.mt.needs[4 * n + 2];
      d[1] = c.mt.needs[4 * n + 3];
      d[2] = (int)(c.need + (size_t)n * LD + c.NVP - s_dyn);
      d[3] = (int)(c.need + (size_t)n * LD + c.NVP + c.NXP - s_dyn);
      d[4] = 0;
    }
    __syncthreads();
    epi_psi_wide<false>(nu_it, cf, th, nb, cur, rmax, 0, 0.0);
    epi_state_wide<XS, false>(nu_it, cf, th, nb, cur, rmax, 0, 0.0);
    __syncthreads();
  }
}

}  // namespace

__global__ void __launch_bounds__(kThreadsS, 1) apg_sparse_kernel(LaunchWin win) {
  cg::grid_group grid = cg::this_grid();
  const SParams& S = g_sp;
  const Params& P = S.P;
  if (threadIdx.x == 0) {
    s_win = win;  // visible after the staging barrier below
    s_tm_on = 0;
  }
  {  // stage model vectors, scaling, sparse operators and this CTA's plan
    double* bnd = s_dyn + S.O_BND;
    double* scl = s_dyn + S.O_SCL;
    const int NXP = P.NXP, NUP = P.NUP, N = P.N;
#pragma unroll 1
    for (int i = threadIdx.x; i < NXP; i += kThreadsS) {
      bnd[i] = P.x_s[i];
      bnd[NXP + i] = P.x_min[i];
      bnd[2 * NXP + i] = P.x_max[i];
      bnd[3 * NXP + 2 * NUP + i] = P.a_diag[i];
      bnd[4 * NXP + 2 * NUP + i] = P.p[i];
    }
#pragma unroll 1
    for (int j = threadIdx.x; j < NUP; j += kThreadsS) {
      bnd[3 * NXP + j] = P.u_min[j];
      bnd[3 * NXP + NUP + j] = P.u_max[j];
    }
#pragma unroll 1
    for (int j = threadIdx.x; j < N; j += kThreadsS) {
      scl[j] = P.scaled ? P.sig_stage[j] : 1.0;
      scl[N + j] = P.scaled ? P.zeta_stage[j] : 1.0;
      scl[2 * N + j] = P.scaled ? P.sig_rcp[j] : 1.0;
      scl[3 * N + j] = P.scaled ? P.zeta_rcp[j] : 1.0;
    }
    if (P.scaled && S.psi_smem) {
      double* psi = s_dyn + S.O_PSI;
#pragma unroll 1
      for (int i = threadIdx.x; i < N * NUP; i += kThreadsS) psi[i] = P.psi_stage[i];
    }
    if (S.sched_resident) {
      int* ss = reinterpret_cast<int*>(s_dyn + S.O_SCHED);
#pragma unroll 1
      for (int i = threadIdx.x; i < S.n_tsched; i += kThreadsS) ss[i] = __ldg(S.tsched + i);
    }
    int* ints = reinterpret_cast<int*>(s_dyn + S.O_INT);
    const int m0 = __ldg(S.meta_ptr + blockIdx.x), m1 = __ldg(S.meta_ptr + blockIdx.x + 1);
#pragma unroll 1
    for (int i = threadIdx.x; i < m1 - m0; i += kThreadsS) ints[i] = __ldg(S.meta + m0 + i);
#pragma unroll 1
    for (int i = threadIdx.x; i < S.n_spi; i += kThreadsS) ints[S.meta_max + i] = __ldg(S.spi + i);
    double* spv = s_dyn + S.O_SPV;
#pragma unroll 1
    for (int i = threadIdx.x; i < S.n_spv; i += kThreadsS) spv[i] = __ldg(S.spv + i);
    __syncthreads();
  }
  const Ctx c = ctx_of();
  const bool resident = c.mt.resident != 0;
  const int nt = c.mt.ntiles;
  const bool trunk = P.n_trunk > 0;
  const bool do_a = win.phase & 1, do_b = win.phase & 2;
  {  // initial dual / ergodic rows
    const int cur0 = (P.slot0 + win.nu0) & 1, ysm0 = win.nu0 & 1;
    if (resident) {
      if (nt > 0) load_rows(c.mt.rows, 4, c.mt.nrows, c.slot, 3, cur0, ysm0);
    } else if (nt > 0) {
      // streamed: the first backward tile is the last one; a forward-only launch
      // (sharded phase 2) starts with tile 0 and its ergodic rows
      const int* td = c.mt.tiles + 4 * (do_a ? nt - 1 : 0);
      load_rows(c.mt.rows + 4 * td[0], 4, td[1], c.slot, do_a ? 1 : 3, cur0, ysm0);
    }
    cp_commit();
    cp_wait<0>();
    __syncthreads();
  }
  if (S.split && S.tops && (int)blockIdx.x >= S.split_c0) {
    double* tv = s_dyn + S.O_SLOT + S.O_TOPS;
    int* ti = reinterpret_cast<int*>(tv + S.n_tpv);
#pragma unroll 1
    for (int i = threadIdx.x; i < S.n_tpv; i += kThreadsS) tv[i] = __ldg(S.tpv + i);
#pragma unroll 1
    for (int i = threadIdx.x; i < S.n_tpi; i += kThreadsS) ti[i] = __ldg(S.tpi + i);
    __syncthreads();
  }
  if (S.split && S.split_heads && (int)blockIdx.x < S.split_c0 && nt == 1) {
    // sum of beta_s over the chain (static during the launch), chain order
    double* hb = s_dyn + S.O_HSUM;
    const int* sg = c.mt.segs + 4 * c.mt.tiles[2];
    const int lo = sg[0], n = sg[1] - lo;
#pragma unroll 1
    for (int k = threadIdx.x; k < c.nv; k += kThreadsS) {
      double b = 0.0;
#pragma unroll 1
      for (int d = 0; d < n; ++d) b = __dadd_rn(b, ldcg(S.beta_s + (size_t)c.mt.edge(c.mt.tiles[0] + lo + d) * c.NVP + k));
      hb[k] = b;
    }
    __syncthreads();
  }
  // static vectors of a resident one-tile CTA in TMEM for the launch
  if (TSMPC_TMSTATIC && nt == 1 && resident && do_a && do_b && !S.sharded &&
      (!S.split || (int)blockIdx.x < S.split_c0))
    tm_static_fill_res();
  double rmax = 0.0;
  unsigned int sub_target = 0;  // trunk-CTA barrier episodes x split_n (split mode)
  double cf = P.coef[win.nu0], th = P.theta[win.nu0];
  for (int nu = win.nu0; nu < win.nu1; ++nu) {
    const int cur = (P.slot0 + nu) & 1;
    const int ysm = nu & 1;
    if (P.tol > 0.0 && nu > win.nu0 && nu % P.check_every == 0) {
      // stopping test on the residual of iteration nu - 1 (its state is in HBM)
      grid.sync();
      const double r = __longlong_as_double(
          (long long)*((volatile unsigned long long*)(P.resid_chk + nu / P.check_every - 1)));
      if (r <= P.tol) {
        if (blockIdx.x == 0 && threadIdx.x == 0) *P.iters_done = nu;
        tm_release();
        return;
      }
    }
    // momentum coefficients of the next iteration, loaded one iteration ahead
    const int nn = nu + 1 < P.iters ? nu + 1 : nu;
    const double cf_n = P.coef[nn], th_n = P.theta[nn];
    if (do_a) {
      for (int t = nt - 1; t >= 0; --t)
        s_tm_on ? bwd_tile<true>(t, cf, ysm, resident ? c.mt.tiles[4 * t] : 0, resident, cur,
                                 S.split && S.split_heads && S.split_flags && nu > win.nu0)
                : bwd_tile<false>(t, cf, ysm, resident ? c.mt.tiles[4 * t] : 0, resident, cur,
                                  S.split && S.split_heads && S.split_flags && nu > win.nu0);
      if (S.sharded && trunk) {
        grid.sync();
        head_prereduce();
        if (S.cut && S.n_xch > 0) {  // the cut: this rank's sums that cross it -> XCH
          grid.sync();
          trunk_sweep(cf, cur, 5);
        }
      }
    }
    if (do_b && trunk && S.split && S.split_flags) {
      // split mode with directed signals instead of grid barriers: chain CTAs
      // publish their chain heads and run the zero-input forward at once; trunk
      // CTAs wait for every chain's heads, sweep, run the trunk forward and
      // publish TR; chain CTAs wait for TR only before their trunk terms.
      long long tb_ = clock64();
      (void)tb_;
      const unsigned it = (unsigned)(nu - win.nu0 + 1);
      if ((int)blockIdx.x < S.split_c0) {
        if (!S.split_heads) signal_arrive(S.sub_ctr + 1);  // else published inside bwd_tile
        for (int t = 0; t < nt; ++t)
          (s_tm_on ? fwd_tile<true>(t, nu, cf, th, ysm, resident ? c.mt.tiles[4 * t] : 0, resident, cur, &rmax)
                  : fwd_tile<false>(t, nu, cf, th, ysm, resident ? c.mt.tiles[4 * t] : 0, resident, cur, &rmax));
        TSMPC_MARK(P, 10, tb_);
        signal_wait(S.sub_ctr + 2, it * (unsigned)S.split_n);
        TSMPC_MARK(P, 9, tb_);
        if (blockIdx.x == 0) {
          const double om = __dsub_rn(1.0, th);
          for (int i = threadIdx.x; i < c.nx; i += kThreadsS)
            P.xavg[i] = __dadd_rn(__dmul_rn(P.xavg[i], om), __dmul_rn(th, c.proot()[i]));
        }
        for (int t = 0; t < nt; ++t) fwd_finish(t, nu, cf, th, ysm, resident, cur, &rmax);
        TSMPC_MARK(P, 3, tb_);
      } else {
        // the previous iteration's trunk-row epilogues (dual rows the sweep reads)
        if (nu > win.nu0) trunk_barrier(S.sub_ctr, (unsigned)S.split_n, sub_target);
        if (!S.split_local) trunk_sweep(cf, cur, 1);  // own terms, before the heads arrive
        signal_wait(S.sub_ctr + 1, it * (unsigned)S.split_c0);
        TSMPC_MARK(P, 9, tb_);
        if (S.split_local) {
          trunk_sweep_local(cf, cur);
          TSMPC_MARK(P, 10, tb_);
        } else {
          trunk_sweep(cf, cur, 2);
          TSMPC_MARK(P, 10, tb_);
          trunk_barrier(S.sub_ctr, (unsigned)S.split_n, sub_target);
          TSMPC_MARK(P, 11, tb_);
        }
        trunk_needs();
        signal_arrive(S.sub_ctr + 2);
        TSMPC_MARK(P, 12, tb_);
        trunk_own_rows(nu, cf, th, cur, &rmax);
        TSMPC_MARK(P, 3, tb_);
      }
    } else if (do_b) {
      [[maybe_unused]] long long tb_s = 0;  // phase timers only
      if (trunk && S.split) {
        // trunk CTAs: sweep, barrier among themselves, trunk forward (-> TR) and
        // trunk-row epilogues; chain CTAs meanwhile: forward with zero trunk input
        long long tb_ = clock64();
        (void)tb_;
        grid.sync();
        TSMPC_MARK(P, 9, tb_);
        if ((int)blockIdx.x >= S.split_c0) {
          if (S.split_local) {
            trunk_sweep_local(cf, cur);
            TSMPC_MARK(P, 10, tb_);
          } else {
            trunk_sweep(cf, cur, 3);
            TSMPC_MARK(P, 10, tb_);
            trunk_barrier(S.sub_ctr, (unsigned)S.split_n, sub_target);
            TSMPC_MARK(P, 11, tb_);
          }
          trunk_needs();
          TSMPC_MARK(P, 12, tb_);
        } else {
          for (int t = 0; t < nt; ++t)
            (s_tm_on ? fwd_tile<true>(t, nu, cf, th, ysm, resident ? c.mt.tiles[4 * t] : 0, resident, cur, &rmax)
                  : fwd_tile<false>(t, nu, cf, th, ysm, resident ? c.mt.tiles[4 * t] : 0, resident, cur, &rmax));
        }
        TSMPC_MARK(P, 10, tb_);
        grid.sync();
        TSMPC_MARK(P, 9, tb_);
        tb_s = tb_;
      } else if (trunk) {
        long long tb_ = clock64();
        (void)tb_;
        if (!S.sharded) grid.sync();
        TSMPC_MARK(P, 9, tb_);
        trunk_sweep(cf, cur, 3);
        TSMPC_MARK(P, 10, tb_);
        grid.sync();
        TSMPC_MARK(P, 9, tb_);
        trunk_needs();
        trunk_own_rows(nu, cf, th, cur, &rmax);
        TSMPC_MARK(P, 12, tb_);
      }
      if (blockIdx.x == 0) {
        const double om = __dsub_rn(1.0, th);
        for (int i = threadIdx.x; i < c.nx; i += kThreadsS)
          P.xavg[i] = __dadd_rn(__dmul_rn(P.xavg[i], om), __dmul_rn(th, c.proot()[i]));
      }
      if (trunk && S.split) {
        // trunk-row epilogues (trunk CTAs) overlap the chain CTAs' trunk terms + epilogue
        if ((int)blockIdx.x >= S.split_c0) trunk_own_rows(nu, cf, th, cur, &rmax);
        for (int t = 0; t < nt; ++t) fwd_finish(t, nu, cf, th, ysm, resident, cur, &rmax);
        TSMPC_MARK(P, 3, tb_s);
      } else {
        for (int t = 0; t < nt; ++t)
          (s_tm_on ? fwd_tile<true>(t, nu, cf, th, ysm, resident ? c.mt.tiles[4 * t] : 0, resident, cur, &rmax)
                  : fwd_tile<false>(t, nu, cf, th, ysm, resident ? c.mt.tiles[4 * t] : 0, resident, cur, &rmax));
      }
    }
    if (do_b) {
      if (nu == P.iters - 1 || P.record_all || is_check(P, nu)) {
        // warp, then CTA, then one global atomic per CTA (same-address global
        // atomics from every warp serialise in L2)
        __shared__ double s_rmax[kThreadsS / 32];
        for (int off = 16; off > 0; off >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, off));
        if ((threadIdx.x & 31) == 0) s_rmax[threadIdx.x >> 5] = rmax;
        __syncthreads();
        if (threadIdx.x == 0) {
          double m = 0.0;
          for (int w = 0; w < kThreadsS / 32; ++w) m = fmax(m, s_rmax[w]);
          if (m > 0.0) {
            const unsigned long long b = (unsigned long long)__double_as_longlong(m);
            if (nu == P.iters - 1 || P.record_all) atomicMax(P.resid + (P.record_all ? nu : 0), b);
            if (is_check(P, nu)) atomicMax(P.resid_chk + nu / P.check_every, b);
          }
        }
        rmax = 0.0;
      }
    }
    cf = cf_n;
    th = th_n;
  }
  tm_release();
  if (P.tol > 0.0 && blockIdx.x == 0 && threadIdx.x == 0) *P.iters_done = win.nu1;
}


// Wide-mode persistent kernel (SParams::wide): per iteration, backward over the
// CTA's tiles (last first) -> grid barrier -> trunk sweep -> grid barrier ->
// needs, own trunk rows, forward + epilogue over the tiles.  The last forward
// tile's epilogue leaves the next iteration's fill of that tile (its first
// backward tile).  Sharded plans run it as two launches per iteration (phase 1:
// backward + head pre-reduction; phase 2: the rest), state in HBM in between.
// TMEM for the static vectors: 512 columns (all of it; one CTA per SM), allocated
// by warp 0 and filled by every thread in its prefetch layout (see kTmB)
__device__ __noinline__ void tm_static_fill() {
  tm_alloc_all();
  const SParams& S = g_sp;
  const Ctx c = ctx_of();
  const Params& P = S.P;
  const int row0 = c.mt.tiles[0], nrows = c.mt.tiles[1];
  const int k = threadIdx.x & (kKW - 1), g = threadIdx.x / kKW;
  const int k8 = threadIdx.x & 63, g8 = threadIdx.x >> 6;
#pragma unroll 1
  for (int m = 0; m < kRW; ++m) {
    const int r = g + kGroups * m;
    const size_t e = r < nrows ? (size_t)c.mt.edge(row0 + r) : 0;
    tm_st1(tm_addr(kTmB + 2 * m), r < nrows && k < c.nv ? ldcg(S.beta_s + e * c.NVP + k) : 0.0);
    tm_st1(tm_addr(kTmU + 2 * m), r < nrows && k < c.nu ? ldcg(P.uhat + e * c.NUP + k) : 0.0);
  }
#pragma unroll 1
  for (int m = 0; m < (kRX + 7) / 8 * 8; ++m) {
    const int r = g8 + kG8 * m;
    const bool ok = m < kRX && c.nx <= 64 && r < nrows && k8 < c.nx;
    tm_st1(tm_addr(kTmE + 2 * m), ok ? ldcg(P.evec + (size_t)c.mt.edge(row0 + r) * c.NXP + k8) : 0.0);
  }
  tm_fill_done();
}

// The cut exchange of a shard plan inside the persistent kernel (SParams::peer_rx,
// LaunchWin.phase & 4; replaces phase 1 -> ncclAllReduce(XCH, sum) -> phase 2).
// Called by every CTA after a grid barrier that completed XCH; the caller runs a
// grid barrier after it before XCH is read.  Every CTA owns the same slice of XCH
// in both halves: it stores its slice into every rank's RX (over NVLink for the
// peers), fences at system scope and bumps every rank's arrival counter once; it
// then waits for world x CTAs arrivals of this generation on its own counter and
// sums the world sender rows of its slice in rank order.  Each entry has one
// non-zero contributor (the owning rank), so the sum is exact, as the all-reduce.
// RX is double-buffered by generation parity: a rank writes generation g + 2 only
// after its own wait of generation g + 1, which every rank passes only after it
// has summed generation g.
__device__ __noinline__ void peer_exchange(unsigned long long gen) {
  const SParams& S = g_sp;
  const size_t xn = (size_t)S.n_xch * S.XCH_LD;
  const int w = S.world;
  const size_t slot = (size_t)(gen & 1ull) * (size_t)w * xn;
  const size_t i0 = (size_t)blockIdx.x * kThreadsS + threadIdx.x, step = (size_t)gridDim.x * kThreadsS;
#pragma unroll 1
  for (size_t i = i0; i < xn; i += step) {
    const double v = ldcg(S.XCH + i);
#pragma unroll 1
    for (int p = 0; p < w; ++p) __stcg(S.peer_rx[p] + slot + (size_t)S.rank * xn + i, v);
  }
  __threadfence_system();
  __syncthreads();
  if ((int)threadIdx.x < w) atomicAdd_system(S.peer_cnt[threadIdx.x], 1ull);
  if (threadIdx.x == 0) {
    spin_until64(S.RXCNT, (gen + 1ull) * S.xch_expect);
    __threadfence_system();
  }
  __syncthreads();
#pragma unroll 1
  for (size_t i = i0; i < xn; i += step) {
    double s = 0.0;
#pragma unroll 1
    for (int p = 0; p < w; ++p) s = __dadd_rn(s, ldcg(S.RX + slot + (size_t)p * xn + i));
    stcg(S.XCH + i, s);
  }
}

// meta windows (SParams::rows_window): copy tile t's rows and chain segments from the
// plan's meta in global memory into the window; ctx_of() rebinds to it
__device__ __noinline__ void win_stage(int t) {
  const SParams& S = g_sp;
  int* ints = reinterpret_cast<int*>(s_dyn + S.O_INT);
  const int* gm = S.meta + __ldg(S.meta_ptr + blockIdx.x);
  const int ntl = ints[0], nrw = ints[1];
  const int row0 = ints[8 + 4 * t], nr = ints[8 + 4 * t + 1], seg0 = ints[8 + 4 * t + 2], ns = ints[8 + 4 * t + 3];
  __syncthreads();  // the previous tile's readers are done with the window
  int* w = ints + S.O_WIN;
  const int* grows = gm + 8 + 4 * ntl + 4 * row0;
  const int* gsegs = gm + 8 + 4 * ntl + 4 * nrw + 4 * seg0;
#pragma unroll 1
  for (int i = threadIdx.x; i < 4 * nr; i += kThreadsS) w[i] = __ldg(grows + i);
#pragma unroll 1
  for (int i = threadIdx.x; i < 4 * ns; i += kThreadsS) w[4 * S.tile_cap + i] = __ldg(gsegs + i);
  if (threadIdx.x == 0) {
    s_row_off = row0;
    s_seg_off = seg0;
  }
  __syncthreads();
}

// block-wide copy of n elements global -> shared, four loads in flight per thread
template <class T>
__device__ __forceinline__ void stage_copy(T* dst, const T* __restrict__ src, int n) {
  int i = threadIdx.x;
#pragma unroll 1
  for (; i + 3 * kThreadsS < n; i += 4 * kThreadsS) {
    const T a = __ldg(src + i), b = __ldg(src + i + kThreadsS), c = __ldg(src + i + 2 * kThreadsS),
            d = __ldg(src + i + 3 * kThreadsS);
    dst[i] = a;
    dst[i + kThreadsS] = b;
    dst[i + 2 * kThreadsS] = c;
    dst[i + 3 * kThreadsS] = d;
  }
#pragma unroll 1
  for (; i < n; i += kThreadsS) dst[i] = __ldg(src + i);
}

template <int XS, bool FGK>
__global__ void __launch_bounds__(kThreadsS, 1) apg_wide_kernel(LaunchWin win) {
  cg::grid_group grid = cg::this_grid();
  const SParams& S = g_sp;
  const Params& P = S.P;
  if (threadIdx.x == 0) {
    s_win = win;  // visible after the staging barrier below
    s_tm_on = 0;
    if (FGK && TSMPC_BULK) {
      mbar_init(&s_bulk_bar, 1);
      s_bulk_phase = 0;
    }
  }
  {  // stage model vectors, scaling, sparse operators and this CTA's plan
    double* bnd = s_dyn + S.O_BND;
    double* scl = s_dyn + S.O_SCL;
    const int NXP = P.NXP, NUP = P.NUP, N = P.N;
#pragma unroll 1
    for (int i = threadIdx.x; i < NXP; i += kThreadsS) {
      bnd[i] = P.x_s[i];
      bnd[NXP + i] = P.x_min[i];
      bnd[2 * NXP + i] = P.x_max[i];
      bnd[3 * NXP + 2 * NUP + i] = P.a_diag[i];
      bnd[4 * NXP + 2 * NUP + i] = P.p[i];
    }
#pragma unroll 1
    for (int j = threadIdx.x; j < NUP; j += kThreadsS) {
      bnd[3 * NXP + j] = P.u_min[j];
      bnd[3 * NXP + NUP + j] = P.u_max[j];
    }
#pragma unroll 1
    for (int j = threadIdx.x; j < N; j += kThreadsS) {
      scl[j] = P.scaled ? P.sig_stage[j] : 1.0;
      scl[N + j] = P.scaled ? P.zeta_stage[j] : 1.0;
      scl[2 * N + j] = P.scaled ? P.sig_rcp[j] : 1.0;
      scl[3 * N + j] = P.scaled ? P.zeta_rcp[j] : 1.0;
    }
    // the contiguous blocks: four loads in flight per thread (a launch of a shard
    // plan restages them twice per iteration)
    if (P.scaled && S.psi_smem) stage_copy(s_dyn + S.O_PSI, P.psi_stage, N * NUP);
    if (S.sched_resident) stage_copy(reinterpret_cast<int*>(s_dyn + S.O_SCHED), S.tsched, S.n_tsched);
    int* ints = reinterpret_cast<int*>(s_dyn + S.O_INT);
    const int m0 = __ldg(S.meta_ptr + blockIdx.x), m1 = __ldg(S.meta_ptr + blockIdx.x + 1);
    if (S.rows_window) {  // everything but the rows and segments (staged per tile)
      const int lo = 8 + 4 * __ldg(S.meta + m0), gap = 4 * (__ldg(S.meta + m0 + 1) + __ldg(S.meta + m0 + 2));
      stage_copy(ints, S.meta + m0, lo);
      stage_copy(ints + lo, S.meta + m0 + lo + gap, m1 - m0 - gap - lo);
      if (threadIdx.x == 0) s_row_off = s_seg_off = 0;
    } else {
      stage_copy(ints, S.meta + m0, m1 - m0);
    }
    stage_copy(ints + S.meta_max, S.spi, S.n_spi);
    stage_copy(s_dyn + S.O_SPV, S.spv, S.n_spv);
    __syncthreads();
  }
  const Ctx c = ctx_of();
  const int nt = c.mt.ntiles;
  const bool trunk = P.n_trunk > 0;
  const bool do_a = win.phase & 1, do_b = win.phase & 2;
  // shard plan running both phases per iteration in this launch (the cut exchange in
  // between over peer memory; without peer tables: a compute-only timing trial)
  const bool fused = FGK && S.sharded && (win.phase & 4);
  const bool chain_cta = (int)blockIdx.x < S.split_c0;
  if (S.split && chain_cta && nt == 1) {
    // per chain, the sum of beta_s over its rows (static during the launch), chain order
    double* hb = s_dyn + S.O_HSUM;
    const int nsg = c.mt.tiles[3], sg0 = c.mt.tiles[2], row0 = c.mt.tiles[0];
#pragma unroll 1
    for (int idx = threadIdx.x; idx < nsg * c.nv; idx += kThreadsS) {
      const int s = idx / c.nv, k = idx - s * c.nv;
      const int* sg = c.mt.segs + 4 * (sg0 + s);
      double b = 0.0;
#pragma unroll 1
      for (int d = sg[0]; d < sg[1]; ++d) b = __dadd_rn(b, ldcg(S.beta_s + (size_t)c.mt.edge(row0 + d) * c.NVP + k));
      hb[s * c.NVP + k] = b;
    }
    __syncthreads();
  }
  if (S.split && S.tops && !chain_cta) {  // trunk CTAs: the combined forward operators
    double* tv = s_dyn + S.O_SLOT + S.O_TOPS;
    int* ti = reinterpret_cast<int*>(tv + S.n_tpv);
#pragma unroll 1
    for (int i = threadIdx.x; i < S.n_tpv; i += kThreadsS) tv[i] = __ldg(S.tpv + i);
#pragma unroll 1
    for (int i = threadIdx.x; i < S.n_tpi; i += kThreadsS) ti[i] = __ldg(S.tpi + i);
    __syncthreads();
  }
  // static vectors of a single-tile CTA resident in TMEM for the launch
  if (TSMPC_TMSTATIC && nt == 1 && do_a && do_b && (!S.sharded || fused) && (!S.split || chain_cta))
    tm_static_fill();
  double rmax = 0.0;
  unsigned int sub_target = 0;  // trunk-CTA barrier episodes x split_n (split mode)
  double cf = P.coef[win.nu0], th = P.theta[win.nu0];
  // FG fill rows: the buffer exists, 16-byte copies line up with the work regions,
  // and the CTA runs the forward of fwd_wide<XS, false> (split-mode and TMEM CTAs
  // keep every fill in shared memory or take it from the dual rows)
  const bool fg_ok = FGK && S.FG != nullptr && !S.split && !s_tm_on &&
                     (((int)(c.A() - s_dyn) | (int)(c.B() - s_dyn) | c.LA | c.NXP | c.NUP | S.FL) & 1) == 0;
  for (int nu = win.nu0; nu < win.nu1; ++nu) {
    const int cur = (P.slot0 + nu) & 1;
    const bool trace = nu == (win.nu0 + win.nu1) / 2;  // timeline stamps (timer builds)
    (void)trace;
#ifdef TSMPC_TIMERS
    if (threadIdx.x == 0) s_trace_on = trace;  // read after the phases' barriers
#endif
    TSMPC_STAMP(P, 0, trace);
    if (P.tol > 0.0 && !S.sharded && nu > win.nu0 && nu % P.check_every == 0) {
      // stopping test on the residual of iteration nu - 1 (its state is in HBM)
      grid.sync();
      const double r = __longlong_as_double(
          (long long)*((volatile unsigned long long*)(P.resid_chk + nu / P.check_every - 1)));
      if (r <= P.tol) {
        if (blockIdx.x == 0 && threadIdx.x == 0) *P.iters_done = nu;
        tm_release();
        return;
      }
    }
    const int nn = nu + 1 < P.iters ? nu + 1 : nu;
    const double cf_n = P.coef[nn], th_n = P.theta[nn];
    // where tile t's epilogue leaves the next iteration's fill: shared memory when
    // this launch runs the next backward and t is the tile it starts with, else FG
    auto pre_of = [&](int t) -> int {
      if (S.wide_prefill && t == nt - 1 && nu + 1 < win.nu1 && do_a) return 1;
      return fg_ok && nu + 1 < P.iters ? 2 : 0;
    };
    if (do_a) {
      for (int t = nt - 1; t >= 0; --t) {
        // fill source: 1 left in shared memory by this launch's previous iteration,
        // 2 left in FG by the previous iteration, 0 the dual rows
        const int pf = S.wide_prefill && t == nt - 1 && nu > win.nu0 ? 1 : (fg_ok && nu > 0 ? 2 : 0);
        if (FGK && S.rows_window) win_stage(t);
        s_tm_on ? bwd_wide<true, FGK>(t, cf, cur, pf) : bwd_wide<false, FGK>(t, cf, cur, pf);
      }
      TSMPC_STAMP(P, 1, trace);
      if (S.sharded && trunk) {
        grid.sync();
        head_prereduce();
        if (S.cut && S.n_xch > 0) {  // the cut: this rank's sums that cross it -> XCH
          grid.sync();
          trunk_sweep(cf, cur, 5);
        }
      }
    }
    if (fused && trunk) {  // shard plan, both phases in this launch: the cut exchange in between
      grid.sync();
      if (S.n_xch > 0 && S.peer_rx != nullptr) {
        peer_exchange(win.xgen + (unsigned long long)(nu - win.nu0));
        grid.sync();
      }
    }
    if (do_b && trunk && S.split) {
      // wide split mode, directed signals: chain CTAs published their heads in the
      // backward and run the zero-input forward at once; trunk CTAs wait for every
      // chain's heads, sweep, run the trunk forward and publish TR; chain CTAs wait
      // for TR only before their trunk terms
      long long tb_ = clock64();
      (void)tb_;
      const unsigned it = (unsigned)(nu - win.nu0 + 1);
      if (chain_cta) {
        for (int t = 0; t < nt; ++t)
          s_tm_on ? fwd_wide<XS, true, FGK>(t, nu, cf, th, cur, &rmax, 0, 0.0)
                  : fwd_wide<XS, false, FGK>(t, nu, cf, th, cur, &rmax, 0, 0.0);
        TSMPC_MARK(P, 10, tb_);
        TSMPC_STAMP(P, 2, trace);
        signal_wait(S.sub_ctr + 2, it * (unsigned)S.split_n);
        TSMPC_STAMP(P, 3, trace);
        TSMPC_MARK(P, 9, tb_);
        if (blockIdx.x == 0) {
          const double om = __dsub_rn(1.0, th);
          for (int i = threadIdx.x; i < c.nx; i += kThreadsS)
            P.xavg[i] = __dadd_rn(__dmul_rn(P.xavg[i], om), __dmul_rn(th, c.proot()[i]));
        }
        for (int t = 0; t < nt; ++t)
          fwd_finish_wide<XS>(t, nu, cf, th, cur, &rmax, S.wide_prefill && t == nt - 1 && nu + 1 < win.nu1, cf_n);
        TSMPC_STAMP(P, 4, trace);
        TSMPC_MARK(P, 3, tb_);
      } else {
        // the previous iteration's trunk-row epilogues (dual rows the sweep reads)
        if (nu > win.nu0) trunk_barrier(S.sub_ctr, (unsigned)S.split_n, sub_target);
        trunk_sweep(cf, cur, 1);  // own terms, before the heads arrive
        TSMPC_STAMP(P, 1, trace);
        signal_wait(S.sub_ctr + 1, it * (unsigned)S.split_c0);
        TSMPC_STAMP(P, 2, trace);
        TSMPC_MARK(P, 9, tb_);
        trunk_sweep(cf, cur, 2);
        TSMPC_STAMP(P, 3, trace);
        TSMPC_MARK(P, 10, tb_);
        trunk_barrier(S.sub_ctr, (unsigned)S.split_n, sub_target);
        TSMPC_STAMP(P, 4, trace);
        TSMPC_MARK(P, 11, tb_);
        trunk_needs();
        signal_arrive(S.sub_ctr + 2);
        TSMPC_STAMP(P, 5, trace);
        TSMPC_MARK(P, 12, tb_);
        trunk_own_rows_wide<XS>(nu, cf, th, cur, &rmax);
        TSMPC_STAMP(P, 6, trace);
        TSMPC_MARK(P, 3, tb_);
      }
    } else if (do_b) {
      if (trunk) {
        long long tb_ = clock64();
        (void)tb_;
        if (!S.sharded) grid.sync();
        TSMPC_MARK(P, 9, tb_);
        trunk_sweep(cf, cur, 3);
        TSMPC_MARK(P, 10, tb_);
        grid.sync();
        TSMPC_MARK(P, 9, tb_);
        trunk_needs();
        trunk_own_rows_wide<XS>(nu, cf, th, cur, &rmax);
        TSMPC_MARK(P, 12, tb_);
      }
      if (blockIdx.x == 0) {
        const double om = __dsub_rn(1.0, th);
        for (int i = threadIdx.x; i < c.nx; i += kThreadsS)
          P.xavg[i] = __dadd_rn(__dmul_rn(P.xavg[i], om), __dmul_rn(th, c.proot()[i]));
      }
      for (int t = 0; t < nt; ++t) {
        if (FGK && S.rows_window) win_stage(t);
        s_tm_on ? fwd_wide<XS, true, FGK>(t, nu, cf, th, cur, &rmax, pre_of(t), cf_n)
                : fwd_wide<XS, false, FGK>(t, nu, cf, th, cur, &rmax, pre_of(t), cf_n);
      }
    }
    if (do_b) {
      if (nu == P.iters - 1 || P.record_all || is_check(P, nu)) {
        __shared__ double s_rmax[kThreadsS / 32];
        for (int off = 16; off > 0; off >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, off));
        if ((threadIdx.x & 31) == 0) s_rmax[threadIdx.x >> 5] = rmax;
        __syncthreads();
        if (threadIdx.x == 0) {
          double m = 0.0;
          for (int w = 0; w < kThreadsS / 32; ++w) m = fmax(m, s_rmax[w]);
          if (m > 0.0) {
            const unsigned long long b = (unsigned long long)__double_as_longlong(m);
            if (nu == P.iters - 1 || P.record_all) atomicMax(P.resid + (P.record_all ? nu : 0), b);
            if (is_check(P, nu)) atomicMax(P.resid_chk + nu / P.check_every, b);
          }
        }
        rmax = 0.0;
      }
    }
    cf = cf_n;
    th = th_n;
  }
  tm_release();
  if (P.tol > 0.0 && blockIdx.x == 0 && threadIdx.x == 0) *P.iters_done = win.nu1;
}

}  // namespace tsmpc

namespace tsmpc {

// the persistent kernel a plan runs: split / streamed / resident modes share
// apg_sparse_kernel; wide plans run apg_wide_kernel<XS> (XS = state components per
// lane of the warp-per-row state epilogue: n_x <= 64 -> 2, <= 128 -> 4)
const void* sparse_kernel_fn(int wide, int nx, bool fg) {
  if (!wide) return (const void*)apg_sparse_kernel;
  if (fg) return nx <= 64 ? (const void*)apg_wide_kernel<2, true> : (const void*)apg_wide_kernel<4, true>;
  return nx <= 64 ? (const void*)apg_wide_kernel<2, false> : (const void*)apg_wide_kernel<4, false>;
}

// g_sp is one per device and shared by every plan of the process: launches from
// different streams are chained through a per-device event so that a launch's
// parameter upload cannot land while another plan's kernel still reads g_sp
// (the kernel occupies the whole GPU anyway, so nothing is lost).
namespace {
struct DevParams {  // what g_sp holds on a device, and the last launch that reads it
  std::mutex mu;
  bool valid = false;
  SParams cur{};
  cudaEvent_t last = nullptr;
  cudaStream_t last_stream = nullptr;
};
DevParams g_dev[64];
}  // namespace

// Upload S into g_sp unless it already holds exactly these bytes.  An upload
// waits for the last launch (on another stream) that may still read g_sp.
cudaError_t sparse_params_upload(const SParams& S, cudaStream_t stream) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  DevParams& d = g_dev[dev];
  std::lock_guard<std::mutex> lock(d.mu);
  if (!d.last) {
    e = cudaEventCreateWithFlags(&d.last, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  if (d.valid && std::memcmp(&d.cur, &S, sizeof(SParams)) == 0) return cudaSuccess;
  if (d.last_stream && d.last_stream != stream) {
    e = cudaStreamWaitEvent(stream, d.last, 0);
    if (e != cudaSuccess) return e;
  }
  d.cur = S;  // stable host copy: the async copy reads it
  d.valid = true;
  return cudaMemcpyToSymbolAsync(g_sp, &d.cur, sizeof(SParams), 0, cudaMemcpyHostToDevice, stream);
}

// Bookkeeping after launches that did not go through sparse_launch (a graph
// replay): later uploads from other streams wait for them.
cudaError_t sparse_note_launch(cudaStream_t stream) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  DevParams& d = g_dev[dev];
  std::lock_guard<std::mutex> lock(d.mu);
  if (!d.last) {
    e = cudaEventCreateWithFlags(&d.last, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  d.last_stream = stream;
  return cudaEventRecord(d.last, stream);
}

// One cooperative launch of the plan's persistent kernel over the window `w`.
cudaError_t sparse_launch(const SParams& S, LaunchWin w, int ctas, size_t smem, cudaStream_t stream) {
  cudaError_t e = sparse_params_upload(S, stream);
  if (e != cudaSuccess) return e;
  void* args[] = {&w};
  e = cudaLaunchCooperativeKernel(sparse_kernel_fn(S.wide, S.P.nx, S.FL > 0), dim3(ctas), dim3(kThreadsS), args, smem, stream);
  if (e != cudaSuccess) return e;
  int dev = 0;
  cudaGetDevice(&dev);
  DevParams& d = g_dev[dev];
  std::lock_guard<std::mutex> lock(d.mu);
  d.last_stream = stream;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream, &cs);
  if (cs != cudaStreamCaptureStatusNone) return cudaSuccess;  // graph capture: no event record
  return cudaEventRecord(d.last, stream);
}

// beta_s = beta M (rows of the stage cache mapped to the structured basis,
// elimination.py:156-157 with L replaced by Ls = L M).  A thread per (edge, column
// k); M by column without its zeros (mc = [ptr | rows], mv values, rows ascending:
// the dense product's order, skipped terms are fma(b, 0, s) = s).
__global__ void beta_rotate_kernel(const double* __restrict__ beta, const int* __restrict__ mc,
                                   const double* __restrict__ mv, double* out, int E, int nv, int NVP) {
  const int* rows = mc + nv + 1;
  const long long total = (long long)E * nv;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(i / nv), k = (int)(i - (long long)e * nv);
    const double* b = beta + (size_t)e * NVP;
    double s = 0.0;
    for (int q = mc[k]; q < mc[k + 1]; ++q) s = fma(b[rows[q]], mv[q], s);
    out[(size_t)e * NVP + k] = s;
  }
}

}  // namespace tsmpc