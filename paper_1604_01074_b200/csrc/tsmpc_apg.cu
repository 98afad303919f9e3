// tsmpc_apg.cu — persistent cooperative APG kernel for sm_100a.
// See tsmpc_kernels.cuh for the algorithm outline and DESIGN.md for the
// derivation, data layout and roofline.
//
// Shared memory is one dynamic array (g_smem) addressed by per-phase offsets so
// that every tile access compiles to LDS/STS (a generic pointer passed across a
// call would turn them into generic loads).  A tile of <= kTileM edge rows uses
//   backward: A = [xiq | psi^] (LDA1 = 180 cols), C = h (LDB1 = 104 cols)
//   forward:  A = S then x     (LDA2 = 100 cols), C = [u | bv + e] (LDB2 = 184)
// i.e. 284 doubles per row in both sweeps.  Every global read of a phase is
// issued up front (one warp per edge row), per-row bias terms are folded into
// the GEMM epilogues and the sequential stage scans touch shared memory only.
#include "tsmpc_kernels.cuh"

namespace cg = cooperative_groups;

namespace tsmpc {

extern __shared__ __align__(16) double g_smem[];

constexpr int kChunks = 4;  // n_x, n_u <= 128: a row is at most 4 x 32 lanes

__device__ __forceinline__ void dmma8x8x4(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// Tile metadata ints after the double region: edge[kTileM], lo[kTileM], hi[kTileM], misc[4]
__device__ __forceinline__ int* meta_base(const Params& P) {
  return reinterpret_cast<int*>(g_smem + P.META_OFF);
}
#define SM_EDGE(P) (meta_base(P))
#define SM_LO(P) (meta_base(P) + kTileM)
#define SM_HI(P) (meta_base(P) + 2 * kTileM)
#define SM_MISC(P) (meta_base(P) + 3 * kTileM)
// per-row 1/(2 p_e) of the current tile (doubles after the metadata ints)
#define SM_INV2P(P) (g_smem + (P).META_OFF + 160)
// model bound vectors, staged once per launch: x_s, x_min, x_max (NXP each), u_min, u_max (NUP)
#define SM_BOUNDS(P) (g_smem + (P).META_OFF + 160 + kTileM)

// Explicit global-space accesses: the state pointers reach the device code through
// kernel parameters, so plain dereferences would compile to generic LD/ST.  The .cg
// variants cache in L2 only, which keeps them coherent with the other CTAs' writes
// (every cross-CTA dependency of the kernel crosses a grid barrier).
__device__ __forceinline__ double gld(const double* p) { return __ldcg(p); }
__device__ __forceinline__ void gst(double* p, double v) { __stcg(p, v); }

// C[rows, nt*8 .. nt*8+7] = A[rows, 0:4*KS] * B + C for every n-tile owned by
// this warp (C holds the per-row bias, staged by the caller's load phase; rows
// >= nrows are overwritten, not accumulated).  A = g_smem[a_off ...] row-major
// with lda = 4 mod 16 (conflict-free fragment loads), B in global memory in
// fragment order [NT][KS][32] (one coalesced 256-byte load per warp and k-step),
// register-prefetched 8 k-steps ahead and reused across the MT m-tiles.
template <int MT>
__device__ __forceinline__ void gemm_tile(const Params& P, int a_off, int lda, int KS, int NT,
                                          const double* __restrict__ Bf, int c_off, int ldc,
                                          int nrows) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ar = lane >> 2, ac = lane & 3;
  const double* As = g_smem + a_off + ar * lda + ac;
  for (int nt = warp; nt < NT; nt += kWarps) {
    double acc[MT][2];
#pragma unroll
    for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = 0.0;
    const double* bp = Bf + (size_t)nt * KS * 32 + lane;
    constexpr int R = MT <= 6 ? 16 : 12;  // B-fragment ring depth (k-steps in flight)
    double bq[R];
#pragma unroll
    for (int q = 0; q < R; ++q) bq[q] = (q < KS) ? __ldg(bp + q * 32) : 0.0;
    for (int ks0 = 0; ks0 < KS; ks0 += R) {
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int ks = ks0 + q;
        if (ks < KS) {
          // all A fragments of the k-step in distinct registers, then the DMMAs read
          // the ring slot directly; the slot is refilled (R k-steps ahead) only after
          // its last use, so no move ever waits on an in-flight load
          double af[MT];
#pragma unroll
          for (int m = 0; m < MT; ++m) af[m] = As[m * 8 * lda + ks * 4];
#pragma unroll
          for (int m = 0; m < MT; ++m) dmma8x8x4(acc[m], af[m], bq[q]);
          if (ks + R < KS) bq[q] = __ldg(bp + (ks + R) * 32);
        }
      }
    }
    const int c0 = nt * 8 + 2 * ac;
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const int r = m * 8 + ar;
      double* cp = g_smem + c_off + r * ldc + c0;
      if (r < nrows) {
        cp[0] = __dadd_rn(acc[m][0], cp[0]);
        cp[1] = __dadd_rn(acc[m][1], cp[1]);
      } else {
        cp[0] = acc[m][0];
        cp[1] = acc[m][1];
      }
    }
  }
}

__device__ __noinline__ void gemm_dispatch(const Params& P, int mt, int a_off, int lda, int KS, int NT,
                                           const double* Bf, int c_off, int ldc, int nrows) {
  switch (mt) {
    case 1: gemm_tile<1>(P, a_off, lda, KS, NT, Bf, c_off, ldc, nrows); break;
    case 2: gemm_tile<2>(P, a_off, lda, KS, NT, Bf, c_off, ldc, nrows); break;
    case 3: gemm_tile<3>(P, a_off, lda, KS, NT, Bf, c_off, ldc, nrows); break;
    case 4: gemm_tile<4>(P, a_off, lda, KS, NT, Bf, c_off, ldc, nrows); break;
    case 5: gemm_tile<5>(P, a_off, lda, KS, NT, Bf, c_off, ldc, nrows); break;
    case 6: gemm_tile<6>(P, a_off, lda, KS, NT, Bf, c_off, ldc, nrows); break;
    case 7: gemm_tile<7>(P, a_off, lda, KS, NT, Bf, c_off, ldc, nrows); break;
    case 8: gemm_tile<8>(P, a_off, lda, KS, NT, Bf, c_off, ldc, nrows); break;
    case 9: gemm_tile<9>(P, a_off, lda, KS, NT, Bf, c_off, ldc, nrows); break;
    case 10: gemm_tile<10>(P, a_off, lda, KS, NT, Bf, c_off, ldc, nrows); break;
    case 11: gemm_tile<11>(P, a_off, lda, KS, NT, Bf, c_off, ldc, nrows); break;
    default: gemm_tile<12>(P, a_off, lda, KS, NT, Bf, c_off, ldc, nrows); break;
  }
}

__device__ __forceinline__ void load_tile(const Params& P, int tile, int& nrows, int& nsegs) {
  const int sg0 = P.tile_seg[tile], sg1 = P.tile_seg[tile + 1];
  const int rbase = P.seg_row[sg0];
  nrows = P.seg_row[sg1] - rbase;
  nsegs = sg1 - sg0;
  int* edge = SM_EDGE(P);
  int* lo = SM_LO(P);
  int* hi = SM_HI(P);
  int* misc = SM_MISC(P);
  __syncthreads();  // the previous tile is done with shared memory
  double* inv2p = SM_INV2P(P);
  for (int i = threadIdx.x; i < nrows; i += kThreads) {
    const int e = P.row_edge[rbase + i];
    edge[i] = e;
    inv2p[i] = P.inv2p[e];
  }
  if (threadIdx.x == 0) misc[0] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < nsegs; i += kThreads) {
    const int l = P.seg_row[sg0 + i] - rbase, h = P.seg_row[sg0 + i + 1] - rbase;
    lo[i] = l;
    hi[i] = h;
    atomicMax(misc, h - l);
  }
  __syncthreads();
}

__device__ __forceinline__ double stage_scale(const double* s, int st, int scaled) {
  return scaled ? s[st] : 1.0;
}

// Extrapolated dual w = y + c (y - y_prev), evaluated in the reference's
// rounding order (engine.py:195-201): no FMA contraction.
__device__ __forceinline__ double extrap(double y, double yp, double c) {
  return __dadd_rn(y, __dmul_rn(c, __dsub_rn(y, yp)));
}

// sum_{c in children(node)} buf[c-1][i] for the edges below `node`
__device__ __forceinline__ double child_sum(const Params& P, const double* buf, int ld, int node, int i) {
  const int c0 = P.child_start[node] - 1, c1 = P.child_stop[node] - 1;
  double acc = 0.0;
  for (int ch = c0; ch < c1; ++ch) acc = __dadd_rn(acc, buf[(size_t)ch * ld + i]);
  return acc;
}

// S of the parent edge of a segment head: the trunk GEMM output (collapsed mode)
// or the parent segment's tail S left in T (level mode).
__device__ __forceinline__ double head_parent_S(const Params& P, int pa, int j) {
  if (pa < 0) return 0.0;
  if (P.collapsed) return P.OUT[(size_t)P.trunk_pos[pa] * P.OUT_LD + j];
  return P.T[(size_t)pa * P.NVP + j];
}

// x_i at the node below trunk position tp: x = a x + (bv + e) down the trunk path.
__device__ __forceinline__ double trunk_x(const Params& P, int tp, int i) {
  double x = P.p[i];
  const double a = P.a_diag[i];
  const int k0 = P.path_ptr[tp], k1 = P.path_ptr[tp + 1];
  for (int k = k0; k < k1; ++k)
    x = __dadd_rn(__dmul_rn(x, a), P.OUT[(size_t)P.path_list[k] * P.OUT_LD + P.X_OFF + i]);
  return x;
}

__device__ void rows_epilogue(const Params& P, int nu, int nrows);

// Backward fill: operand rows [s | psi^] of GEMM 1 (A region) and its bias beta
// (C region); a warp owns a row and issues each part's loads before using them.
// Templated on the 32-lane chunk counts of x (XC) and u (UC >= chunks of n_v).
template <int XC, int UC>
__device__ __noinline__ void fill_rows_t(const Params& P, int nu, int nrows) {
  const int LDA = P.LDA1, LDB = P.LDB1;
  double* const SA = g_smem;
  double* const SB = g_smem + kTileM * LDA;
  const int* const edge = SM_EDGE(P);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int E = P.n_edges;
  const int cur = (P.slot0 + nu) & 1;
  const double* __restrict__ Y = P.ybuf[cur];
  const double* __restrict__ Yp = P.ybuf[cur ^ 1];
  const bool apg = P.mode == kModeApg;
  const double c = apg ? P.coef[nu] : 0.0;
  const size_t zoff = (size_t)E * P.NXP, poff = 2 * zoff;
  for (int r = warp; r < nrows; r += kWarps) {
    const int e = edge[r];
    const int st = __ldg(P.edge_stage + e);
    double* row = SA + r * LDA;
    {  // s = D_sig w_sig + D_zeta w_zeta
      const double* ys = Y + (size_t)e * P.NXP + lane;
      const double* yps = Yp + (size_t)e * P.NXP + lane;
      double a[XC] = {}, b[XC] = {}, g[XC] = {}, h[XC] = {};
#pragma unroll
      for (int q = 0; q < XC; ++q) {
        if (lane + 32 * q < P.nx) {
          a[q] = gld(ys + 32 * q);
          g[q] = gld(ys + zoff + 32 * q);
          if (apg) {
            b[q] = gld(yps + 32 * q);
            h[q] = gld(yps + zoff + 32 * q);
          }
        }
      }
      const double ds = stage_scale(P.sig_stage, st, P.scaled);
      const double dz = stage_scale(P.zeta_stage, st, P.scaled);
#pragma unroll
      for (int q = 0; q < XC; ++q) {
        const int i = lane + 32 * q;
        if (i < P.NXP) {
          double v = 0.0;
          if (i < P.nx) {
            const double ws = apg ? extrap(a[q], b[q], c) : a[q];
            const double wz = apg ? extrap(g[q], h[q], c) : g[q];
            v = __dadd_rn(__dmul_rn(ws, ds), __dmul_rn(wz, dz));
          }
          row[i] = v;
        }
      }
    }
    {  // psi^ = D_psi w_psi, and beta into the C tile (zero pad columns)
      const double* yp_ = Y + poff + (size_t)e * P.NUP + lane;
      const double* ypp = Yp + poff + (size_t)e * P.NUP + lane;
      const double* bt = P.beta + (size_t)e * P.NVP + lane;
      const double* pst = P.psi_stage + (size_t)st * P.NUP + lane;
      double pv[UC] = {}, pp[UC] = {}, bb[UC] = {}, ps[UC];
#pragma unroll
      for (int q = 0; q < UC; ++q) {
        const int j = lane + 32 * q;
        ps[q] = 1.0;
        if (j < P.nu) {
          pv[q] = gld(yp_ + 32 * q);
          if (apg) pp[q] = gld(ypp + 32 * q);
          if (P.scaled) ps[q] = __ldg(pst + 32 * q);
        }
        if (j < P.nv) bb[q] = __ldg(bt + 32 * q);
      }
#pragma unroll
      for (int q = 0; q < UC; ++q) {
        const int j = lane + 32 * q;
        if (j < P.NT1 * 8) SB[r * LDB + j] = bb[q];
        if (j < P.NUP) {
          double v = 0.0;
          if (j < P.nu) {
            const double wp = apg ? extrap(pv[q], pp[q], c) : pv[q];
            v = P.scaled ? __dmul_rn(wp, ps[q]) : wp;
          }
          row[P.NXP + j] = v;
        }
      }
    }
  }
}

__device__ __noinline__ void fill_rows(const Params& P, int nu, int nrows) {
  const int xc = (P.nx + 31) >> 5, uc = (P.nu + 31) >> 5;
#define TSMPC_FILL(X, U) case (X) * 8 + (U): fill_rows_t<X, U>(P, nu, nrows); break;
  switch (xc * 8 + uc) {
    TSMPC_FILL(1, 1) TSMPC_FILL(1, 2) TSMPC_FILL(1, 3) TSMPC_FILL(1, 4)
    TSMPC_FILL(2, 1) TSMPC_FILL(2, 2) TSMPC_FILL(2, 3) TSMPC_FILL(2, 4)
    TSMPC_FILL(3, 1) TSMPC_FILL(3, 2) TSMPC_FILL(3, 3) TSMPC_FILL(3, 4)
    TSMPC_FILL(4, 1) TSMPC_FILL(4, 2) TSMPC_FILL(4, 3) TSMPC_FILL(4, 4)
    default: break;
  }
#undef TSMPC_FILL
}

// ---------------------------------------------------------------------------
// backward sweep of one tile
// ---------------------------------------------------------------------------
__device__ __noinline__ void bwd_tile(const Params& P, int tile, int nu) {
  int nrows, nsegs;
  load_tile(P, tile, nrows, nsegs);
  long long tm_ = clock64();
  (void)tm_;
  const int LDA = P.LDA1, LDB = P.LDB1;
  double* const SA = g_smem;
  double* const SB = g_smem + kTileM * LDA;
  const int* const edge = SM_EDGE(P);
  const int* const slo = SM_LO(P);
  const int* const shi = SM_HI(P);
  const int tid = threadIdx.x;

  // (1) operand rows [s | psi^] + GEMM-1 bias beta (warp per row)
  fill_rows(P, nu, nrows);
  __syncthreads();
  TSMPC_MARK(P, 0, tm_);

  // (2) xiq scan, tail -> head:  xiq_e = s_e + A' sum_{children} xiq_c
  if (P.diagA) {
    for (int idx = tid; idx < nsegs * P.nx; idx += kThreads) {
      const int s = idx / P.nx, i = idx - s * P.nx;
      const int lo = slo[s], hi = shi[s];
      const double acc = child_sum(P, P.XIQG, P.NXP, edge[hi - 1] + 1, i);
      const double a = P.a_diag[i];
      double x = __dadd_rn(SA[(hi - 1) * LDA + i], __dmul_rn(acc, a));
      SA[(hi - 1) * LDA + i] = x;
      for (int r = hi - 2; r >= lo; --r) {
        x = __dadd_rn(SA[r * LDA + i], __dmul_rn(x, a));
        SA[r * LDA + i] = x;
      }
      P.XIQG[(size_t)edge[lo] * P.NXP + i] = x;
    }
  } else {
    // dense A (level mode only): depth-synchronous GEMV steps; step 0 reads the
    // children sums straight from global memory (the C tile already holds beta)
    const int maxlen = SM_MISC(P)[0];
    for (int d = 0; d < maxlen; ++d) {
      for (int idx = tid; idx < nsegs * P.nx; idx += kThreads) {
        const int s = idx / P.nx, i = idx - s * P.nx;
        const int lo = slo[s], hi = shi[s];
        const int r = hi - 1 - d;
        if (r < lo) continue;
        // step d writes row r and reads only row r+1 (or the children sums): no hazard
        double q = 0.0;
        if (d == 0) {
          const int tail_node = edge[hi - 1] + 1;
          for (int j = 0; j < P.nx; ++j)
            q = fma(child_sum(P, P.XIQG, P.NXP, tail_node, j), P.A[(size_t)j * P.nx + i], q);
        } else {
          const double* prev = SA + (r + 1) * LDA;
          for (int j = 0; j < P.nx; ++j) q = fma(prev[j], P.A[(size_t)j * P.nx + i], q);
        }
        SA[r * LDA + i] = __dadd_rn(SA[r * LDA + i], q);
      }
      __syncthreads();
    }
    for (int idx = tid; idx < nsegs * P.nx; idx += kThreads) {
      const int s = idx / P.nx, i = idx - s * P.nx;
      const int lo = slo[s];
      P.XIQG[(size_t)edge[lo] * P.NXP + i] = SA[lo * LDA + i];
    }
  }
  __syncthreads();
  TSMPC_MARK(P, 1, tm_);

  // (3) GEMM 1: h = [xiq | psi^] [Bbar ; L] + beta
  gemm_dispatch(P, (nrows + 7) >> 3, 0, LDA, P.KS1, P.NT1, P.W1f, kTileM * LDA, LDB, nrows);
  __syncthreads();
  TSMPC_MARK(P, 2, tm_);

  // (4) g scan, tail -> head: g_e = (beta_e + h_e) + sum_children g_c ; t_e = g_e / (2 p_e)
  for (int idx = tid; idx < nsegs * P.nv; idx += kThreads) {
    const int s = idx / P.nv, j = idx - s * P.nv;
    const int lo = slo[s], hi = shi[s];
    double g = child_sum(P, P.GG, P.NVP, edge[hi - 1] + 1, j);
    for (int r = hi - 1; r >= lo; --r) {
      const int e = edge[r];
      g = __dadd_rn(SB[r * LDB + j], g);
      P.T[(size_t)e * P.NVP + j] = __dmul_rn(g, SM_INV2P(P)[r]);
    }
    P.GG[(size_t)edge[lo] * P.NVP + j] = g;
  }
  TSMPC_MARK(P, 3, tm_);
}

// ---------------------------------------------------------------------------
// forward sweep of one tile (+ prox / dual update epilogue in APG mode)
// ---------------------------------------------------------------------------
__device__ __noinline__ void fwd_tile(const Params& P, int tile, int nu) {
  int nrows, nsegs;
  load_tile(P, tile, nrows, nsegs);
  long long tm_ = clock64();
  (void)tm_;
  const int LDA = P.LDA2, LDB = P.LDB2;
  double* const SA = g_smem;
  double* const SB = g_smem + kTileM * LDA;
  const int* const edge = SM_EDGE(P);
  const int* const slo = SM_LO(P);
  const int* const shi = SM_HI(P);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K2 = P.KS2 * 4;

  // (1a) stage t rows (zero-padded to K2 columns) and GEMM 2's bias [uhat | e]
  for (int r = warp; r < nrows; r += kWarps) {
    const int e = edge[r];
    const double* tr = P.T + (size_t)e * P.NVP + lane;
    const double* uhp = P.uhat + (size_t)e * P.NUP + lane;
    const double* evp = P.evec + (size_t)e * P.NXP + lane;
    double v[kChunks] = {}, uh[kChunks] = {}, ev[kChunks] = {};
#pragma unroll
    for (int q = 0; q < kChunks; ++q) {
      const int j = lane + 32 * q;
      if (j < P.nv) v[q] = gld(tr + 32 * q);
      if (P.uhat && j < P.nu) uh[q] = __ldg(uhp + 32 * q);
      if (P.evec && j < P.nx) ev[q] = __ldg(evp + 32 * q);
    }
#pragma unroll
    for (int q = 0; q < kChunks; ++q) {
      const int j = lane + 32 * q;
      if (j < K2) SA[r * LDA + j] = v[q];
      if (j < P.NU8) SB[r * LDB + j] = uh[q];
      if (j < LDB - P.NU8) SB[r * LDB + P.NU8 + j] = ev[q];
    }
  }
  __syncthreads();
  TSMPC_MARK(P, 4, tm_);
  // (1b) S scan, head -> tail: S_e = t_e + S_parent  (in shared memory)
  for (int idx = tid; idx < nsegs * P.nv; idx += kThreads) {
    const int s = idx / P.nv, j = idx - s * P.nv;
    const int lo = slo[s], hi = shi[s];
    const int pa = P.anc[edge[lo] + 1] - 1;
    double S = head_parent_S(P, pa, j);
    for (int r = lo; r < hi; ++r) {
      S = __dadd_rn(SA[r * LDA + j], S);
      SA[r * LDA + j] = S;
    }
    if (!P.collapsed) P.T[(size_t)edge[hi - 1] * P.NVP + j] = S;  // the children's heads read it
  }
  __syncthreads();
  TSMPC_MARK(P, 5, tm_);

  // (2) GEMM 2: [u | bv + e] = S [Psi | Phi] + [uhat | e]
  gemm_dispatch(P, (nrows + 7) >> 3, 0, LDA, P.KS2, P.NT2, P.W2f, kTileM * LDA, LDB, nrows);
  __syncthreads();
  TSMPC_MARK(P, 6, tm_);

  // (3) x scan, head -> tail: x = A x_anc + (bv + e)   (x kept in the A region)
  if (P.diagA) {
    for (int idx = tid; idx < nsegs * P.nx; idx += kThreads) {
      const int s = idx / P.nx, i = idx - s * P.nx;
      const int lo = slo[s], hi = shi[s];
      const int an = P.anc[edge[lo] + 1];
      double xa = P.collapsed ? (an == 0 ? P.p[i] : trunk_x(P, P.trunk_pos[an - 1], i))
                              : P.X[(size_t)an * P.NXP + i];
      const double a = P.a_diag[i];
      for (int r = lo; r < hi; ++r) {
        xa = __dadd_rn(__dmul_rn(xa, a), SB[r * LDB + P.NU8 + i]);
        SA[r * LDA + i] = xa;
      }
      if (!P.collapsed) P.X[(size_t)(edge[hi - 1] + 1) * P.NXP + i] = xa;
    }
  } else {
    const int maxlen = SM_MISC(P)[0];
    for (int d = 0; d < maxlen; ++d) {
      for (int idx = tid; idx < nsegs * P.nx; idx += kThreads) {
        const int s = idx / P.nx, i = idx - s * P.nx;
        const int lo = slo[s], hi = shi[s];
        const int r = lo + d;
        if (r >= hi) continue;
        const int e = edge[r];
        const double* prev = (d == 0) ? (P.X + (size_t)P.anc[e + 1] * P.NXP) : (SA + (r - 1) * LDA);
        double q = 0.0;
        for (int j = 0; j < P.nx; ++j) q = fma(P.A[(size_t)i * P.nx + j], prev[j], q);
        SA[r * LDA + i] = __dadd_rn(q, SB[r * LDB + P.NU8 + i]);
      }
      __syncthreads();
    }
    for (int idx = tid; idx < nsegs * P.nx; idx += kThreads) {
      const int s = idx / P.nx, i = idx - s * P.nx;
      const int hi = shi[s];
      P.X[(size_t)(edge[hi - 1] + 1) * P.NXP + i] = SA[(hi - 1) * LDA + i];
    }
  }
  __syncthreads();
  TSMPC_MARK(P, 7, tm_);
  rows_epilogue(P, nu, nrows);
  TSMPC_MARK(P, 8, tm_);
}

#include "tsmpc_epilogue.cuh"

__device__ __noinline__ void rows_epilogue(const Params& P, int nu, int nrows) {
  if (P.mode != kModeApg) {  // STEP: store x, u
    const int LDA = P.LDA2, LDB = P.LDB2;
    const double* const SA = g_smem;
    const double* const SB = g_smem + kTileM * LDA;
    const int* const edge = SM_EDGE(P);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int r = warp; r < nrows; r += kWarps) {
      const int e = edge[r];
      for (int j = lane; j < P.nu; j += 32) P.U[(size_t)e * P.NUP + j] = SB[r * LDB + j];
      for (int i = lane; i < P.nx; i += 32) P.X[(size_t)(e + 1) * P.NXP + i] = SA[r * LDA + i];
    }
    return;
  }
  const int xc = (P.nx + 31) >> 5, uc = (P.nu + 31) >> 5;
#define TSMPC_EPI(X, U) case (X) * 8 + (U): rows_epilogue_t<X, U>(P, nu, nrows); break;
  switch (xc * 8 + uc) {
    TSMPC_EPI(1, 1) TSMPC_EPI(1, 2) TSMPC_EPI(1, 3) TSMPC_EPI(1, 4)
    TSMPC_EPI(2, 1) TSMPC_EPI(2, 2) TSMPC_EPI(2, 3) TSMPC_EPI(2, 4)
    TSMPC_EPI(3, 1) TSMPC_EPI(3, 2) TSMPC_EPI(3, 3) TSMPC_EPI(3, 4)
    TSMPC_EPI(4, 1) TSMPC_EPI(4, 2) TSMPC_EPI(4, 3) TSMPC_EPI(4, 4)
    default: break;
  }
#undef TSMPC_EPI
}

// ---------------------------------------------------------------------------
// collapsed trunk (diagonal A).  With g_a = sum over the trunk subtree of a of
// (beta_k + [xiq_k | psi^_k] W1) plus the chain-head sums G_c below it, linearity
// gives, per trunk edge a (b runs over the trunk path root .. a):
//   K_a = sum_b inv2p_b (sum_{k in sub(b)} beta_k + sum_{heads c in sub(b)} G_c)
//   Y_a = sum_b inv2p_b  sum_{k in sub(b)} [xiq_k | psi^_k]
//   S_a = K_a + Y_a W1,   [u_a - uhat_a | bv_a] = S_a W2 = K_a W2 + Y_a (W1 W2)
// The first two are per-component tree recursions (one CTA per component slice,
// no cross-component coupling because A is diagonal); the last is one GEMM of the
// T trunk rows against the fused [[I, W2], [W1, W1 W2]] operator.
// ---------------------------------------------------------------------------

// v + sum over the children ch of trunk row tp: trunk children contribute
// KY[child][col], chain-head children hb[ch][hcol] (skipped when hb is null).
// Children of a node are contiguous edges, hence contiguous trunk positions.
__device__ __forceinline__ double child_acc(const Params& P, int tp, int ch0, int ch1, int col,
                                            const double* hb, int hld, int hcol, double v) {
  const int tc = P.trunk_child0[tp];
  const int n = ch1 - ch0;
  if (tc >= 0) {
#pragma unroll 4
    for (int k = 0; k < n; ++k) v = __dadd_rn(v, P.KY[(size_t)(tc + k) * P.KY_LD + col]);
  } else if (tc == -1) {
    if (hb) {
#pragma unroll 4
      for (int ch = ch0; ch < ch1; ++ch) v = __dadd_rn(v, hb[(size_t)ch * hld + hcol]);
    }
  } else {
    for (int ch = ch0; ch < ch1; ++ch) {
      const int cp = P.trunk_pos[ch];
      if (cp >= 0) v = __dadd_rn(v, P.KY[(size_t)cp * P.KY_LD + col]);
      else if (hb) v = __dadd_rn(v, hb[(size_t)ch * hld + hcol]);
    }
  }
  return v;
}

// Phase B: component-sliced trunk recursion -> KY = [K | Yx | Ypsi] (and XIQG for
// trunk edges).
__device__ __noinline__ void trunk_sweep(const Params& P, int nu) {
  const int ncomp = P.nv + P.nx + P.nu;
  const int c_lo = (int)((long long)ncomp * blockIdx.x / gridDim.x);
  const int c_hi = (int)((long long)ncomp * (blockIdx.x + 1) / gridDim.x);
  const int nc = c_hi - c_lo;
  if (nc <= 0) return;
  const int E = P.n_edges;
  const bool apg = P.mode == kModeApg;
  const int cur = (P.slot0 + nu) & 1;
  const double* __restrict__ Y = P.ybuf[cur];
  const double* __restrict__ Yp = P.ybuf[cur ^ 1];
  const double c = apg ? P.coef[nu] : 0.0;
  const size_t zoff = (size_t)E * P.NXP, poff = 2 * zoff;
  // bottom-up over edge stages (children live in later stages)
  for (int st = P.N - 1; st >= 0; --st) {
    const int t0 = P.trunk_stage_ptr[st], t1 = P.trunk_stage_ptr[st + 1];
    if (t0 == t1) continue;  // block-uniform
    for (int idx = threadIdx.x; idx < (t1 - t0) * nc; idx += kThreads) {
      const int tp = t0 + idx / nc, q = c_lo + idx % nc;
      const int a = P.trunk_edge[tp];
      const int node = a + 1;
      const int ch0 = P.child_start[node] - 1, ch1 = P.child_stop[node] - 1;
      double* ky = P.KY + (size_t)tp * P.KY_LD;
      if (q < P.nv) {  // K part: beta sums (+ chain heads' G)
        const int j = q;
        ky[j] = child_acc(P, tp, ch0, ch1, j, P.GG, P.NVP, j, P.beta[(size_t)a * P.NVP + j]);
      } else if (q < P.nv + P.nx) {  // xiq and its subtree sum
        const int i = q - P.nv;
        const int es = P.edge_stage[a];
        const size_t o = (size_t)a * P.NXP + i;
        const double ws = apg ? extrap(Y[o], Yp[o], c) : Y[o];
        const double wz = apg ? extrap(Y[zoff + o], Yp[zoff + o], c) : Y[zoff + o];
        const double s = __dadd_rn(__dmul_rn(ws, stage_scale(P.sig_stage, es, P.scaled)),
                                   __dmul_rn(wz, stage_scale(P.zeta_stage, es, P.scaled)));
        double xs = 0.0;
#pragma unroll 4
        for (int ch = ch0; ch < ch1; ++ch) xs = __dadd_rn(xs, P.XIQG[(size_t)ch * P.NXP + i]);
        const double zs = child_acc(P, tp, ch0, ch1, P.NVP + i, nullptr, 0, 0, 0.0);
        const double xiq = __dadd_rn(s, __dmul_rn(xs, P.a_diag[i]));
        P.XIQG[o] = xiq;
        ky[P.NVP + i] = __dadd_rn(xiq, zs);
      } else {  // psi^ subtree sum
        const int j = q - P.nv - P.nx;
        const int es = P.edge_stage[a];
        const size_t o = poff + (size_t)a * P.NUP + j;
        const double wp = apg ? extrap(Y[o], Yp[o], c) : Y[o];
        const double v = P.scaled ? __dmul_rn(wp, P.psi_stage[(size_t)es * P.NUP + j]) : wp;
        ky[P.NVP + P.NXP + j] = child_acc(P, tp, ch0, ch1, P.NVP + P.NXP + j, nullptr, 0, 0, v);
      }
    }
    __syncthreads();
  }
  // top-down: K_a, Y_a = own * inv2p_a + parent's
  for (int st = 0; st < P.N; ++st) {
    const int t0 = P.trunk_stage_ptr[st], t1 = P.trunk_stage_ptr[st + 1];
    if (t0 == t1) continue;
    for (int idx = threadIdx.x; idx < (t1 - t0) * nc; idx += kThreads) {
      const int tp = t0 + idx / nc, q = c_lo + idx % nc;
      const int a = P.trunk_edge[tp];
      const int col = q < P.nv ? q : (q < P.nv + P.nx ? P.NVP + (q - P.nv) : P.NVP + P.NXP + (q - P.nv - P.nx));
      const int pa = P.anc[a + 1] - 1;
      double v = __dmul_rn(P.KY[(size_t)tp * P.KY_LD + col], P.inv2p[a]);
      if (pa >= 0) v = __dadd_rn(v, P.KY[(size_t)P.trunk_pos[pa] * P.KY_LD + col]);
      P.KY[(size_t)tp * P.KY_LD + col] = v;
    }
    __syncthreads();
  }
}

// Phase B with the CTA's component slice staged in shared memory (the tile region
// is free between the sweeps): one parallel round of global loads (own terms and
// chain-head contributions, which do not depend on the recursion), then the
// bottom-up / top-down recursions touch shared memory only, then one store round.
// Zs[tp][k]: beta sums (K) or subtree sums Z (Yx, Ypsi); Xs[tp][k]: xiq (Yx).
__device__ __noinline__ void trunk_sweep_smem(const Params& P, int nu) {
  const int T = P.n_trunk;
  const int ncomp = P.nv + P.nx + P.nu;
  const int c_lo = (int)((long long)ncomp * blockIdx.x / gridDim.x);
  const int c_hi = (int)((long long)ncomp * (blockIdx.x + 1) / gridDim.x);
  const int nc = c_hi - c_lo;
  if (nc <= 0) return;
  double* const Zs = g_smem;
  double* const Xs = g_smem + (size_t)T * nc;
  const int E = P.n_edges;
  const bool apg = P.mode == kModeApg;
  const int cur = (P.slot0 + nu) & 1;
  const double* __restrict__ Y = P.ybuf[cur];
  const double* __restrict__ Yp = P.ybuf[cur ^ 1];
  const double c = apg ? P.coef[nu] : 0.0;
  const size_t zoff = (size_t)E * P.NXP, poff = 2 * zoff;
  __syncthreads();  // shared memory is free
  // (1) own terms + chain-head children (independent of the recursion)
  for (int idx = threadIdx.x; idx < T * nc; idx += kThreads) {
    const int tp = idx / nc, k = idx - tp * nc, q = c_lo + k;
    const int a = P.trunk_edge[tp];
    const int node = a + 1;
    const int ch0 = P.child_start[node] - 1, ch1 = P.child_stop[node] - 1;
    const int tc = P.trunk_child0[tp];  // >= 0: no chain-head children
    double z = 0.0, x = 0.0;
    if (q < P.nv) {
      z = __ldg(P.beta + (size_t)a * P.NVP + q);
      if (tc < 0)
        for (int ch = ch0; ch < ch1; ++ch)
          if (tc == -1 || P.trunk_pos[ch] < 0) z = __dadd_rn(z, gld(P.GG + (size_t)ch * P.NVP + q));
    } else if (q < P.nv + P.nx) {
      const int i = q - P.nv;
      const int es = __ldg(P.edge_stage + a);
      const size_t o = (size_t)a * P.NXP + i;
      const double ws = apg ? extrap(gld(Y + o), gld(Yp + o), c) : gld(Y + o);
      const double wz = apg ? extrap(gld(Y + zoff + o), gld(Yp + zoff + o), c) : gld(Y + zoff + o);
      const double s = __dadd_rn(__dmul_rn(ws, stage_scale(P.sig_stage, es, P.scaled)),
                                 __dmul_rn(wz, stage_scale(P.zeta_stage, es, P.scaled)));
      double h = 0.0;
      if (tc < 0)
        for (int ch = ch0; ch < ch1; ++ch)
          if (tc == -1 || P.trunk_pos[ch] < 0) h = __dadd_rn(h, gld(P.XIQG + (size_t)ch * P.NXP + i));
      x = __dadd_rn(s, __dmul_rn(h, P.a_diag[i]));  // s + a * (head-children xiq)
    } else {
      const int j = q - P.nv - P.nx;
      const int es = __ldg(P.edge_stage + a);
      const size_t o = poff + (size_t)a * P.NUP + j;
      const double wp = apg ? extrap(gld(Y + o), gld(Yp + o), c) : gld(Y + o);
      z = P.scaled ? __dmul_rn(wp, __ldg(P.psi_stage + (size_t)es * P.NUP + j)) : wp;
    }
    Zs[idx] = z;
    Xs[idx] = x;
  }
  __syncthreads();
  // (2) bottom-up: add the trunk children (shared memory only)
  for (int st = P.N - 1; st >= 0; --st) {
    const int t0 = P.trunk_stage_ptr[st], t1 = P.trunk_stage_ptr[st + 1];
    if (t0 == t1) continue;  // block-uniform
    for (int idx = t0 * nc + threadIdx.x; idx < t1 * nc; idx += kThreads) {
      const int tp = idx / nc, k = idx - tp * nc, q = c_lo + k;
      const int tc = P.trunk_child0[tp];
      if (tc == -1) {
        if (q >= P.nv && q < P.nv + P.nx) Zs[idx] = Xs[idx];  // leaf of the trunk: Z = xiq
        continue;
      }
      const int a = P.trunk_edge[tp];
      const int node = a + 1;
      const int n = P.child_stop[node] - P.child_start[node];
      double zs = 0.0, xs = 0.0;
      for (int m = 0; m < n; ++m) {
        const int cp = tc >= 0 ? tc + m : P.trunk_pos[P.child_start[node] - 1 + m];
        if (cp < 0) continue;
        zs = __dadd_rn(zs, Zs[cp * nc + k]);
        xs = __dadd_rn(xs, Xs[cp * nc + k]);
      }
      if (q >= P.nv && q < P.nv + P.nx) {
        const double xiq = __dadd_rn(Xs[idx], __dmul_rn(xs, P.a_diag[q - P.nv]));
        Xs[idx] = xiq;
        Zs[idx] = __dadd_rn(xiq, zs);
      } else {
        Zs[idx] = __dadd_rn(Zs[idx], zs);
      }
    }
    __syncthreads();
  }
  // (3) top-down: K_a, Y_a = own * inv2p_a + parent's
  for (int st = 0; st < P.N; ++st) {
    const int t0 = P.trunk_stage_ptr[st], t1 = P.trunk_stage_ptr[st + 1];
    if (t0 == t1) continue;
    for (int idx = t0 * nc + threadIdx.x; idx < t1 * nc; idx += kThreads) {
      const int tp = idx / nc, k = idx - tp * nc;
      const int pp = P.trunk_parent[tp];
      double v = __dmul_rn(Zs[idx], __ldg(P.inv2p + P.trunk_edge[tp]));
      if (pp >= 0) v = __dadd_rn(v, Zs[pp * nc + k]);
      Zs[idx] = v;
    }
    __syncthreads();
  }
  // (4) results: KY columns of the slice, xiq of the trunk edges
  for (int idx = threadIdx.x; idx < T * nc; idx += kThreads) {
    const int tp = idx / nc, k = idx - tp * nc, q = c_lo + k;
    const int col = q < P.nv ? q : (q < P.nv + P.nx ? P.NVP + (q - P.nv) : P.NVP + P.NXP + (q - P.nv - P.nx));
    gst(P.KY + (size_t)tp * P.KY_LD + col, Zs[idx]);
    if (q >= P.nv && q < P.nv + P.nx) gst(P.XIQG + (size_t)P.trunk_edge[tp] * P.NXP + (q - P.nv), Xs[idx]);
  }
}

// Phase C: OUT = KY * MT + [0 | uhat | e] for all trunk rows.  Work item = (n-tile,
// block of 4 m-tiles); the 13 warps of a CTA split the k-steps and reduce their
// partial tiles through shared memory in a fixed order (deterministic).
__device__ __noinline__ void trunk_gemm(const Params& P) {
  const int T = P.n_trunk;
  constexpr int MTB = 4;
  const int mblocks = (T + 8 * MTB - 1) / (8 * MTB);
  const int items = P.NTT * mblocks;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ar = lane >> 2, ac = lane & 3;
  double* const red = g_smem;  // [kWarps][MTB][32][2]
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    const int nt = it % P.NTT, mb = it / P.NTT;
    const int k0 = (int)((long long)P.KSK * warp / kWarps), k1 = (int)((long long)P.KSK * (warp + 1) / kWarps);
    double acc[MTB][2];
#pragma unroll
    for (int m = 0; m < MTB; ++m) acc[m][0] = acc[m][1] = 0.0;
    const double* bp = P.MTf + (size_t)nt * P.KSK * 32 + lane;
#pragma unroll 2
    for (int ks = k0; ks < k1; ++ks) {
      const double b = __ldg(bp + (size_t)ks * 32);
#pragma unroll
      for (int m = 0; m < MTB; ++m) {
        const int row = (mb * MTB + m) * 8 + ar;
        const double a = row < T ? P.KY[(size_t)row * P.KY_LD + ks * 4 + ac] : 0.0;
        dmma8x8x4(acc[m], a, b);
      }
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < MTB; ++m) {
      red[((warp * MTB + m) * 32 + lane) * 2] = acc[m][0];
      red[((warp * MTB + m) * 32 + lane) * 2 + 1] = acc[m][1];
    }
    __syncthreads();
    if (warp < MTB) {
      const int m = warp;
      double v0 = 0.0, v1 = 0.0;
      for (int w = 0; w < kWarps; ++w) {
        v0 = __dadd_rn(v0, red[((w * MTB + m) * 32 + lane) * 2]);
        v1 = __dadd_rn(v1, red[((w * MTB + m) * 32 + lane) * 2 + 1]);
      }
      const int row = (mb * MTB + m) * 8 + ar;
      if (row < T) {
        const int e = P.trunk_edge[row];
        const int col = nt * 8 + 2 * ac;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cc = col + h;
          double bias = 0.0;
          if (cc >= P.U_OFF && cc < P.U_OFF + P.nu && P.uhat) bias = P.uhat[(size_t)e * P.NUP + cc - P.U_OFF];
          if (cc >= P.X_OFF && cc < P.X_OFF + P.nx && P.evec) bias = P.evec[(size_t)e * P.NXP + cc - P.X_OFF];
          P.OUT[(size_t)row * P.OUT_LD + cc] = __dadd_rn(h ? v1 : v0, bias);
        }
      }
    }
  }
}

// Phase D (trunk part): x by the trunk path recursion, u from OUT, then the
// standard row epilogue, for the trunk rows owned by this CTA.
__device__ __noinline__ void trunk_rows(const Params& P, int nu) {
  const int T = P.n_trunk;
  const int LDA = P.LDA2, LDB = P.LDB2;
  double* const SA = g_smem;
  double* const SB = g_smem + kTileM * LDA;
  int* const edge = SM_EDGE(P);
  // trunk row tp goes to CTA C-1-(tp mod C): round-robin from the last CTA, which
  // the balanced chain assignment leaves with the fewest chain rows
  const int C = gridDim.x;
  const int first = C - 1 - (int)blockIdx.x;
  const int mine = first < T ? (T - 1 - first) / C + 1 : 0;
  for (int k0 = 0; k0 < mine; k0 += kTileM) {
    const int nrows = min(kTileM, mine - k0);
    __syncthreads();
    for (int r = threadIdx.x; r < nrows; r += kThreads) edge[r] = P.trunk_edge[first + (k0 + r) * C];
    for (int idx = threadIdx.x; idx < nrows * P.nx; idx += kThreads) {
      const int r = idx / P.nx, i = idx - r * P.nx;
      SA[r * LDA + i] = trunk_x(P, first + (k0 + r) * C, i);
    }
    for (int idx = threadIdx.x; idx < nrows * P.nu; idx += kThreads) {
      const int r = idx / P.nu, j = idx - r * P.nu;
      SB[r * LDB + j] = P.OUT[(size_t)(first + (k0 + r) * C) * P.OUT_LD + P.U_OFF + j];
    }
    __syncthreads();
    rows_epilogue(P, nu, nrows);
  }
}

__global__ void __launch_bounds__(kThreads, 1) apg_persistent_kernel(const __grid_constant__ Params P) {
  cg::grid_group grid = cg::this_grid();
  const int cta = blockIdx.x;
  const int D = P.n_levels;
  {  // model bound vectors for the epilogue, once per launch
    double* bnd = SM_BOUNDS(P);
    for (int i = threadIdx.x; i < P.NXP; i += kThreads) {
      bnd[i] = P.x_s[i];
      bnd[P.NXP + i] = P.x_min[i];
      bnd[2 * P.NXP + i] = P.x_max[i];
    }
    for (int j = threadIdx.x; j < P.NUP; j += kThreads) {
      bnd[3 * P.NXP + j] = P.u_min[j];
      bnd[3 * P.NXP + P.NUP + j] = P.u_max[j];
    }
    __syncthreads();
  }
  if (P.collapsed) {
    // leaf segments = level-0 tiles; trunk collapsed: 3 grid barriers / iteration
    const int* lt = P.lvl_tiles + cta;
    const bool trunk = P.n_trunk > 0;
    for (int nu = 0; nu < P.iters; ++nu) {
      for (int t = lt[0]; t < lt[1]; ++t) bwd_tile(P, t, nu);
      if (trunk) {
        long long tb_ = clock64();
        grid.sync();
        TSMPC_MARK(P, 9, tb_);
        if (P.trunk_smem) trunk_sweep_smem(P, nu);
        else trunk_sweep(P, nu);
        TSMPC_MARK(P, 10, tb_);
        grid.sync();
        TSMPC_MARK(P, 9, tb_);
        trunk_gemm(P);
        TSMPC_MARK(P, 11, tb_);
        grid.sync();
        TSMPC_MARK(P, 9, tb_);
      }
      if (P.mode == kModeApg && cta == 0) {
        const double th = P.theta[nu];
        const double om = __dsub_rn(1.0, th);
        for (int i = threadIdx.x; i < P.nx; i += kThreads)
          P.xavg[i] = __dadd_rn(__dmul_rn(P.xavg[i], om), __dmul_rn(th, P.p[i]));
      }
      if (trunk) {
        long long tr_ = clock64();
        trunk_rows(P, nu);
        TSMPC_MARK(P, 12, tr_);
      }
      for (int t = lt[0]; t < lt[1]; ++t) fwd_tile(P, t, nu);
    }
    return;
  }
  for (int nu = 0; nu < P.iters; ++nu) {
    for (int l = D - 1; l >= 0; --l) {
      const int* lt = P.lvl_tiles + l * P.n_ctas + cta;
      for (int t = lt[0]; t < lt[1]; ++t) bwd_tile(P, t, nu);
      if (l > 0) { long long tb_ = clock64(); grid.sync(); TSMPC_MARK(P, 9, tb_); }
    }
    if (P.mode == kModeApg && cta == 0) {
      const double th = P.theta[nu];
      const double om = __dsub_rn(1.0, th);
      for (int i = threadIdx.x; i < P.nx; i += kThreads)
        P.xavg[i] = __dadd_rn(__dmul_rn(P.xavg[i], om), __dmul_rn(th, P.p[i]));
    }
    for (int l = 0; l < D; ++l) {
      const int* lt = P.lvl_tiles + l * P.n_ctas + cta;
      for (int t = lt[0]; t < lt[1]; ++t) fwd_tile(P, t, nu);
      if (l < D - 1) { long long tb_ = clock64(); grid.sync(); TSMPC_MARK(P, 9, tb_); }
    }
  }
}

}  // namespace tsmpc
