// tsmpc_apg.cu — persistent cooperative APG kernel for sm_100a.
// See tsmpc_kernels.cuh for the algorithm outline and DESIGN.md for the
// derivation, data layout and roofline.
#include "tsmpc_kernels.cuh"

namespace cg = cooperative_groups;

namespace tsmpc {

__device__ __forceinline__ void dmma8x8x4(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// C[rows, nt*8 .. nt*8+7] = A[rows, 0:4*KS] * B for every n-tile owned by this
// warp.  A is a shared-memory tile (row-major, lda = 4 mod 16 for conflict-free
// fragment loads), B is global memory in fragment order [NT][KS][32] so each
// warp-wide B load is one coalesced 256-byte transaction; B fragments are
// register-prefetched 8 k-steps ahead and reused across all MT m-tiles.
template <int MT>
__device__ __forceinline__ void gemm_tile(const double* __restrict__ As, int lda, int KS, int NT,
                                          const double* __restrict__ Bf, double* __restrict__ Cs,
                                          int ldc) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ar = lane >> 2, ac = lane & 3;
  for (int nt = warp; nt < NT; nt += kWarps) {
    double acc[MT][2];
#pragma unroll
    for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = 0.0;
    const double* bp = Bf + (size_t)nt * KS * 32 + lane;
    double bq[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) bq[q] = (q < KS) ? __ldg(bp + q * 32) : 0.0;
    const double* ap = As + ar * lda + ac;
    for (int ks0 = 0; ks0 < KS; ks0 += 8) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int ks = ks0 + q;
        if (ks < KS) {
          const double b = bq[q];
          if (ks + 8 < KS) bq[q] = __ldg(bp + (ks + 8) * 32);
#pragma unroll
          for (int m = 0; m < MT; ++m) dmma8x8x4(acc[m], ap[m * 8 * lda + ks * 4], b);
        }
      }
    }
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      double* cp = Cs + (m * 8 + ar) * ldc + nt * 8 + 2 * ac;
      cp[0] = acc[m][0];
      cp[1] = acc[m][1];
    }
  }
}

__device__ __noinline__ void gemm_dispatch(int mt, const double* As, int lda, int KS, int NT,
                                           const double* Bf, double* Cs, int ldc) {
  switch (mt) {
    case 1: gemm_tile<1>(As, lda, KS, NT, Bf, Cs, ldc); break;
    case 2: gemm_tile<2>(As, lda, KS, NT, Bf, Cs, ldc); break;
    case 3: gemm_tile<3>(As, lda, KS, NT, Bf, Cs, ldc); break;
    case 4: gemm_tile<4>(As, lda, KS, NT, Bf, Cs, ldc); break;
    case 5: gemm_tile<5>(As, lda, KS, NT, Bf, Cs, ldc); break;
    case 6: gemm_tile<6>(As, lda, KS, NT, Bf, Cs, ldc); break;
    case 7: gemm_tile<7>(As, lda, KS, NT, Bf, Cs, ldc); break;
    default: gemm_tile<8>(As, lda, KS, NT, Bf, Cs, ldc); break;
  }
}

struct Smem {
  double* A;   // kTileM x LDA
  double* B;   // kTileM x LDB
  int* edge;   // kTileM
  int* lo;     // kTileM
  int* hi;     // kTileM
  int* misc;   // [0] = longest segment of the tile
};

__device__ __forceinline__ void load_tile(const Params& P, int tile, const Smem& sm, int& nrows,
                                          int& nsegs) {
  const int sg0 = P.tile_seg[tile], sg1 = P.tile_seg[tile + 1];
  const int rbase = P.seg_row[sg0];
  nrows = P.seg_row[sg1] - rbase;
  nsegs = sg1 - sg0;
  __syncthreads();  // the previous tile is done with shared memory
  for (int i = threadIdx.x; i < nrows; i += kThreads) sm.edge[i] = P.row_edge[rbase + i];
  if (threadIdx.x == 0) sm.misc[0] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < nsegs; i += kThreads) {
    const int lo = P.seg_row[sg0 + i] - rbase, hi = P.seg_row[sg0 + i + 1] - rbase;
    sm.lo[i] = lo;
    sm.hi[i] = hi;
    atomicMax(sm.misc, hi - lo);
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

// ---------------------------------------------------------------------------
// backward sweep of one tile
// ---------------------------------------------------------------------------
__device__ void bwd_tile(const Params& P, int tile, int nu, const Smem& sm) {
  int nrows, nsegs;
  load_tile(P, tile, sm, nrows, nsegs);
  const int tid = threadIdx.x;
  const int E = P.n_edges;
  const int cur = (P.slot0 + nu) & 1;
  const double* Y = P.ybuf[cur];
  const double* Yp = P.ybuf[cur ^ 1];
  const bool apg = P.mode == kModeApg;
  const double c = apg ? P.coef[nu] : 0.0;
  const int K1 = P.KS1 * 4;
  const size_t zoff = (size_t)E * P.NXP, poff = 2 * (size_t)E * P.NXP;

  // (1) operand rows [s | psi^] in shared memory
  for (int idx = tid; idx < nrows * K1; idx += kThreads) {
    const int r = idx / K1, k = idx - r * K1;
    const int e = sm.edge[r];
    const int st = P.edge_stage[e];
    double v = 0.0;
    if (k < P.NXP) {
      if (k < P.nx) {
        const size_t o = (size_t)e * P.NXP + k;
        const double ws = apg ? extrap(Y[o], Yp[o], c) : Y[o];
        const double wz = apg ? extrap(Y[zoff + o], Yp[zoff + o], c) : Y[zoff + o];
        v = __dadd_rn(__dmul_rn(ws, stage_scale(P.sig_stage, st, P.scaled)),
                      __dmul_rn(wz, stage_scale(P.zeta_stage, st, P.scaled)));
      }
    } else {
      const int j = k - P.NXP;
      if (j < P.nu) {
        const size_t o = poff + (size_t)e * P.NUP + j;
        const double wp = apg ? extrap(Y[o], Yp[o], c) : Y[o];
        v = P.scaled ? __dmul_rn(wp, P.psi_stage[(size_t)st * P.NUP + j]) : wp;
      }
    }
    sm.A[r * P.LDA + k] = v;
  }
  __syncthreads();

  // (2) xiq scan, tail -> head:  xiq_e = s_e + A' sum_{children} xiq_c
  if (P.diagA) {
    for (int idx = tid; idx < nsegs * P.nx; idx += kThreads) {
      const int s = idx / P.nx, i = idx - s * P.nx;
      const int lo = sm.lo[s], hi = sm.hi[s];
      const int tail_node = sm.edge[hi - 1] + 1;
      const int c0 = P.child_start[tail_node] - 1, c1 = P.child_stop[tail_node] - 1;
      double acc = 0.0;
      for (int ch = c0; ch < c1; ++ch) acc = __dadd_rn(acc, P.XIQG[(size_t)ch * P.NXP + i]);
      const double a = P.a_diag[i];
      double x = __dadd_rn(sm.A[(hi - 1) * P.LDA + i], __dmul_rn(acc, a));
      sm.A[(hi - 1) * P.LDA + i] = x;
      for (int r = hi - 2; r >= lo; --r) {
        x = __dadd_rn(sm.A[r * P.LDA + i], __dmul_rn(x, a));
        sm.A[r * P.LDA + i] = x;
      }
      P.XIQG[(size_t)sm.edge[lo] * P.NXP + i] = x;
    }
  } else {
    // dense A: children sums into B scratch, then depth-synchronous GEMV steps
    for (int idx = tid; idx < nsegs * P.nx; idx += kThreads) {
      const int s = idx / P.nx, i = idx - s * P.nx;
      const int tail_node = sm.edge[sm.hi[s] - 1] + 1;
      const int c0 = P.child_start[tail_node] - 1, c1 = P.child_stop[tail_node] - 1;
      double acc = 0.0;
      for (int ch = c0; ch < c1; ++ch) acc = __dadd_rn(acc, P.XIQG[(size_t)ch * P.NXP + i]);
      sm.B[s * P.LDB + i] = acc;
    }
    __syncthreads();
    const int maxlen = sm.misc[0];
    for (int d = 0; d < maxlen; ++d) {
      for (int idx = tid; idx < nsegs * P.nx; idx += kThreads) {
        const int s = idx / P.nx, i = idx - s * P.nx;
        const int lo = sm.lo[s], hi = sm.hi[s];
        const int r = hi - 1 - d;
        if (r < lo) continue;
        // step d writes row r and reads only row r+1 (or the children sum): no hazard
        const double* prev = (d == 0) ? (sm.B + s * P.LDB) : (sm.A + (r + 1) * P.LDA);
        double q = 0.0;
        for (int j = 0; j < P.nx; ++j) q = fma(prev[j], P.A[(size_t)j * P.nx + i], q);
        sm.A[r * P.LDA + i] = __dadd_rn(sm.A[r * P.LDA + i], q);
      }
      __syncthreads();
    }
    for (int idx = tid; idx < nsegs * P.nx; idx += kThreads) {
      const int s = idx / P.nx, i = idx - s * P.nx;
      const int lo = sm.lo[s];
      P.XIQG[(size_t)sm.edge[lo] * P.NXP + i] = sm.A[lo * P.LDA + i];
    }
  }
  __syncthreads();

  // (3) GEMM 1: h = [xiq | psi^] [Bbar ; L]
  gemm_dispatch((nrows + 7) >> 3, sm.A, P.LDA, P.KS1, P.NT1, P.W1f, sm.B, P.LDB);
  __syncthreads();

  // (4) g scan, tail -> head: g_e = (beta_e + sum_children g_c) + h_e ; t_e = g_e / (2 p_e)
  for (int idx = tid; idx < nsegs * P.nv; idx += kThreads) {
    const int s = idx / P.nv, j = idx - s * P.nv;
    const int lo = sm.lo[s], hi = sm.hi[s];
    const int tail_node = sm.edge[hi - 1] + 1;
    const int c0 = P.child_start[tail_node] - 1, c1 = P.child_stop[tail_node] - 1;
    double acc = 0.0;
    for (int ch = c0; ch < c1; ++ch) acc = __dadd_rn(acc, P.GG[(size_t)ch * P.NVP + j]);
    double g = 0.0;
    for (int r = hi - 1; r >= lo; --r) {
      const int e = sm.edge[r];
      g = __dadd_rn(__dadd_rn(P.beta[(size_t)e * P.NVP + j], acc), sm.B[r * P.LDB + j]);
      acc = g;
      P.T[(size_t)e * P.NVP + j] = __dmul_rn(g, P.inv2p[e]);
    }
    P.GG[(size_t)sm.edge[lo] * P.NVP + j] = g;
  }
}

// ---------------------------------------------------------------------------
// forward sweep of one tile (+ prox / dual update epilogue in APG mode)
// ---------------------------------------------------------------------------
__device__ void fwd_tile(const Params& P, int tile, int nu, const Smem& sm) {
  int nrows, nsegs;
  load_tile(P, tile, sm, nrows, nsegs);
  const int tid = threadIdx.x;
  const int K2 = P.KS2 * 4;
  const bool apg = P.mode == kModeApg;
  const bool last = (nu == P.iters - 1) || !apg;

  // (1) S scan, head -> tail: S_e = t_e + S_parent
  for (int idx = tid; idx < nsegs * K2; idx += kThreads) {
    const int s = idx / K2, j = idx - s * K2;
    const int lo = sm.lo[s], hi = sm.hi[s];
    if (j >= P.nv) {
      for (int r = lo; r < hi; ++r) sm.A[r * P.LDA + j] = 0.0;
      continue;
    }
    const int head = sm.edge[lo];
    const int pa = P.anc[head + 1] - 1;
    double S = (pa >= 0) ? P.T[(size_t)pa * P.NVP + j] : 0.0;
    for (int r = lo; r < hi; ++r) {
      S = __dadd_rn(P.T[(size_t)sm.edge[r] * P.NVP + j], S);
      sm.A[r * P.LDA + j] = S;
    }
    P.T[(size_t)sm.edge[hi - 1] * P.NVP + j] = S;  // the children's heads read it
  }
  __syncthreads();

  // (2) GEMM 2: [du | bv] = S [Psi | Phi]
  gemm_dispatch((nrows + 7) >> 3, sm.A, P.LDA, P.KS2, P.NT2, P.W2f, sm.B, P.LDB);
  __syncthreads();

  // (3) x scan, head -> tail: x = A x_anc + bv + e   (x kept in sm.A)
  if (P.diagA) {
    for (int idx = tid; idx < nsegs * P.nx; idx += kThreads) {
      const int s = idx / P.nx, i = idx - s * P.nx;
      const int lo = sm.lo[s], hi = sm.hi[s];
      const int an = P.anc[sm.edge[lo] + 1];
      double xa = P.X[(size_t)an * P.NXP + i];
      const double a = P.a_diag[i];
      for (int r = lo; r < hi; ++r) {
        const int e = sm.edge[r];
        const double ev = P.evec ? P.evec[(size_t)e * P.NXP + i] : 0.0;
        const double x = __dadd_rn(__dadd_rn(__dmul_rn(xa, a), sm.B[r * P.LDB + P.NU8 + i]), ev);
        sm.A[r * P.LDA + i] = x;
        if (last) P.X[(size_t)(e + 1) * P.NXP + i] = x;
        xa = x;
      }
      if (!last) P.X[(size_t)(sm.edge[hi - 1] + 1) * P.NXP + i] = xa;
    }
  } else {
    const int maxlen = sm.misc[0];
    for (int d = 0; d < maxlen; ++d) {
      for (int idx = tid; idx < nsegs * P.nx; idx += kThreads) {
        const int s = idx / P.nx, i = idx - s * P.nx;
        const int lo = sm.lo[s], hi = sm.hi[s];
        const int r = lo + d;
        if (r >= hi) continue;
        const int e = sm.edge[r];
        const double* prev = (d == 0) ? (P.X + (size_t)P.anc[e + 1] * P.NXP) : (sm.A + (r - 1) * P.LDA);
        double q = 0.0;
        for (int j = 0; j < P.nx; ++j) q = fma(P.A[(size_t)i * P.nx + j], prev[j], q);
        const double ev = P.evec ? P.evec[(size_t)e * P.NXP + i] : 0.0;
        sm.A[r * P.LDA + i] = __dadd_rn(__dadd_rn(q, sm.B[r * P.LDB + P.NU8 + i]), ev);
      }
      __syncthreads();
    }
    for (int idx = tid; idx < nsegs * P.nx; idx += kThreads) {
      const int s = idx / P.nx, i = idx - s * P.nx;
      const int lo = sm.lo[s], hi = sm.hi[s];
      for (int r = lo; r < hi; ++r) {
        if (last || r == hi - 1) P.X[(size_t)(sm.edge[r] + 1) * P.NXP + i] = sm.A[r * P.LDA + i];
      }
    }
  }
  __syncthreads();

  // (4) per-row epilogue: one warp per edge row
  const int warp = tid >> 5, lane = tid & 31;
  if (!apg) {
    for (int idx = tid; idx < nrows * P.nu; idx += kThreads) {
      const int r = idx / P.nu, j = idx - r * P.nu;
      const int e = sm.edge[r];
      const double uh = P.uhat ? P.uhat[(size_t)e * P.NUP + j] : 0.0;
      P.U[(size_t)e * P.NUP + j] = __dadd_rn(sm.B[r * P.LDB + j], uh);
    }
    return;
  }
  const int E = P.n_edges;
  const int cur = (P.slot0 + nu) & 1;
  const double* Y = P.ybuf[cur];
  double* Yn = P.ybuf[cur ^ 1];  // y_prev slot receives y_next
  const double c = P.coef[nu];
  const double th = P.theta[nu];
  const double om = __dsub_rn(1.0, th);
  const double lam = P.lam;
  const double lam_p = 1.0 / lam;  // prox parameter (engine.py:555)
  const size_t zoff = (size_t)E * P.NXP, poff = 2 * (size_t)E * P.NXP;
  double rmax = 0.0;
  for (int r = warp; r < nrows; r += kWarps) {
    const int e = sm.edge[r];
    const int node = e + 1;
    const int st = P.edge_stage[e];
    const double ds = stage_scale(P.sig_stage, st, P.scaled);
    const double dz = stage_scale(P.zeta_stage, st, P.scaled);
    // --- state copies: two weighted-distance prox blocks (engine.py:146-180)
    double xs[4], ws[4], wz[4], ts[4], tz[4];
    double ss = 0.0, sz = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = lane + 32 * q;
      if (i < P.nx) {
        const size_t o = (size_t)e * P.NXP + i;
        const double x = sm.A[r * P.LDA + i];
        xs[q] = x;
        ws[q] = extrap(Y[o], Yn[o], c);
        wz[q] = extrap(Y[zoff + o], Yn[zoff + o], c);
        // t_arg = w / lam + D Hz   (engine.py:552-554)
        ts[q] = __dadd_rn(__ddiv_rn(ws[q], lam), __dmul_rn(x, ds));
        tz[q] = __dadd_rn(__ddiv_rn(wz[q], lam), __dmul_rn(x, dz));
        const double ps = fmax(ts[q], __dmul_rn(ds, P.x_s[i]));
        const double pz = fmin(fmax(tz[q], __dmul_rn(dz, P.x_min[i])), __dmul_rn(dz, P.x_max[i]));
        const double gs = __dsub_rn(ps, ts[q]), gz = __dsub_rn(pz, tz[q]);
        ss = fma(gs, gs, ss);
        sz = fma(gz, gz, sz);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      ss += __shfl_xor_sync(0xffffffffu, ss, off);
      sz += __shfl_xor_sync(0xffffffffu, sz, off);
    }
    const double dist_s = sqrt(ss), dist_z = sqrt(sz);
    const double wgt_s = __ddiv_rn(__dmul_rn(lam_p, P.Wx), ds);
    const double wgt_z = __ddiv_rn(__dmul_rn(lam_p, P.gamma_d), dz);
    const double fs = dist_s > wgt_s ? __ddiv_rn(wgt_s, dist_s) : 1.0;
    const double fz = dist_z > wgt_z ? __ddiv_rn(wgt_z, dist_z) : 1.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = lane + 32 * q;
      if (i < P.nx) {
        const size_t o = (size_t)e * P.NXP + i;
        const double x = xs[q];
        const double hs = __dmul_rn(x, ds), hz = __dmul_rn(x, dz);
        const double ps = fmax(ts[q], __dmul_rn(ds, P.x_s[i]));
        const double pz = fmin(fmax(tz[q], __dmul_rn(dz, P.x_min[i])), __dmul_rn(dz, P.x_max[i]));
        const double t_s = __dadd_rn(ts[q], __dmul_rn(fs, __dsub_rn(ps, ts[q])));
        const double t_z = __dadd_rn(tz[q], __dmul_rn(fz, __dsub_rn(pz, tz[q])));
        Yn[o] = __dadd_rn(ws[q], __dmul_rn(lam, __dsub_rn(hs, t_s)));
        Yn[zoff + o] = __dadd_rn(wz[q], __dmul_rn(lam, __dsub_rn(hz, t_z)));
        if (last || P.record_all) {
          rmax = fmax(rmax, fabs(__dsub_rn(x, __ddiv_rn(t_s, ds))));
          rmax = fmax(rmax, fabs(__dsub_rn(x, __ddiv_rn(t_z, dz))));
        }
        const size_t oa = (size_t)node * P.NXP + i;
        P.xavg[oa] = __dadd_rn(__dmul_rn(P.xavg[oa], om), __dmul_rn(th, x));
      }
    }
    // --- input copy: box projection (engine.py:182)
    for (int j = lane; j < P.nu; j += 32) {
      const size_t o = poff + (size_t)e * P.NUP + j;
      const size_t ou = (size_t)e * P.NUP + j;
      const double uh = P.uhat ? P.uhat[ou] : 0.0;
      const double u = __dadd_rn(sm.B[r * P.LDB + j], uh);
      const double dp = P.scaled ? P.psi_stage[(size_t)st * P.NUP + j] : 1.0;
      const double w = extrap(Y[o], Yn[o], c);
      const double hp = __dmul_rn(u, dp);
      const double a = __dadd_rn(__ddiv_rn(w, lam), hp);
      const double t = fmin(fmax(a, __dmul_rn(dp, P.u_min[j])), __dmul_rn(dp, P.u_max[j]));
      Yn[o] = __dadd_rn(w, __dmul_rn(lam, __dsub_rn(hp, t)));
      if (last || P.record_all) rmax = fmax(rmax, fabs(__dsub_rn(u, __ddiv_rn(t, dp))));
      P.uavg[ou] = __dadd_rn(__dmul_rn(P.uavg[ou], om), __dmul_rn(th, u));
      if (last) P.U[ou] = u;
    }
  }
  if (last || P.record_all) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, off));
    if (lane == 0 && rmax > 0.0)
      atomicMax(P.resid + (P.record_all ? nu : 0), (unsigned long long)__double_as_longlong(rmax));
  }
}

__global__ void __launch_bounds__(kThreads, 1) apg_persistent_kernel(Params P) {
  extern __shared__ __align__(16) double smem[];
  Smem sm;
  sm.A = smem;
  sm.B = sm.A + kTileM * P.LDA;
  sm.edge = reinterpret_cast<int*>(sm.B + kTileM * P.LDB);
  sm.lo = sm.edge + kTileM;
  sm.hi = sm.lo + kTileM;
  sm.misc = sm.hi + kTileM;
  cg::grid_group grid = cg::this_grid();
  const int cta = blockIdx.x;
  const int D = P.n_levels;
  for (int nu = 0; nu < P.iters; ++nu) {
    for (int l = D - 1; l >= 0; --l) {
      const int* lt = P.lvl_tiles + l * P.n_ctas + cta;
      for (int t = lt[0]; t < lt[1]; ++t) bwd_tile(P, t, nu, sm);
      if (l > 0) grid.sync();
    }
    if (P.mode == kModeApg && cta == 0) {
      const double th = P.theta[nu];
      const double om = __dsub_rn(1.0, th);
      for (int i = threadIdx.x; i < P.nx; i += kThreads)
        P.xavg[i] = __dadd_rn(__dmul_rn(P.xavg[i], om), __dmul_rn(th, P.p[i]));
    }
    for (int l = 0; l < D; ++l) {
      const int* lt = P.lvl_tiles + l * P.n_ctas + cta;
      for (int t = lt[0]; t < lt[1]; ++t) fwd_tile(P, t, nu, sm);
      if (l < D - 1) grid.sync();
    }
  }
}

size_t smem_bytes(int LDA, int LDB) {
  return sizeof(double) * (size_t)kTileM * (LDA + LDB) + sizeof(int) * (3 * kTileM + 4);
}

}  // namespace tsmpc
