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

namespace cg = cooperative_groups;

namespace tsmpc {

extern __shared__ __align__(16) double s_dyn[];

namespace {

// ---- meta layout (ints, per CTA) -------------------------------------------
//   [0] ntiles [1] nrows [2] nsegs [3] nneed [4] nlev [5] nown [6] resident [7] 0
//   tiles : ntiles x {row0, nrows, seg0, nsegs}
//   rows  : nrows  x {edge, stage, inv2p lo, inv2p hi}
//   segs  : nsegs  x {lo, hi, pneed, 0}         (lo/hi relative to the tile)
//   needs : nneed  x {trunk pos, pneed, edge, stage}   (sorted by depth)
//   lev   : nlev + 1 need offsets per depth
//   own   : nown need indices (trunk rows whose epilogue this CTA runs)
struct Meta {
  const int* m;
  int ntiles, nrows, nsegs, nneed, nlev, nown, resident;
  const int *tiles, *rows, *segs, *needs, *lev, *own;
  __device__ void bind(const int* base) {
    m = base;
    ntiles = m[0]; nrows = m[1]; nsegs = m[2]; nneed = m[3]; nlev = m[4]; nown = m[5]; resident = m[6];
    tiles = m + 8;
    rows = tiles + 4 * ntiles;
    segs = rows + 4 * nrows;
    needs = segs + 4 * nsegs;
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
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

struct Ctx {
  const SParams* S;
  const Params* P;
  Meta mt;
  double* bnd;     // x_s, x_min, x_max (NXP each), u_min, u_max (NUP each)
  const int* spi;  // sparse index pool (shared)
  const double* spv;
  double* need;    // need rows [S | x | u]
  double* work;    // XI | Z | H  (backward),  XB | DU | H=S  (forward)
  double* slot;
  int NXP, NUP, NVP, YW, SL;
  int nx, nu, nv, E;
  __device__ double* XI() const { return work; }
  __device__ double* Z() const { return work + kTileS * NXP; }
  __device__ double* H() const { return work + kTileS * (NXP + NUP); }
};

// slot row pointers: Y0 | Y1 | XA | UA | T
__device__ __forceinline__ double* slot_row(const Ctx& c, int srow) { return c.slot + (size_t)srow * c.SL; }

// Issue cp.async copies of one tile's slot rows.  parts: 1 = both dual rows,
// 2 = ergodic rows.  ysm = smem dual index that receives HBM slot `cur`.
__device__ void load_slot(const Ctx& c, int row0, int nrows, int srow0, int parts, int cur, int ysm) {
  const Params& P = *c.P;
  const int hx = c.NXP / 2, hu = c.NUP / 2;
  const int per_y = 2 * hx + hu;               // 16-byte chunks of one dual row
  const int nch = ((parts & 1) ? 2 * per_y : 0) + ((parts & 2) ? hx + hu : 0);
  const size_t E = (size_t)c.E;
  for (int idx = threadIdx.x; idx < nrows * nch; idx += kThreadsS) {
    const int r = idx / nch;
    int k = idx - r * nch;
    const int e = c.mt.edge(row0 + r);
    double* srow = slot_row(c, srow0 + r);
    if (parts & 1) {
      if (k < 2 * per_y) {
        const int which = k < per_y ? 0 : 1;     // 0: HBM slot cur, 1: cur ^ 1
        const int kk = k - which * per_y;
        const double* Y = P.ybuf[cur ^ which];
        double* dst = srow + (size_t)(ysm ^ which) * c.YW;
        const double* src;
        if (kk < hx) src = Y + (size_t)e * c.NXP + 2 * kk, dst += 2 * kk;
        else if (kk < 2 * hx) src = Y + E * c.NXP + (size_t)e * c.NXP + 2 * (kk - hx), dst += c.NXP + 2 * (kk - hx);
        else src = Y + 2 * E * c.NXP + (size_t)e * c.NUP + 2 * (kk - 2 * hx), dst += 2 * c.NXP + 2 * (kk - 2 * hx);
        cp16(dst, src);
        continue;
      }
      k -= 2 * per_y;
    }
    double* xa = srow + 2 * c.YW;
    if (k < hx) cp16(xa + 2 * k, P.xavg + (size_t)(e + 1) * c.NXP + 2 * k);
    else cp16(xa + c.NXP + 2 * (k - hx), P.uavg + (size_t)e * c.NUP + 2 * (k - hx));
  }
}

// ----------------------------------------------------------------------------
// epilogue: prox_g (engine.py:146-183), dual update, ergodic averages, residual
// (engine.py:546-575) for nrows rows.  Row r: edge ge(r), stage gs(r); x at
// xrow(r), u at urow(r), dual rows (y at index ysm, y_prev at ysm ^ 1) and
// ergodic rows in the slot-format row srow(r).  y+ replaces y_prev in place.
// wt: also write y+ and the ergodic rows to HBM (slot `ncur` receives y+).
// ----------------------------------------------------------------------------
template <class EdgeOf, class StageOf, class XOf, class UOf, class SOf>
__device__ void epilogue(const Ctx& c, int nu_it, int nrows, EdgeOf ge, StageOf gs, XOf xrow, UOf urow,
                         SOf srow, int ysm, bool wt, int ncur, double& rmax) {
  const Params& P = *c.P;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool last = nu_it == P.iters - 1;
  const bool want = last || P.record_all;
  const double cf = P.coef[nu_it], th = P.theta[nu_it], om = __dsub_rn(1.0, th);
  const double lam = P.lam, ilam = P.inv_lam, lam_p = 1.0 / lam;
  const size_t E = (size_t)c.E;
  double* Yn = P.ybuf[ncur];
  const double* xs_s = c.bnd;
  const double* xmn_s = c.bnd + c.NXP;
  const double* xmx_s = c.bnd + 2 * c.NXP;
  const double* umn_s = c.bnd + 3 * c.NXP;
  const double* umx_s = c.bnd + 3 * c.NXP + c.NUP;
  // --- state copies: warp per row, two weighted-distance prox blocks
  for (int r = warp; r < nrows; r += kWarpsS) {
    const int e = ge(r), st = gs(r);
    double* row = srow(r);
    double* yc = row + (size_t)ysm * c.YW;
    double* yp = row + (size_t)(ysm ^ 1) * c.YW;
    double* xa = row + 2 * c.YW;
    const double* x = xrow(r);
    const double ds = P.scaled ? __ldg(P.sig_stage + st) : 1.0;
    const double dz = P.scaled ? __ldg(P.zeta_stage + st) : 1.0;
    const double rds = P.scaled ? __ldg(P.sig_rcp + st) : 1.0;
    const double rdz = P.scaled ? __ldg(P.zeta_rcp + st) : 1.0;
    double ts[4], tz[4], ws[4], wz[4];
    double ss = 0.0, sz = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = lane + 32 * q;
      ts[q] = tz[q] = ws[q] = wz[q] = 0.0;
      if (i < c.nx) {
        ws[q] = extrap(yc[i], yp[i], cf);
        wz[q] = extrap(yc[c.NXP + i], yp[c.NXP + i], cf);
        const double xi = x[i];
        ts[q] = __dadd_rn(__dmul_rn(ws[q], ilam), __dmul_rn(xi, ds));
        tz[q] = __dadd_rn(__dmul_rn(wz[q], ilam), __dmul_rn(xi, dz));
        const double ps = fmax(ts[q], __dmul_rn(ds, xs_s[i]));
        const double pz = fmin(fmax(tz[q], __dmul_rn(dz, xmn_s[i])), __dmul_rn(dz, xmx_s[i]));
        const double gs_ = __dsub_rn(ps, ts[q]), gz = __dsub_rn(pz, tz[q]);
        ss = fma(gs_, gs_, ss);
        sz = fma(gz, gz, sz);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      ss += __shfl_xor_sync(0xffffffffu, ss, off);
      sz += __shfl_xor_sync(0xffffffffu, sz, off);
    }
    const double dist_s = sqrt(ss), dist_z = sqrt(sz);
    const double wgt_s = __dmul_rn(__dmul_rn(lam_p, P.Wx), rds);
    const double wgt_z = __dmul_rn(__dmul_rn(lam_p, P.gamma_d), rdz);
    const double fs = dist_s > wgt_s ? __ddiv_rn(wgt_s, dist_s) : 1.0;
    const double fz = dist_z > wgt_z ? __ddiv_rn(wgt_z, dist_z) : 1.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = lane + 32 * q;
      if (i < c.nx) {
        const double xi = x[i];
        const double hs = __dmul_rn(xi, ds), hz = __dmul_rn(xi, dz);
        const double ps = fmax(ts[q], __dmul_rn(ds, xs_s[i]));
        const double pz = fmin(fmax(tz[q], __dmul_rn(dz, xmn_s[i])), __dmul_rn(dz, xmx_s[i]));
        const double t_s = __dadd_rn(ts[q], __dmul_rn(fs, __dsub_rn(ps, ts[q])));
        const double t_z = __dadd_rn(tz[q], __dmul_rn(fz, __dsub_rn(pz, tz[q])));
        const double ns = __dadd_rn(ws[q], __dmul_rn(lam, __dsub_rn(hs, t_s)));
        const double nz = __dadd_rn(wz[q], __dmul_rn(lam, __dsub_rn(hz, t_z)));
        yp[i] = ns;
        yp[c.NXP + i] = nz;
        if (want) {
          rmax = fmax(rmax, fabs(__dsub_rn(xi, __dmul_rn(t_s, rds))));
          rmax = fmax(rmax, fabs(__dsub_rn(xi, __dmul_rn(t_z, rdz))));
        }
        const double na = __dadd_rn(__dmul_rn(xa[i], om), __dmul_rn(th, xi));
        xa[i] = na;
        if (wt) {
          stcg(Yn + (size_t)e * c.NXP + i, ns);
          stcg(Yn + E * c.NXP + (size_t)e * c.NXP + i, nz);
          stcg(P.xavg + (size_t)(e + 1) * c.NXP + i, na);
        }
        if (last) stcg(P.X + (size_t)(e + 1) * c.NXP + i, xi);
      }
    }
  }
  // --- input copy: box projection (engine.py:182), element-parallel
  for (int idx = threadIdx.x; idx < nrows * c.nu; idx += kThreadsS) {
    const int r = idx / c.nu, j = idx - r * c.nu;
    const int e = ge(r), st = gs(r);
    double* row = srow(r);
    double* yc = row + (size_t)ysm * c.YW + 2 * c.NXP;
    double* yp = row + (size_t)(ysm ^ 1) * c.YW + 2 * c.NXP;
    double* ua = row + 2 * c.YW + c.NXP;
    const double u = urow(r)[j];
    const double dp = P.scaled ? __ldg(P.psi_stage + (size_t)st * c.NUP + j) : 1.0;
    const double w = extrap(yc[j], yp[j], cf);
    const double hp = __dmul_rn(u, dp);
    const double a = __dadd_rn(__dmul_rn(w, ilam), hp);
    const double t = fmin(fmax(a, __dmul_rn(dp, umn_s[j])), __dmul_rn(dp, umx_s[j]));
    const double ny = __dadd_rn(w, __dmul_rn(lam, __dsub_rn(hp, t)));
    yp[j] = ny;
    if (want) {
      const double rdp = P.scaled ? __ldg(P.psi_rcp + (size_t)st * c.NUP + j) : 1.0;
      rmax = fmax(rmax, fabs(__dsub_rn(u, __dmul_rn(t, rdp))));
    }
    const double na = __dadd_rn(__dmul_rn(ua[j], om), __dmul_rn(th, u));
    ua[j] = na;
    if (wt) {
      stcg(Yn + 2 * E * c.NXP + (size_t)e * c.NUP + j, ny);
      stcg(P.uavg + (size_t)e * c.NUP + j, na);
    }
    if (last) stcg(P.U + (size_t)e * c.NUP + j, u);
  }
}

// ----------------------------------------------------------------------------
// backward sweep of tile ti (reference factor.py:142-156)
// ----------------------------------------------------------------------------
__device__ void bwd_tile(const Ctx& c, int ti, int nu_it, int ysm, int srow0, bool resident, int cur) {
  const Params& P = *c.P;
  const SParams& S = *c.S;
  const int* td = c.mt.tiles + 4 * ti;
  const int row0 = td[0], nrows = td[1], seg0 = td[2], nsegs = td[3];
  const int tid = threadIdx.x;
  const int nx = c.nx, nu = c.nu, nv = c.nv;
  const bool apg = true;
  const double cf = P.coef[nu_it];
  double* XI = c.XI();
  double* Z = c.Z();
  double* H = c.H();
  long long tm_ = clock64();
  (void)tm_;
  // prefetch beta_s (the bias of h) for this thread's (row, k) elements
  constexpr int kPer = (kTileS * 128 + kThreadsS - 1) / kThreadsS;
  double bpre[kPer];
#pragma unroll
  for (int m = 0; m < kPer; ++m) {
    const int idx = tid + m * kThreadsS;
    bpre[m] = 0.0;
    if (idx < nrows * nv) {
      const int r = idx / nv, k = idx - r * nv;
      bpre[m] = ldcg(S.beta_s + (size_t)c.mt.edge(row0 + r) * c.NVP + k);
    }
  }
  if (!resident) {
    cp_wait<0>();
    __syncthreads();
  }
  // (1) fill: s = D_sig w_sig + D_zeta w_zeta ; psi^ = D_psi w_psi
  for (int idx = tid; idx < nrows * (nx + nu); idx += kThreadsS) {
    const int r = idx / (nx + nu), k = idx - r * (nx + nu);
    const int st = c.mt.stage(row0 + r);
    const double* yc = slot_row(c, srow0 + r) + (size_t)ysm * c.YW;
    const double* yp = slot_row(c, srow0 + r) + (size_t)(ysm ^ 1) * c.YW;
    if (k < nx) {
      const double ws = apg ? extrap(yc[k], yp[k], cf) : yc[k];
      const double wz = apg ? extrap(yc[c.NXP + k], yp[c.NXP + k], cf) : yc[c.NXP + k];
      const double ds = P.scaled ? __ldg(P.sig_stage + st) : 1.0;
      const double dz = P.scaled ? __ldg(P.zeta_stage + st) : 1.0;
      XI[r * c.NXP + k] = __dadd_rn(__dmul_rn(ws, ds), __dmul_rn(wz, dz));
    } else {
      const int j = k - nx;
      const double wp = apg ? extrap(yc[2 * c.NXP + j], yp[2 * c.NXP + j], cf) : yc[2 * c.NXP + j];
      Z[r * c.NUP + j] = P.scaled ? __dmul_rn(wp, __ldg(P.psi_stage + (size_t)st * c.NUP + j)) : wp;
    }
  }
  __syncthreads();
  TSMPC_MARK(P, 0, tm_);
  // streamed CTAs: the slot is free again -> prefetch the next tile's dual rows
  // (or, after the last backward tile, the ergodic rows the forward sweep needs)
  if (!resident) {
    if (ti > 0) {
      const int* tn = c.mt.tiles + 4 * (ti - 1);
      load_slot(c, tn[0], tn[1], 0, 1, cur, ysm);
    } else {
      load_slot(c, row0, nrows, 0, 2, cur, ysm);
    }
    cp_commit();
  }
  // (2) xiq scan, tail -> head (leaf tails have no children)
  const double* adiag = c.bnd + 3 * c.NXP + 2 * c.NUP;
  for (int idx = tid; idx < nsegs * nx; idx += kThreadsS) {
    const int s = idx / nx, i = idx - s * nx;
    const int* sg = c.mt.segs + 4 * (seg0 + s);
    const int lo = sg[0], hi = sg[1];
    const double a = adiag[i];
    double x = XI[(hi - 1) * c.NXP + i];
    for (int r = hi - 2; r >= lo; --r) {
      x = __dadd_rn(XI[r * c.NXP + i], __dmul_rn(x, a));
      XI[r * c.NXP + i] = x;
    }
    if (sg[2] >= 0) stcg(P.XIQG + (size_t)c.mt.edge(row0 + lo) * c.NXP + i, x);
  }
  __syncthreads();
  TSMPC_MARK(P, 1, tm_);
  // (3) z = psi^ + B' xiq   (CSC of B: column j -> rows i)
  {
    const int* cp = c.spi + S.Bc_ptr;
    const int* ci = c.spi + S.Bc_idx;
    const double* cv = c.spv + S.Bc_val;
    for (int idx = tid; idx < nrows * nu; idx += kThreadsS) {
      const int r = idx / nu, j = idx - r * nu;
      double z = Z[r * c.NUP + j];
      for (int q = cp[j]; q < cp[j + 1]; ++q) z = fma(cv[q], XI[r * c.NXP + ci[q]], z);
      Z[r * c.NUP + j] = z;
    }
  }
  __syncthreads();
  // (4) h = beta_s + Ls' z   (CSC of Ls: column k -> rows j)
  {
    const int* cp = c.spi + S.Lc_ptr;
    const int* ci = c.spi + S.Lc_idx;
    const double* cv = c.spv + S.Lc_val;
#pragma unroll
    for (int m = 0; m < kPer; ++m) {
      const int idx = tid + m * kThreadsS;
      if (idx < nrows * nv) {
        const int r = idx / nv, k = idx - r * nv;
        double h = 0.0;
        for (int q = cp[k]; q < cp[k + 1]; ++q) h = fma(cv[q], Z[r * c.NUP + ci[q]], h);
        H[r * c.NVP + k] = __dadd_rn(bpre[m], h);
      }
    }
  }
  __syncthreads();
  TSMPC_MARK(P, 2, tm_);
  // (5) g scan, tail -> head: g_e = h_e + g_child ; t_e = g_e / (2 p_e)
  for (int idx = tid; idx < nsegs * nv; idx += kThreadsS) {
    const int s = idx / nv, k = idx - s * nv;
    const int* sg = c.mt.segs + 4 * (seg0 + s);
    const int lo = sg[0], hi = sg[1];
    double g = 0.0;
    for (int r = hi - 1; r >= lo; --r) {
      g = __dadd_rn(H[r * c.NVP + k], g);
      const double t = __dmul_rn(g, c.mt.inv2p(row0 + r));
      if (resident) slot_row(c, srow0 + r)[2 * c.YW + c.NXP + c.NUP + k] = t;
      else stcg(S.TG + (size_t)c.mt.edge(row0 + r) * c.NVP + k, t);
    }
    if (sg[2] >= 0) stcg(P.GG + (size_t)c.mt.edge(row0 + lo) * c.NVP + k, g);
  }
  __syncthreads();
  TSMPC_MARK(P, 3, tm_);
}

// ----------------------------------------------------------------------------
// forward sweep of tile ti (factor.py:158-170) + epilogue
// ----------------------------------------------------------------------------
__device__ void fwd_tile(const Ctx& c, int ti, int nu_it, int ysm, int srow0, bool resident, int cur,
                         double& rmax) {
  const Params& P = *c.P;
  const SParams& S = *c.S;
  const int* td = c.mt.tiles + 4 * ti;
  const int row0 = td[0], nrows = td[1], seg0 = td[2], nsegs = td[3];
  const int tid = threadIdx.x;
  const int nx = c.nx, nu = c.nu, nv = c.nv;
  double* XB = c.XI();
  double* DU = c.Z();
  double* SS = c.H();
  long long tm_ = clock64();
  (void)tm_;
  if (!resident) {
    // t rows of this tile -> S region; then (after the previous epilogue) the slot
    const int hv = c.NVP / 2;
    for (int idx = tid; idx < nrows * hv; idx += kThreadsS) {
      const int r = idx / hv, k = idx - r * hv;
      cp16(SS + r * c.NVP + 2 * k, S.TG + (size_t)c.mt.edge(row0 + r) * c.NVP + 2 * k);
    }
    cp_commit();
    if (ti > 0) load_slot(c, row0, nrows, 0, 3, cur, ysm);
    cp_commit();
  }
  // prefetch the static biases: uhat (u = uhat + du) and e (x recursion)
  constexpr int kPerU = (kTileS * 128 + kThreadsS - 1) / kThreadsS;
  double upre[kPerU], epre[kPerU];
#pragma unroll
  for (int m = 0; m < kPerU; ++m) {
    const int idx = tid + m * kThreadsS;
    upre[m] = epre[m] = 0.0;
    if (idx < nrows * nu) {
      const int r = idx / nu, j = idx - r * nu;
      upre[m] = ldcg(P.uhat + (size_t)c.mt.edge(row0 + r) * c.NUP + j);
    }
    if (idx < nrows * nx) {
      const int r = idx / nx, i = idx - r * nx;
      epre[m] = ldcg(P.evec + (size_t)c.mt.edge(row0 + r) * c.NXP + i);
    }
  }
  if (!resident) {
    cp_wait<1>();
    __syncthreads();
  }
  // (1) S scan, head -> tail: S_e = t_e + S_parent
  for (int idx = tid; idx < nsegs * nv; idx += kThreadsS) {
    const int s = idx / nv, k = idx - s * nv;
    const int* sg = c.mt.segs + 4 * (seg0 + s);
    const int lo = sg[0], hi = sg[1], pn = sg[2];
    double Sv = pn >= 0 ? c.need[(size_t)pn * c.S->need_ld + k] : 0.0;
    for (int r = lo; r < hi; ++r) {
      const double t = resident ? slot_row(c, srow0 + r)[2 * c.YW + c.NXP + c.NUP + k] : SS[r * c.NVP + k];
      Sv = __dadd_rn(t, Sv);
      SS[r * c.NVP + k] = Sv;
    }
  }
  __syncthreads();
  TSMPC_MARK(P, 4, tm_);
  // (2) du = Lt S   (CSR of Lt: row j -> columns k)
  {
    const int* rp = c.spi + S.Lr_ptr;
    const int* ri = c.spi + S.Lr_idx;
    const double* rv = c.spv + S.Lr_val;
    for (int idx = tid; idx < nrows * nu; idx += kThreadsS) {
      const int r = idx / nu, j = idx - r * nu;
      double d = 0.0;
      for (int q = rp[j]; q < rp[j + 1]; ++q) d = fma(rv[q], SS[r * c.NVP + ri[q]], d);
      DU[r * c.NUP + j] = d;
    }
  }
  __syncthreads();
  // (3) bv + e = B du + e   (CSR of B: row i -> columns j)
  {
    const int* rp = c.spi + S.Br_ptr;
    const int* ri = c.spi + S.Br_idx;
    const double* rv = c.spv + S.Br_val;
#pragma unroll
    for (int m = 0; m < kPerU; ++m) {
      const int idx = tid + m * kThreadsS;
      if (idx < nrows * nx) {
        const int r = idx / nx, i = idx - r * nx;
        double b = 0.0;
        for (int q = rp[i]; q < rp[i + 1]; ++q) b = fma(rv[q], DU[r * c.NUP + ri[q]], b);
        XB[r * c.NXP + i] = __dadd_rn(b, epre[m]);
      }
    }
  }
  __syncthreads();
  TSMPC_MARK(P, 6, tm_);
  // (4) u = uhat + du ; x scan, head -> tail: x = a .* x_anc + (bv + e)
#pragma unroll
  for (int m = 0; m < kPerU; ++m) {
    const int idx = tid + m * kThreadsS;
    if (idx < nrows * nu) {
      const int r = idx / nu, j = idx - r * nu;
      DU[r * c.NUP + j] = __dadd_rn(DU[r * c.NUP + j], upre[m]);
    }
  }
  {
    const double* adiag = c.bnd + 3 * c.NXP + 2 * c.NUP;
    for (int idx = tid; idx < nsegs * nx; idx += kThreadsS) {
      const int s = idx / nx, i = idx - s * nx;
      const int* sg = c.mt.segs + 4 * (seg0 + s);
      const int lo = sg[0], hi = sg[1], pn = sg[2];
      double x = pn >= 0 ? c.need[(size_t)pn * c.S->need_ld + c.NVP + i] : P.p[i];
      const double a = adiag[i];
      for (int r = lo; r < hi; ++r) {
        x = __dadd_rn(__dmul_rn(x, a), XB[r * c.NXP + i]);
        XB[r * c.NXP + i] = x;
      }
    }
  }
  if (!resident) cp_wait<0>();
  __syncthreads();
  TSMPC_MARK(P, 7, tm_);
  // (5) epilogue
  const Meta& mt = c.mt;
  epilogue(
      c, nu_it, nrows, [&](int r) { return mt.edge(row0 + r); }, [&](int r) { return mt.stage(row0 + r); },
      [&](int r) { return XB + r * c.NXP; }, [&](int r) { return DU + r * c.NUP; },
      [&](int r) { return slot_row(c, srow0 + r); }, ysm, !resident || nu_it == P.iters - 1, cur ^ 1, rmax);
  __syncthreads();
  TSMPC_MARK(P, 8, tm_);
}

// ----------------------------------------------------------------------------
// phase B: component-sliced trunk sweep -> KY (see tsmpc_apg.cu trunk_sweep_smem
// for the recursion; here the schedule is staged in shared memory first)
// ----------------------------------------------------------------------------
__device__ void trunk_sweep(const Ctx& c, int nu_it, int cur) {
  const Params& P = *c.P;
  const SParams& S = *c.S;
  const int ncomp = c.nv + c.nx + c.nu;
  const int c_lo = (int)((long long)ncomp * blockIdx.x / gridDim.x);
  const int c_hi = (int)((long long)ncomp * (blockIdx.x + 1) / gridDim.x);
  const int nc = c_hi - c_lo;
  if (nc <= 0) return;
  const int* g = S.tsched;
  const int T = __ldg(g), nlev = __ldg(g + 1);
  double* Zs = c.work;
  double* Xs = Zs + (size_t)T * nc;
  int* sch = reinterpret_cast<int*>(Xs + (size_t)T * nc);
  for (int i = threadIdx.x; i < S.n_tsched; i += kThreadsS) sch[i] = __ldg(g + i);
  __syncthreads();
  const int* lev = sch + 4;
  const int* pos = lev + nlev + 1;
  const int* tch = pos + 8 * T;
  const int* hch = tch + sch[2];
  const size_t E = (size_t)c.E;
  const double* Y = P.ybuf[cur];
  const double* Yp = P.ybuf[cur ^ 1];
  const double cf = P.coef[nu_it];
  const double* adiag = c.bnd + 3 * c.NXP + 2 * c.NUP;
  // (1) own terms + chain-head children (one parallel round of loads)
  for (int idx = threadIdx.x; idx < T * nc; idx += kThreadsS) {
    const int tp = idx / nc, k = idx - tp * nc, q = c_lo + k;
    const int* ps = pos + 8 * tp;
    const int a = ps[0], st = ps[1], h0 = ps[5], nh = ps[6];
    double z = 0.0, x = 0.0;
    if (q < c.nv) {
      z = ldcg(S.beta_s + (size_t)a * c.NVP + q);
      for (int m = 0; m < nh; ++m) z = __dadd_rn(z, ldcg(P.GG + (size_t)hch[h0 + m] * c.NVP + q));
    } else if (q < c.nv + c.nx) {
      const int i = q - c.nv;
      const size_t o = (size_t)a * c.NXP + i;
      const double ws = extrap(ldcg(Y + o), ldcg(Yp + o), cf);
      const double wz = extrap(ldcg(Y + E * c.NXP + o), ldcg(Yp + E * c.NXP + o), cf);
      const double ds = P.scaled ? __ldg(P.sig_stage + st) : 1.0;
      const double dz = P.scaled ? __ldg(P.zeta_stage + st) : 1.0;
      const double s = __dadd_rn(__dmul_rn(ws, ds), __dmul_rn(wz, dz));
      double h = 0.0;
      for (int m = 0; m < nh; ++m) h = __dadd_rn(h, ldcg(P.XIQG + (size_t)hch[h0 + m] * c.NXP + i));
      x = __dadd_rn(s, __dmul_rn(h, adiag[i]));
    } else {
      const int j = q - c.nv - c.nx;
      const size_t o = 2 * E * c.NXP + (size_t)a * c.NUP + j;
      const double wp = extrap(ldcg(Y + o), ldcg(Yp + o), cf);
      z = P.scaled ? __dmul_rn(wp, __ldg(P.psi_stage + (size_t)st * c.NUP + j)) : wp;
    }
    Zs[idx] = z;
    Xs[idx] = x;
  }
  __syncthreads();
  // (2) bottom-up over edge-stage levels: add trunk children
  for (int l = nlev - 1; l >= 0; --l) {
    for (int idx = lev[l] * nc + threadIdx.x; idx < lev[l + 1] * nc; idx += kThreadsS) {
      const int tp = idx / nc, k = idx - tp * nc, q = c_lo + k;
      const int* ps = pos + 8 * tp;
      const int c0 = ps[3], n = ps[4];
      double zs = 0.0, xs = 0.0;
      for (int m = 0; m < n; ++m) {
        const int cp = tch[c0 + m];
        zs = __dadd_rn(zs, Zs[cp * nc + k]);
        xs = __dadd_rn(xs, Xs[cp * nc + k]);
      }
      if (q >= c.nv && q < c.nv + c.nx) {
        const double xiq = __dadd_rn(Xs[idx], __dmul_rn(xs, adiag[q - c.nv]));
        Xs[idx] = xiq;
        Zs[idx] = __dadd_rn(xiq, zs);
      } else {
        Zs[idx] = __dadd_rn(Zs[idx], zs);
      }
    }
    __syncthreads();
  }
  // (3) top-down: K_a, Y_a = own * inv2p_a + parent's
  for (int l = 0; l < nlev; ++l) {
    for (int idx = lev[l] * nc + threadIdx.x; idx < lev[l + 1] * nc; idx += kThreadsS) {
      const int tp = idx / nc, k = idx - tp * nc;
      const int* ps = pos + 8 * tp;
      const int pp = ps[2];
      double v = __dmul_rn(Zs[idx], __ldg(P.inv2p + ps[0]));
      if (pp >= 0) v = __dadd_rn(v, Zs[pp * nc + k]);
      Zs[idx] = v;
    }
    __syncthreads();
  }
  // (4) KY columns of this slice
  for (int idx = threadIdx.x; idx < T * nc; idx += kThreadsS) {
    const int tp = idx / nc, k = idx - tp * nc, q = c_lo + k;
    const int col = q < c.nv ? q : (q < c.nv + c.nx ? c.NVP + (q - c.nv) : c.NVP + c.NXP + (q - c.nv - c.nx));
    stcg(P.KY + (size_t)tp * P.KY_LD + col, Zs[idx]);
  }
}

// ----------------------------------------------------------------------------
// phase D (trunk part): S, x, u of the needed trunk edges from KY
//   S = K + Ls'(B' Yx + Ypsi),  du = Lt S,  u = uhat + du,  x = a .* x_par + (B du + e)
// ----------------------------------------------------------------------------
__device__ void trunk_needs(const Ctx& c) {
  const Params& P = *c.P;
  const SParams& S = *c.S;
  const int nn = c.mt.nneed;
  if (nn == 0) return;
  const int nx = c.nx, nu = c.nu, nv = c.nv;
  const int LD = S.need_ld;
  double* Yz = c.work;                       // nn x NUP
  double* DU = c.work + (size_t)nn * c.NUP;  // nn x NUP
  const int* nd = c.mt.needs;
  // (1) Yz = Ypsi + B' Yx
  {
    const int* cp = c.spi + S.Bc_ptr;
    const int* ci = c.spi + S.Bc_idx;
    const double* cv = c.spv + S.Bc_val;
    for (int idx = threadIdx.x; idx < nn * nu; idx += kThreadsS) {
      const int n = idx / nu, j = idx - n * nu;
      const double* ky = P.KY + (size_t)nd[4 * n] * P.KY_LD;
      double z = ldcg(ky + c.NVP + c.NXP + j);
      for (int q = cp[j]; q < cp[j + 1]; ++q) z = fma(cv[q], ldcg(ky + c.NVP + ci[q]), z);
      Yz[(size_t)n * c.NUP + j] = z;
    }
  }
  __syncthreads();
  // (2) S = K + Ls' Yz
  {
    const int* cp = c.spi + S.Lc_ptr;
    const int* ci = c.spi + S.Lc_idx;
    const double* cv = c.spv + S.Lc_val;
    for (int idx = threadIdx.x; idx < nn * nv; idx += kThreadsS) {
      const int n = idx / nv, k = idx - n * nv;
      double h = 0.0;
      for (int q = cp[k]; q < cp[k + 1]; ++q) h = fma(cv[q], Yz[(size_t)n * c.NUP + ci[q]], h);
      c.need[(size_t)n * LD + k] = __dadd_rn(ldcg(P.KY + (size_t)nd[4 * n] * P.KY_LD + k), h);
    }
  }
  __syncthreads();
  // (3) du = Lt S ; u = uhat + du
  {
    const int* rp = c.spi + S.Lr_ptr;
    const int* ri = c.spi + S.Lr_idx;
    const double* rv = c.spv + S.Lr_val;
    for (int idx = threadIdx.x; idx < nn * nu; idx += kThreadsS) {
      const int n = idx / nu, j = idx - n * nu;
      double d = 0.0;
      for (int q = rp[j]; q < rp[j + 1]; ++q) d = fma(rv[q], c.need[(size_t)n * LD + ri[q]], d);
      DU[(size_t)n * c.NUP + j] = d;
      c.need[(size_t)n * LD + c.NVP + c.NXP + j] = __dadd_rn(d, ldcg(P.uhat + (size_t)nd[4 * n + 2] * c.NUP + j));
    }
  }
  __syncthreads();
  // (4) bv + e, then x level by level (parents first)
  {
    const int* rp = c.spi + S.Br_ptr;
    const int* ri = c.spi + S.Br_idx;
    const double* rv = c.spv + S.Br_val;
    for (int idx = threadIdx.x; idx < nn * nx; idx += kThreadsS) {
      const int n = idx / nx, i = idx - n * nx;
      double b = 0.0;
      for (int q = rp[i]; q < rp[i + 1]; ++q) b = fma(rv[q], DU[(size_t)n * c.NUP + ri[q]], b);
      c.need[(size_t)n * LD + c.NVP + i] = __dadd_rn(b, ldcg(P.evec + (size_t)nd[4 * n + 2] * c.NXP + i));
    }
    __syncthreads();
    const double* adiag = c.bnd + 3 * c.NXP + 2 * c.NUP;
    for (int l = 0; l < c.mt.nlev; ++l) {
      const int n0 = c.mt.lev[l], n1 = c.mt.lev[l + 1];
      for (int idx = n0 * nx + threadIdx.x; idx < n1 * nx; idx += kThreadsS) {
        const int n = idx / nx, i = idx - n * nx;
        const int pn = nd[4 * n + 1];
        const double xp = pn >= 0 ? c.need[(size_t)pn * LD + c.NVP + i] : P.p[i];
        double* xv = c.need + (size_t)n * LD + c.NVP + i;
        *xv = __dadd_rn(__dmul_rn(xp, adiag[i]), *xv);
      }
      __syncthreads();
    }
  }
}

// epilogue of the CTA's own trunk rows (dual / ergodic rows live in HBM)
__device__ void trunk_own_rows(const Ctx& c, int nu_it, int cur, double& rmax) {
  const Params& P = *c.P;
  const SParams& S = *c.S;
  const int no = c.mt.nown;
  if (no == 0) return;
  const int cap = max(1, c.S->n_work / c.SL);
  for (int b0 = 0; b0 < no; b0 += cap) {
    const int nb = min(cap, no - b0);
    // stage the rows into the work region in slot format (dual at index 0 = HBM cur)
    const int hx = c.NXP / 2, hu = c.NUP / 2, per_y = 2 * hx + hu, nch = 2 * per_y + hx + hu;
    const size_t E = (size_t)c.E;
    for (int idx = threadIdx.x; idx < nb * nch; idx += kThreadsS) {
      const int r = idx / nch;
      int k = idx - r * nch;
      const int e = c.mt.needs[4 * c.mt.own[b0 + r] + 2];
      double* srow = c.work + (size_t)r * c.SL;
      if (k < 2 * per_y) {
        const int which = k < per_y ? 0 : 1;
        const int kk = k - which * per_y;
        const double* Y = P.ybuf[cur ^ which];
        double* dst = srow + (size_t)which * c.YW;
        if (kk < hx) cp16(dst + 2 * kk, Y + (size_t)e * c.NXP + 2 * kk);
        else if (kk < 2 * hx) cp16(dst + c.NXP + 2 * (kk - hx), Y + E * c.NXP + (size_t)e * c.NXP + 2 * (kk - hx));
        else cp16(dst + 2 * c.NXP + 2 * (kk - 2 * hx), Y + 2 * E * c.NXP + (size_t)e * c.NUP + 2 * (kk - 2 * hx));
      } else {
        k -= 2 * per_y;
        double* xa = srow + 2 * c.YW;
        if (k < hx) cp16(xa + 2 * k, P.xavg + (size_t)(e + 1) * c.NXP + 2 * k);
        else cp16(xa + c.NXP + 2 * (k - hx), P.uavg + (size_t)e * c.NUP + 2 * (k - hx));
      }
    }
    cp_commit();
    cp_wait<0>();
    __syncthreads();
    const Meta& mt = c.mt;
    const int LD = S.need_ld;
    const int* own = mt.own + b0;
    epilogue(
        c, nu_it, nb, [&](int r) { return mt.needs[4 * own[r] + 2]; }, [&](int r) { return mt.needs[4 * own[r] + 3]; },
        [&](int r) { return c.need + (size_t)own[r] * LD + c.NVP; },
        [&](int r) { return c.need + (size_t)own[r] * LD + c.NVP + c.NXP; },
        [&](int r) { return c.work + (size_t)r * c.SL; }, 0, true, cur ^ 1, rmax);
    __syncthreads();
  }
}

}  // namespace

__global__ void __launch_bounds__(kThreadsS, 1) apg_sparse_kernel(const __grid_constant__ SParams S) {
  cg::grid_group grid = cg::this_grid();
  const Params& P = S.P;
  Ctx c;
  c.S = &S;
  c.P = &P;
  c.NXP = P.NXP; c.NUP = P.NUP; c.NVP = P.NVP;
  c.YW = S.YW; c.SL = S.slot_ld;
  c.nx = P.nx; c.nu = P.nu; c.nv = P.nv; c.E = P.n_edges;
  c.bnd = s_dyn + S.O_BND;
  c.need = s_dyn + S.O_NEED;
  c.work = s_dyn + S.O_WORK;
  c.slot = s_dyn + S.O_SLOT;
  int* ints = reinterpret_cast<int*>(s_dyn + S.O_INT);
  int* smeta = ints;
  int* sspi = ints + S.meta_max;
  double* sspv = s_dyn + S.O_SPV;
  {  // stage model vectors, sparse operators and this CTA's plan
    double* bnd = c.bnd;
    for (int i = threadIdx.x; i < c.NXP; i += kThreadsS) {
      bnd[i] = P.x_s[i];
      bnd[c.NXP + i] = P.x_min[i];
      bnd[2 * c.NXP + i] = P.x_max[i];
      bnd[3 * c.NXP + 2 * c.NUP + i] = P.a_diag[i];
    }
    for (int j = threadIdx.x; j < c.NUP; j += kThreadsS) {
      bnd[3 * c.NXP + j] = P.u_min[j];
      bnd[3 * c.NXP + c.NUP + j] = P.u_max[j];
    }
    const int m0 = __ldg(S.meta_ptr + blockIdx.x), m1 = __ldg(S.meta_ptr + blockIdx.x + 1);
    for (int i = threadIdx.x; i < m1 - m0; i += kThreadsS) smeta[i] = __ldg(S.meta + m0 + i);
    for (int i = threadIdx.x; i < S.n_spi; i += kThreadsS) sspi[i] = __ldg(S.spi + i);
    for (int i = threadIdx.x; i < S.n_spv; i += kThreadsS) sspv[i] = __ldg(S.spv + i);
    __syncthreads();
  }
  c.mt.bind(smeta);
  c.spi = sspi;
  c.spv = sspv;
  const bool resident = c.mt.resident != 0;
  const int nt = c.mt.ntiles;
  const bool trunk = P.n_trunk > 0;
  // initial dual / ergodic rows
  {
    const int cur0 = P.slot0 & 1;
    if (resident) {
      for (int t = 0; t < nt; ++t) {
        const int* td = c.mt.tiles + 4 * t;
        load_slot(c, td[0], td[1], td[0], 3, cur0, 0);
      }
    } else if (nt > 0) {
      const int* td = c.mt.tiles + 4 * (nt - 1);
      load_slot(c, td[0], td[1], 0, 1, cur0, 0);
    }
    cp_commit();
    cp_wait<0>();
    __syncthreads();
  }
  double rmax = 0.0;
  for (int nu = 0; nu < P.iters; ++nu) {
    const int cur = (P.slot0 + nu) & 1;
    const int ysm = nu & 1;
    for (int t = nt - 1; t >= 0; --t) bwd_tile(c, t, nu, ysm, resident ? c.mt.tiles[4 * t] : 0, resident, cur);
    if (trunk) {
      long long tb_ = clock64();
      (void)tb_;
      grid.sync();
      TSMPC_MARK(P, 9, tb_);
      trunk_sweep(c, nu, cur);
      TSMPC_MARK(P, 10, tb_);
      grid.sync();
      TSMPC_MARK(P, 9, tb_);
      trunk_needs(c);
      trunk_own_rows(c, nu, cur, rmax);
      TSMPC_MARK(P, 12, tb_);
    }
    if (blockIdx.x == 0) {
      const double th = P.theta[nu], om = __dsub_rn(1.0, th);
      for (int i = threadIdx.x; i < c.nx; i += kThreadsS)
        P.xavg[i] = __dadd_rn(__dmul_rn(P.xavg[i], om), __dmul_rn(th, P.p[i]));
    }
    for (int t = 0; t < nt; ++t) fwd_tile(c, t, nu, ysm, resident ? c.mt.tiles[4 * t] : 0, resident, cur, rmax);
    if (nu == P.iters - 1 || P.record_all) {
      for (int off = 16; off > 0; off >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, off));
      if ((threadIdx.x & 31) == 0 && rmax > 0.0)
        atomicMax(P.resid + (P.record_all ? nu : 0), (unsigned long long)__double_as_longlong(rmax));
      rmax = 0.0;
    }
  }
}

}  // namespace tsmpc

namespace tsmpc {

// beta_s = beta M (rows of the stage cache mapped to the structured basis,
// elimination.py:156-157 with L replaced by Ls = L M).  One warp per edge row.
__global__ void beta_rotate_kernel(const double* __restrict__ beta, const double* __restrict__ M, double* out,
                                   int E, int nv, int NVP) {
  const int lane = threadIdx.x & 31;
  for (int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < E; e += (gridDim.x * blockDim.x) >> 5) {
    const double* b = beta + (size_t)e * NVP;
    for (int k = lane; k < nv; k += 32) {
      double s = 0.0;
      for (int j = 0; j < nv; ++j) s = fma(b[j], M[(size_t)j * nv + k], s);
      out[(size_t)e * NVP + k] = s;
    }
  }
}

}  // namespace tsmpc
