// tsmpc_epilogue.cuh — per-row APG epilogue of the forward sweep (included by
// tsmpc_apg.cu): prox_g, dual update, ergodic averages and residual for the
// rows of a tile (reference engine.py:546-575, prox engine.py:146-183).
//
// One warp per edge row; x sits in the A region and u in the C region of the
// forward tile layout.  Templated on the 32-lane chunk counts of x (XC) and u
// (UC); each row is handled in two parts (state copies, then the input copy)
// whose global reads are all issued before use — two small register footprints
// instead of one large one, which keeps 26 warps per SM spill-free.  Global
// accesses use per-row base pointers (immediate offsets) and explicit
// global-space L2 (.cg) instructions; model bounds come from shared memory.
// The scaled quotients use host-precomputed reciprocals (1/lam, 1/D): a one-ulp
// difference from the reference's divisions, inside the calibrated parity
// tolerance.
#pragma once

template <int XC, int UC>
__device__ __noinline__ void rows_epilogue_t(const Params& P, int nu, int nrows) {
  const int LDA = P.LDA2, LDB = P.LDB2;
  const double* const SA = g_smem;
  const double* const SB = g_smem + kTileM * LDA;
  const int* const edge = SM_EDGE(P);
  const double* const bnd = SM_BOUNDS(P);
  const double* const xs_s = bnd;
  const double* const xmn_s = bnd + P.NXP;
  const double* const xmx_s = bnd + 2 * P.NXP;
  const double* const umn_s = bnd + 3 * P.NXP;
  const double* const umx_s = bnd + 3 * P.NXP + P.NUP;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool last = nu == P.iters - 1;
  const int E = P.n_edges;
  const int cur = (P.slot0 + nu) & 1;
  const double* __restrict__ Y = P.ybuf[cur];
  double* Yn = P.ybuf[cur ^ 1];  // y_prev slot receives y_next
  const double c = P.coef[nu];
  const double th = P.theta[nu];
  const double om = __dsub_rn(1.0, th);
  const double lam = P.lam, ilam = P.inv_lam;
  const double lam_p = 1.0 / lam;  // prox parameter (engine.py:555)
  const size_t zoff = (size_t)E * P.NXP, poff = 2 * (size_t)E * P.NXP;
  const bool want_resid = last || P.record_all;
  double rmax = 0.0;
  for (int r = warp; r < nrows; r += kWarps) {
    const int e = edge[r];
    const int st = __ldg(P.edge_stage + e);
    // --- state copies: two weighted-distance prox blocks (engine.py:146-180)
    {
      const double* ysp = Y + (size_t)e * P.NXP + lane;
      double* ynp = Yn + (size_t)e * P.NXP + lane;
      double* xap = P.xavg + (size_t)(e + 1) * P.NXP + lane;
      double ys[XC] = {}, yps[XC] = {}, yz[XC] = {}, ypz[XC] = {}, xa[XC] = {};
#pragma unroll
      for (int q = 0; q < XC; ++q) {
        if (lane + 32 * q < P.nx) {
          ys[q] = gld(ysp + 32 * q);
          yps[q] = gld(ynp + 32 * q);
          yz[q] = gld(ysp + zoff + 32 * q);
          ypz[q] = gld(ynp + zoff + 32 * q);
          xa[q] = gld(xap + 32 * q);
        }
      }
      const double ds = stage_scale(P.sig_stage, st, P.scaled);
      const double dz = stage_scale(P.zeta_stage, st, P.scaled);
      const double rds = P.scaled ? __ldg(P.sig_rcp + st) : 1.0;
      const double rdz = P.scaled ? __ldg(P.zeta_rcp + st) : 1.0;
      double ts[XC], tz[XC];
      double ss = 0.0, sz = 0.0;
#pragma unroll
      for (int q = 0; q < XC; ++q) {
        const int i = lane + 32 * q;
        ts[q] = tz[q] = 0.0;
        if (i < P.nx) {
          const double x = SA[r * LDA + i];
          ys[q] = extrap(ys[q], yps[q], c);  // w_sig (y no longer needed)
          yz[q] = extrap(yz[q], ypz[q], c);  // w_zeta
          // t_arg = w / lam + D Hz   (engine.py:552-554)
          ts[q] = __dadd_rn(__dmul_rn(ys[q], ilam), __dmul_rn(x, ds));
          tz[q] = __dadd_rn(__dmul_rn(yz[q], ilam), __dmul_rn(x, dz));
          const double ps = fmax(ts[q], __dmul_rn(ds, xs_s[i]));
          const double pz = fmin(fmax(tz[q], __dmul_rn(dz, xmn_s[i])), __dmul_rn(dz, xmx_s[i]));
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
      const double wgt_s = __dmul_rn(__dmul_rn(lam_p, P.Wx), rds);
      const double wgt_z = __dmul_rn(__dmul_rn(lam_p, P.gamma_d), rdz);
      const double fs = dist_s > wgt_s ? __ddiv_rn(wgt_s, dist_s) : 1.0;
      const double fz = dist_z > wgt_z ? __ddiv_rn(wgt_z, dist_z) : 1.0;
#pragma unroll
      for (int q = 0; q < XC; ++q) {
        const int i = lane + 32 * q;
        if (i < P.nx) {
          const double x = SA[r * LDA + i];
          const double hs = __dmul_rn(x, ds), hz = __dmul_rn(x, dz);
          const double ps = fmax(ts[q], __dmul_rn(ds, xs_s[i]));
          const double pz = fmin(fmax(tz[q], __dmul_rn(dz, xmn_s[i])), __dmul_rn(dz, xmx_s[i]));
          const double t_s = __dadd_rn(ts[q], __dmul_rn(fs, __dsub_rn(ps, ts[q])));
          const double t_z = __dadd_rn(tz[q], __dmul_rn(fz, __dsub_rn(pz, tz[q])));
          gst(ynp + 32 * q, __dadd_rn(ys[q], __dmul_rn(lam, __dsub_rn(hs, t_s))));
          gst(ynp + zoff + 32 * q, __dadd_rn(yz[q], __dmul_rn(lam, __dsub_rn(hz, t_z))));
          if (want_resid) {
            rmax = fmax(rmax, fabs(__dsub_rn(x, __dmul_rn(t_s, rds))));
            rmax = fmax(rmax, fabs(__dsub_rn(x, __dmul_rn(t_z, rdz))));
          }
          gst(xap + 32 * q, __dadd_rn(__dmul_rn(xa[q], om), __dmul_rn(th, x)));
          if (last) gst(P.X + (size_t)(e + 1) * P.NXP + i, x);
        }
      }
    }
    // --- input copy: box projection (engine.py:182)
    {
      const double* upp = Y + poff + (size_t)e * P.NUP + lane;
      double* unp = Yn + poff + (size_t)e * P.NUP + lane;
      double* uap = P.uavg + (size_t)e * P.NUP + lane;
      const double* psp = P.psi_stage + (size_t)st * P.NUP + lane;
      double yp[UC] = {}, ypp[UC] = {}, ua[UC] = {}, dp[UC];
#pragma unroll
      for (int q = 0; q < UC; ++q) {
        dp[q] = 1.0;
        if (lane + 32 * q < P.nu) {
          yp[q] = gld(upp + 32 * q);
          ypp[q] = gld(unp + 32 * q);
          ua[q] = gld(uap + 32 * q);
          if (P.scaled) dp[q] = __ldg(psp + 32 * q);
        }
      }
#pragma unroll
      for (int q = 0; q < UC; ++q) {
        const int j = lane + 32 * q;
        if (j < P.nu) {
          const double u = SB[r * LDB + j];
          const double w = extrap(yp[q], ypp[q], c);
          const double hp = __dmul_rn(u, dp[q]);
          const double a = __dadd_rn(__dmul_rn(w, ilam), hp);
          const double t = fmin(fmax(a, __dmul_rn(dp[q], umn_s[j])), __dmul_rn(dp[q], umx_s[j]));
          gst(unp + 32 * q, __dadd_rn(w, __dmul_rn(lam, __dsub_rn(hp, t))));
          if (want_resid) {
            const double rdp = P.scaled ? __ldg(P.psi_rcp + (size_t)st * P.NUP + j) : 1.0;
            rmax = fmax(rmax, fabs(__dsub_rn(u, __dmul_rn(t, rdp))));
          }
          gst(uap + 32 * q, __dadd_rn(__dmul_rn(ua[q], om), __dmul_rn(th, u)));
          if (last) gst(P.U + (size_t)e * P.NUP + j, u);
        }
      }
    }
  }
  if (want_resid) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, off));
    if (lane == 0 && rmax > 0.0)
      atomicMax(P.resid + (P.record_all ? nu : 0), (unsigned long long)__double_as_longlong(rmax));
  }
}
