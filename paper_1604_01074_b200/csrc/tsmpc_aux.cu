// tsmpc_aux.cu — per-edge kernels around the persistent APG loop:
//   prox_g as a standalone operator        (engine.py:146-183)
//   dual-gradient operator for compute_lambda's power iteration (engine.py:286-337)
//   duality gap                            (engine.py:347-480)
//   deterministic fixed-order reductions (bitwise run-to-run reproducible sums)
// All kernels use one warp per edge row; rows are at most 128 wide (4 per lane).
#include "tsmpc_aux.cuh"

namespace cg = cooperative_groups;

namespace tsmpc {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}
__device__ __forceinline__ double clip(double v, double lo, double hi) { return fmin(fmax(v, lo), hi); }

// ---------------------------------------------------------------- reductions
// out[c] = sum_i vals[i * ncols + c], fixed order (one block, 1024 threads).
__global__ void __launch_bounds__(1024) reduce_cols_kernel(const double* __restrict__ vals, int n,
                                                           int ncols, double* __restrict__ out) {
  __shared__ double red[1024];
  for (int c = 0; c < ncols; ++c) {
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += 1024) s += vals[(size_t)i * ncols + c];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = 512; w > 0; w >>= 1) {
      if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[c] = red[0];
    __syncthreads();
  }
}

// ---------------------------------------------------------------- prox_g
__global__ void prox_kernel(ProxArgs a) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = gw; r < a.rows; r += nw) {
    const int st = a.edge_stage ? a.edge_stage[r] : 0;
    const double ds = a.sig_stage ? a.sig_stage[st] : 1.0;
    const double dz = a.zeta_stage ? a.zeta_stage[st] : 1.0;
    double ss = 0.0, sz = 0.0;
    for (int i = lane; i < a.nx; i += 32) {
      const double ts = a.t_sig[(size_t)r * a.nx + i], tz = a.t_zeta[(size_t)r * a.nx + i];
      const double gs = fmax(ts, ds * a.x_s[i]) - ts;
      const double gz = clip(tz, dz * a.x_min[i], dz * a.x_max[i]) - tz;
      ss = fma(gs, gs, ss);
      sz = fma(gz, gz, sz);
    }
    ss = warp_sum(ss);
    sz = warp_sum(sz);
    const double ws = a.lam * a.Wx / ds, wz = a.lam * a.gamma_d / dz;
    const double ds_ = sqrt(ss), dz_ = sqrt(sz);
    const double fs = ds_ > ws ? ws / ds_ : 1.0, fz = dz_ > wz ? wz / dz_ : 1.0;
    for (int i = lane; i < a.nx; i += 32) {
      const size_t o = (size_t)r * a.nx + i;
      const double ts = a.t_sig[o], tz = a.t_zeta[o];
      a.o_sig[o] = ts + fs * (fmax(ts, ds * a.x_s[i]) - ts);
      a.o_zeta[o] = tz + fz * (clip(tz, dz * a.x_min[i], dz * a.x_max[i]) - tz);
    }
    for (int j = lane; j < a.nu; j += 32) {
      const size_t o = (size_t)r * a.nu + j;
      const double dp = a.psi_stage ? a.psi_stage[(size_t)st * a.nu + j] : 1.0;
      a.o_psi[o] = clip(a.t_psi[o], dp * a.u_min[j], dp * a.u_max[j]);
    }
  }
}

// ---------------------------------------------------------------- power iteration
// rows[e] = (sum y_sig^2, sum y_zeta^2, sum y_psi^2)
__global__ void dual_sq_rows_kernel(EdgeCtx c, const double* __restrict__ y, double* rows) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const size_t zoff = (size_t)c.E * c.NXP, poff = 2 * zoff;
  for (int e = gw; e < c.E; e += nw) {
    double s = 0, z = 0, p = 0;
    for (int i = lane; i < c.nx; i += 32) {
      const double a = y[(size_t)e * c.NXP + i], b = y[zoff + (size_t)e * c.NXP + i];
      s = fma(a, a, s);
      z = fma(b, b, z);
    }
    for (int j = lane; j < c.nu; j += 32) {
      const double a = y[poff + (size_t)e * c.NUP + j];
      p = fma(a, a, p);
    }
    s = warp_sum(s); z = warp_sum(z); p = warp_sum(p);
    if (lane == 0) { rows[3 * e] = s; rows[3 * e + 1] = z; rows[3 * e + 2] = p; }
  }
}

// y /= sqrt(sq[0] + sq[1] + sq[2])
__global__ void dual_normalize_kernel(EdgeCtx c, double* y, const double* sq) {
  const double norm = sqrt((sq[0] + sq[1]) + sq[2]);
  const size_t n = 2 * (size_t)c.E * c.NXP + (size_t)c.E * c.NUP;
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x)
    y[k] = y[k] / norm;
}

// Dy = S (z0 - H z);  rows[e] = (<y,Dy> by block, <Dy,Dy> by block); y <- Dy
__global__ void dual_apply_kernel(EdgeCtx c, double* y, const double* __restrict__ X,
                                  const double* __restrict__ U, const double* __restrict__ Z0X,
                                  const double* __restrict__ Z0U, double* rows) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const size_t zoff = (size_t)c.E * c.NXP, poff = 2 * zoff;
  for (int e = gw; e < c.E; e += nw) {
    const int st = c.edge_stage[e];
    const double ds = c.sig_stage ? c.sig_stage[st] : 1.0;
    const double dz = c.zeta_stage ? c.zeta_stage[st] : 1.0;
    double a[6] = {0, 0, 0, 0, 0, 0};
    for (int i = lane; i < c.nx; i += 32) {
      const size_t ox = (size_t)(e + 1) * c.NXP + i, o = (size_t)e * c.NXP + i;
      const double d = Z0X[ox] - X[ox];
      const double dsg = d * ds, dzt = d * dz;
      a[0] = fma(y[o], dsg, a[0]);
      a[1] = fma(y[zoff + o], dzt, a[1]);
      a[3] = fma(dsg, dsg, a[3]);
      a[4] = fma(dzt, dzt, a[4]);
      y[o] = dsg;
      y[zoff + o] = dzt;
    }
    for (int j = lane; j < c.nu; j += 32) {
      const size_t o = (size_t)e * c.NUP + j;
      const double dp = c.psi_stage ? c.psi_stage[(size_t)st * c.NUP + j] : 1.0;
      const double d = (Z0U[o] - U[o]) * dp;
      a[2] = fma(y[poff + o], d, a[2]);
      a[5] = fma(d, d, a[5]);
      y[poff + o] = d;
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) a[k] = warp_sum(a[k]);
    if (lane == 0)
      for (int k = 0; k < 6; ++k) rows[6 * (size_t)e + k] = a[k];
  }
}

// ---------------------------------------------------------------- duality gap
// Dual side, part 1: y_hat = projection of the unscaled dual onto dom g*, plus
// the conjugate terms (engine.py:435-455).  cols[e*10 + 7..9].
__global__ void gap_dual_project_kernel(EdgeCtx c, const double* __restrict__ y, double* what,
                                        double* cols) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const size_t zoff = (size_t)c.E * c.NXP, poff = 2 * zoff;
  for (int e = gw; e < c.E; e += nw) {
    const int st = c.edge_stage[e];
    const double ds = c.sig_stage ? c.sig_stage[st] : 1.0;
    const double dz = c.zeta_stage ? c.zeta_stage[st] : 1.0;
    double ns = 0, nz = 0;
    for (int i = lane; i < c.nx; i += 32) {
      const size_t o = (size_t)e * c.NXP + i;
      const double s = fmin(y[o] * ds, 0.0), z = y[zoff + o] * dz;
      ns = fma(s, s, ns);
      nz = fma(z, z, nz);
    }
    ns = sqrt(warp_sum(ns));
    nz = sqrt(warp_sum(nz));
    const double fs = ns > c.Wx ? c.Wx / ns : 1.0;
    const double fz = nz > c.gamma_d ? c.gamma_d / nz : 1.0;
    const bool os = ns > c.Wx, oz = nz > c.gamma_d;
    double k7 = 0, k8 = 0, k9 = 0;
    for (int i = lane; i < c.nx; i += 32) {
      const size_t o = (size_t)e * c.NXP + i;
      double s = fmin(y[o] * ds, 0.0), z = y[zoff + o] * dz;
      if (os) s *= fs;
      if (oz) z *= fz;
      what[o] = s;
      what[zoff + o] = z;
      k7 = fma(s, c.x_s[i], k7);
      k8 += z > 0 ? z * c.x_max[i] : z * c.x_min[i];
    }
    for (int j = lane; j < c.nu; j += 32) {
      const size_t o = (size_t)e * c.NUP + j;
      const double dp = c.psi_stage ? c.psi_stage[(size_t)st * c.NUP + j] : 1.0;
      const double p = y[poff + o] * dp;
      what[poff + o] = p;
      k9 += p > 0 ? p * c.u_max[j] : p * c.u_min[j];
    }
    k7 = warp_sum(k7); k8 = warp_sum(k8); k9 = warp_sum(k9);
    if (lane == 0) {
      cols[10 * (size_t)e + 7] = k7;
      cols[10 * (size_t)e + 8] = k8;
      cols[10 * (size_t)e + 9] = k9;
    }
  }
}

// p_e (W_alpha price_stage . u_e + du' Wu du), du = u_e - u_parent (or q).
__device__ double smooth_term(const EdgeCtx& c, int e, const double* U, int ldu, double* sh) {
  const int lane = threadIdx.x & 31;
  const int st = c.edge_stage[e];
  const int pa = c.anc[e + 1] - 1;
  double econ = 0.0;
  for (int j = lane; j < c.nu; j += 32) {
    const double u = U[(size_t)e * ldu + j];
    const double up = pa >= 0 ? U[(size_t)pa * ldu + j] : c.q[j];
    sh[j] = u - up;
    econ = fma(c.prices[(size_t)st * c.nu + j], u, econ);
  }
  __syncwarp();
  double quad = 0.0;
  for (int j = lane; j < c.nu; j += 32) {
    double wd = 0.0;  // non-zeros of row j of Wu, ascending columns (diagonal for water networks)
    for (int q = c.wu_ptr[j]; q < c.wu_ptr[j + 1]; ++q) wd = fma(c.wu_val[q], sh[c.wu_idx[q]], wd);
    quad = fma(sh[j], wd, quad);
  }
  __syncwarp();
  econ = warp_sum(econ);
  quad = warp_sum(quad);
  return c.prob_edge[e] * (c.W_alpha * econ + quad);
}

// Dual side, part 2 (after the solve step at y_hat): pairing <H z, y_hat> and the
// smooth cost of z_hat.u (engine.py:474-479).  cols[e*10 + 3..6].
__global__ void gap_dual_terms_kernel(EdgeCtx c, const double* __restrict__ what,
                                      const double* __restrict__ X, const double* __restrict__ U,
                                      double* cols) {
  __shared__ double shm[8][128];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const size_t zoff = (size_t)c.E * c.NXP, poff = 2 * zoff;
  for (int e = gw; e < c.E; e += nw) {
    double k3 = 0, k4 = 0, k5 = 0;
    for (int i = lane; i < c.nx; i += 32) {
      const double x = X[(size_t)(e + 1) * c.NXP + i];
      k3 = fma(x, what[(size_t)e * c.NXP + i], k3);
      k4 = fma(x, what[zoff + (size_t)e * c.NXP + i], k4);
    }
    for (int j = lane; j < c.nu; j += 32) k5 = fma(U[(size_t)e * c.NUP + j], what[poff + (size_t)e * c.NUP + j], k5);
    k3 = warp_sum(k3); k4 = warp_sum(k4); k5 = warp_sum(k5);
    const double k6 = smooth_term(c, e, U, c.NUP, shm[wl]);
    if (lane == 0) {
      cols[10 * (size_t)e + 3] = k3;
      cols[10 * (size_t)e + 4] = k4;
      cols[10 * (size_t)e + 5] = k5;
      cols[10 * (size_t)e + 6] = k6;
    }
  }
}

// Primal side, part 1 (n_e == 1): exact multiplier bisection (engine.py:383-405).
__device__ __forceinline__ double balance1(const EdgeCtx& c, const double* u, double mu) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int j = lane; j < c.nu; j += 32) {
    const double a = c.Ej[j];
    s = fma(clip(u[j] - mu * a, c.u_min[j], c.u_max[j]), a, s);
  }
  return warp_sum(s);
}

__global__ void gap_project_bisect_kernel(EdgeCtx c, const double* __restrict__ uavg, double* uf) {
  __shared__ double shm[8][128];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  double* u = shm[wl];
  for (int e = gw; e < c.E; e += nw) {
    for (int j = lane; j < c.nu; j += 32) u[j] = uavg[(size_t)e * c.NUP + j];
    __syncwarp();
    const double b = c.jrhs[(size_t)e * c.ne];
    double lo = -1.0, hi = 1.0;
    for (int it = 0; it < 60; ++it) {
      const bool need = balance1(c, u, lo) < b;
      const bool high = balance1(c, u, hi) > b;
      if (!need && !high) break;
      if (need) lo *= 2.0;
      if (high) hi *= 2.0;
    }
    for (int it = 0; it < 80; ++it) {
      const double mid = 0.5 * (lo + hi);
      const bool th = balance1(c, u, mid) > b;
      lo = th ? mid : lo;
      hi = th ? hi : mid;
    }
    const double mu = 0.5 * (lo + hi);
    for (int j = lane; j < c.nu; j += 32)
      uf[(size_t)e * c.NUP + j] = clip(u[j] - mu * c.Ej[j], c.u_min[j], c.u_max[j]);
    __syncwarp();
  }
}

// ya = x - (x E' - target) pinv'   (per warp; r in shared scratch)
__device__ __forceinline__ void affine_project(const EdgeCtx& c, const double* x, const double* tgt,
                                               double* r, double* ya) {
  const int lane = threadIdx.x & 31;
  for (int k = 0; k < c.ne; ++k) {
    double s = 0.0;
    for (int j = lane; j < c.nu; j += 32) s = fma(x[j], c.Emat[(size_t)k * c.nu + j], s);
    s = warp_sum(s);
    if (lane == 0) r[k] = s - tgt[k];
  }
  __syncwarp();
  for (int j = lane; j < c.nu; j += 32) {
    double s = 0.0;
    for (int k = 0; k < c.ne; ++k) s = fma(r[k], c.EpinvT[(size_t)k * c.nu + j], s);
    ya[j] = x[j] - s;
  }
  __syncwarp();
}

// Primal side, part 1 (n_e > 1): Dykstra between the junction plane and the box
// (engine.py:407-419).  Cooperative: the stopping test is a max over every edge.
__global__ void __launch_bounds__(256) gap_project_dykstra_kernel(EdgeCtx c, double* xit, double* inc,
                                                                  double* uf,
                                                                  unsigned long long* slots) {
  __shared__ double sx[8][128], sy[8][128], sr[8][64];
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int it = 0; it < 200; ++it) {
    double mx = 0.0;
    for (int e = gw; e < c.E; e += nw) {
      double* x = sx[wl];
      for (int j = lane; j < c.nu; j += 32) x[j] = xit[(size_t)e * c.NUP + j];
      __syncwarp();
      affine_project(c, x, c.jrhs + (size_t)e * c.ne, sr[wl], sy[wl]);
      for (int j = lane; j < c.nu; j += 32) {
        const size_t o = (size_t)e * c.NUP + j;
        const double t = sy[wl][j] + inc[o];
        const double xn = clip(t, c.u_min[j], c.u_max[j]);
        inc[o] = t - xn;
        mx = fmax(mx, fabs(xn - x[j]));
        xit[o] = xn;
      }
      __syncwarp();
    }
    mx = warp_max(mx);
    if (lane == 0 && mx > 0.0) atomicMax(slots + it, (unsigned long long)__double_as_longlong(mx));
    grid.sync();
    const double gmax = __longlong_as_double((long long)*((volatile unsigned long long*)(slots + it)));
    if (gmax < 1e-13) break;
  }
  for (int e = gw; e < c.E; e += nw) {
    double* x = sx[wl];
    for (int j = lane; j < c.nu; j += 32) x[j] = xit[(size_t)e * c.NUP + j];
    __syncwarp();
    affine_project(c, x, c.jrhs + (size_t)e * c.ne, sr[wl], sy[wl]);
    for (int j = lane; j < c.nu; j += 32) uf[(size_t)e * c.NUP + j] = sy[wl][j];
    __syncwarp();
  }
}

// Dykstra without grid barriers (engine.py:407-419).  The reference stops every
// edge at the first sweep whose change, maxed over ALL edges, is < 1e-13.  Each
// edge's iterates do not depend on the others, so: pass 1 runs every edge's 200
// sweeps in shared memory and records the per-sweep max change (atomicMax into
// slots[it]); pass 2 finds the global stopping sweep K from slots and re-runs each
// edge for exactly K + 1 sweeps (or 200), then applies the final affine projection.
// The junction operators are sparse (a junction touches a few flows): E by row
// and E_pinv^T by column are staged in shared memory; warp per edge.
__global__ void __launch_bounds__(256) gap_dykstra_pass_kernel(EdgeCtx c, const double* __restrict__ u0,
                                                               unsigned long long* slots, int pass,
                                                               double* uf) {
  extern __shared__ double dsm[];
  // sparse E (rows) and E_pinv^T (columns) staged in shared memory
  double* ev = dsm;                                   // er_nnz
  double* pv = ev + c.er_nnz;                         // pc_nnz
  double* wsm = pv + c.pc_nnz + (c.pc_nnz + c.er_nnz & 1);  // 16-byte aligned per-warp scratch
  int* ei = reinterpret_cast<int*>(wsm + 8 * 448);    // er_ptr (ne+1) | er_idx | pc_ptr (nu+1) | pc_idx
  int* ep = ei;
  int* eix = ep + c.ne + 1;
  int* pp = eix + c.er_nnz;
  int* pix = pp + c.nu + 1;
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < c.er_nnz; i += blockDim.x) { ev[i] = c.er_val[i]; eix[i] = c.er_idx[i]; }
  for (int i = threadIdx.x; i < c.pc_nnz; i += blockDim.x) { pv[i] = c.pc_val[i]; pix[i] = c.pc_idx[i]; }
  for (int i = threadIdx.x; i <= c.ne; i += blockDim.x) ep[i] = c.er_ptr[i];
  for (int i = threadIdx.x; i <= c.nu; i += blockDim.x) pp[i] = c.pc_ptr[i];
  __syncthreads();
  // ya = x - (x E' - target) pinv'  (engine.py:409), non-zeros only, ascending order
  auto project = [&](const double* xx, const double* tgt, double* rr, double* ya) {
    for (int k = lane; k < c.ne; k += 32) {
      double s = 0.0;
      for (int q = ep[k]; q < ep[k + 1]; ++q) s = fma(xx[eix[q]], ev[q], s);
      rr[k] = s - tgt[k];
    }
    __syncwarp();
    for (int jj = lane; jj < c.nu; jj += 32) {
      double s = 0.0;
      for (int q = pp[jj]; q < pp[jj + 1]; ++q) s = fma(rr[pix[q]], pv[q], s);
      ya[jj] = xx[jj] - s;
    }
    __syncwarp();
  };
  double* x = wsm + (size_t)wl * 448;
  double* y = x + 128;
  double* r = y + 128;
  double* inc = r + 64;
  int n_it = 200;
  if (pass == 2) {
    for (int it = 0; it < 200; ++it) {
      const double g = __longlong_as_double((long long)slots[it]);
      if (g < 1e-13) { n_it = it + 1; break; }
    }
  }
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int e = gw; e < c.E; e += nw) {
    for (int j = lane; j < c.nu; j += 32) {
      x[j] = u0[(size_t)e * c.NUP + j];
      inc[j] = 0.0;
    }
    __syncwarp();
    const double* tgt = c.jrhs + (size_t)e * c.ne;
    for (int it = 0; it < n_it; ++it) {
      project(x, tgt, r, y);
      double mx = 0.0;
      for (int j = lane; j < c.nu; j += 32) {
        const double t = y[j] + inc[j];
        const double xn = clip(t, c.u_min[j], c.u_max[j]);
        inc[j] = t - xn;
        mx = fmax(mx, fabs(xn - x[j]));
        x[j] = xn;
      }
      __syncwarp();
      if (pass == 1) {
        mx = warp_max(mx);
        if (lane == 0 && mx > 0.0) atomicMax(slots + it, (unsigned long long)__double_as_longlong(mx));
      }
    }
    if (pass == 2) {
      project(x, tgt, r, y);
      for (int j = lane; j < c.nu; j += 32) uf[(size_t)e * c.NUP + j] = y[j];
      __syncwarp();
    }
  }
}

// Dykstra in lockstep (cooperative launch): the same iterates and stopping sweep
// as the two passes above, without running every edge for all 200 sweeps.  Edges
// advance kDykBlk sweeps at a time (state round-trips through st, two buffers of
// [x | inc] rows), recording the per-sweep max change; after each block one grid
// barrier makes slots[] final, and every thread reads the same stopping sweep K.
// The edges then restart from the state at the start of K's block and run the
// K + 1 - blk0 sweeps left before the final affine projection (as pass 2 would).
constexpr int kDykBlk = 8;
constexpr int kDykMax = 200;

__global__ void __launch_bounds__(256) gap_dykstra_coop_kernel(EdgeCtx c, const double* __restrict__ u0,
                                                               unsigned long long* slots, double* st,
                                                               double* uf) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double dsm[];
  __shared__ double wmax[8][kDykBlk];
  double* ev = dsm;
  double* pv = ev + c.er_nnz;
  double* wsm = pv + c.pc_nnz + (c.pc_nnz + c.er_nnz & 1);
  int* ep = reinterpret_cast<int*>(wsm + 8 * 448);
  int* eix = ep + c.ne + 1;
  int* pp = eix + c.er_nnz;
  int* pix = pp + c.nu + 1;
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < c.er_nnz; i += blockDim.x) { ev[i] = c.er_val[i]; eix[i] = c.er_idx[i]; }
  for (int i = threadIdx.x; i < c.pc_nnz; i += blockDim.x) { pv[i] = c.pc_val[i]; pix[i] = c.pc_idx[i]; }
  for (int i = threadIdx.x; i <= c.ne; i += blockDim.x) ep[i] = c.er_ptr[i];
  for (int i = threadIdx.x; i <= c.nu; i += blockDim.x) pp[i] = c.pc_ptr[i];
  __syncthreads();
  auto project = [&](const double* xx, const double* tgt, double* rr, double* ya) {
    for (int k = lane; k < c.ne; k += 32) {
      double s = 0.0;
      for (int q = ep[k]; q < ep[k + 1]; ++q) s = fma(xx[eix[q]], ev[q], s);
      rr[k] = s - tgt[k];
    }
    __syncwarp();
    for (int jj = lane; jj < c.nu; jj += 32) {
      double s = 0.0;
      for (int q = pp[jj]; q < pp[jj + 1]; ++q) s = fma(rr[pix[q]], pv[q], s);
      ya[jj] = xx[jj] - s;
    }
    __syncwarp();
  };
  double* x = wsm + (size_t)wl * 448;
  double* y = x + 128;
  double* r = y + 128;
  double* inc = r + 64;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const size_t SW = 2 * (size_t)c.NUP;  // one [x | inc] state row
  double* SA = st;                      // state at the start of the current block
  double* SB = st + (size_t)c.E * SW;   // state at its end
  // runs sweeps [it0, it1) of edge e from state (x, inc) in shared memory
  auto sweeps = [&](int e, int it0, int it1, bool record) {
    const double* tgt = c.jrhs + (size_t)e * c.ne;
    for (int it = it0; it < it1; ++it) {
      project(x, tgt, r, y);
      double mx = 0.0;
      for (int j = lane; j < c.nu; j += 32) {
        const double t = y[j] + inc[j];
        const double xn = clip(t, c.u_min[j], c.u_max[j]);
        inc[j] = t - xn;
        mx = fmax(mx, fabs(xn - x[j]));
        x[j] = xn;
      }
      __syncwarp();
      if (record) {  // per-warp maxima over its edges; reduced per CTA below
        mx = warp_max(mx);
        if (lane == 0) wmax[wl][it - it0] = fmax(wmax[wl][it - it0], mx);
      }
    }
  };
  int K = -1, blk0 = 0;
  for (int blk = 0; blk < kDykMax; blk += kDykBlk) {
    const int it1 = min(blk + kDykBlk, kDykMax);
    if (lane < kDykBlk) wmax[wl][lane] = 0.0;
    __syncwarp();
    for (int e = gw; e < c.E; e += nw) {
      const double* sa = SA + (size_t)e * SW;
      for (int j = lane; j < c.nu; j += 32) {
        x[j] = blk == 0 ? u0[(size_t)e * c.NUP + j] : __ldcg(sa + j);
        inc[j] = blk == 0 ? 0.0 : __ldcg(sa + c.NUP + j);
      }
      __syncwarp();
      sweeps(e, blk, it1, true);
      double* sb = SB + (size_t)e * SW;
      for (int j = lane; j < c.nu; j += 32) {
        __stcg(sb + j, x[j]);
        __stcg(sb + c.NUP + j, inc[j]);
      }
      if (blk == 0) {  // the block-start state of block 0, for a restart
        for (int j = lane; j < c.nu; j += 32) {
          __stcg(SA + (size_t)e * SW + j, u0[(size_t)e * c.NUP + j]);
          __stcg(SA + (size_t)e * SW + c.NUP + j, 0.0);
        }
      }
      __syncwarp();
    }
    // one global atomic per CTA and sweep (same-address global atomics from every
    // warp serialise in L2)
    __syncthreads();
    if (threadIdx.x < it1 - blk) {
      double m = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, wmax[w][threadIdx.x]);
      if (m > 0.0) atomicMax(slots + blk + threadIdx.x, (unsigned long long)__double_as_longlong(m));
    }
    grid.sync();
    for (int it = blk; it < it1; ++it) {
      const double g = __longlong_as_double((long long)*((volatile unsigned long long*)(slots + it)));
      if (g < 1e-13) { K = it; break; }
    }
    if (K >= 0) { blk0 = blk; break; }
    double* t = SA; SA = SB; SB = t;
  }
  // K found: restart K's block and stop after sweep K; else SA holds the state
  // after all kDykMax sweeps
  const int n_left = K >= 0 ? K + 1 - blk0 : 0;
  for (int e = gw; e < c.E; e += nw) {
    const double* sa = SA + (size_t)e * SW;
    for (int j = lane; j < c.nu; j += 32) {
      x[j] = __ldcg(sa + j);
      inc[j] = __ldcg(sa + c.NUP + j);
    }
    __syncwarp();
    sweeps(e, 0, n_left, false);
    project(x, c.jrhs + (size_t)e * c.ne, r, y);
    for (int j = lane; j < c.nu; j += 32) uf[(size_t)e * c.NUP + j] = y[j];
    __syncwarp();
  }
}

// The lockstep Dykstra above with one thread per (edge, junction row): when the
// junction rows touch disjoint flows, the projection onto {E u = d} splits into
// independent rows, so a thread keeps its row's flows, Dykstra increments and
// block-start state in registers.  Per element the operations and their order
// are those of the warp kernels (row dot in ascending flow order, fma(r, p, 0)),
// so the result is bitwise the same.  Flows no junction touches settle after one
// sweep at clip(x0) (projection = identity) and only feed the sweep-0 maximum.
__global__ void __launch_bounds__(256) gap_dykstra_comp_kernel(EdgeCtx c, const DykComp* __restrict__ comps,
                                                                  int ncomp, const int* __restrict__ free_u,
                                                                  int nfree, const double* __restrict__ u0,
                                                                  unsigned long long* slots, double* uf) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned long long cta_max[kDykBlk];
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  {
    double m0 = 0.0;
    for (int i = tid; i < c.E * nfree; i += nth) {
      const int e = i / nfree, j = free_u[i - e * nfree];
      const double x0 = u0[(size_t)e * c.NUP + j];
      const double t = (x0 - 0.0) + 0.0;
      const double xn = clip(t, c.u_min[j], c.u_max[j]);
      m0 = fmax(m0, fabs(xn - x0));
      uf[(size_t)e * c.NUP + j] = xn - 0.0;
    }
    m0 = warp_max(m0);
    if (lane == 0 && m0 > 0.0) atomicMax(slots, (unsigned long long)__double_as_longlong(m0));
  }
  const bool active = tid < c.E * ncomp;
  int e = 0, n = 0, emask = 0, pmask = 0;
  double x[kDykCU], inc[kDykCU], lo[kDykCU], hi[kDykCU], ce[kDykCU], cp[kDykCU], xs[kDykCU], is[kDykCU];
  int ui[kDykCU];
  double tg = 0.0;
  if (active) {
    e = tid / ncomp;
    const DykComp& q = comps[tid - e * ncomp];
    n = q.n;
    emask = q.emask;
    pmask = q.pmask;
    tg = c.jrhs[(size_t)e * c.ne + q.row];
#pragma unroll
    for (int i = 0; i < kDykCU; ++i) {
      ui[i] = i < n ? q.u[i] : 0;
      ce[i] = q.e[i];
      cp[i] = q.p[i];
      x[i] = i < n ? u0[(size_t)e * c.NUP + ui[i]] : 0.0;
      lo[i] = c.u_min[ui[i]];
      hi[i] = c.u_max[ui[i]];
      inc[i] = 0.0;
    }
  }
  auto project_row = [&](double* y) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < kDykCU; ++i)
      if (i < n && (emask >> i & 1)) s = fma(x[i], ce[i], s);
    const double rr = s - tg;
#pragma unroll
    for (int i = 0; i < kDykCU; ++i) y[i] = x[i] - ((pmask >> i & 1) ? fma(rr, cp[i], 0.0) : 0.0);
  };
  auto sweep = [&]() -> double {
    double y[kDykCU], mx = 0.0;
    project_row(y);
#pragma unroll
    for (int i = 0; i < kDykCU; ++i)
      if (i < n) {
        const double t = y[i] + inc[i];
        const double xn = clip(t, lo[i], hi[i]);
        inc[i] = t - xn;
        mx = fmax(mx, fabs(xn - x[i]));
        x[i] = xn;
      }
    return mx;
  };
  int K = -1, blk0 = 0;
  for (int blk = 0; blk < kDykMax; blk += kDykBlk) {
#pragma unroll
    for (int i = 0; i < kDykCU; ++i) {
      xs[i] = x[i];
      is[i] = inc[i];
    }
    double mxs[kDykBlk];
#pragma unroll
    for (int s = 0; s < kDykBlk; ++s) mxs[s] = (active && blk + s < kDykMax) ? sweep() : 0.0;
    // per-sweep maxima: warp, then CTA (shared atomics), then one global atomic
    // per CTA and sweep (thousands of same-address global atomics serialise in L2)
    if (threadIdx.x < kDykBlk) cta_max[threadIdx.x] = 0ull;
    __syncthreads();
#pragma unroll
    for (int s = 0; s < kDykBlk; ++s) {
      const double m = warp_max(mxs[s]);
      if (lane == 0 && m > 0.0) atomicMax(cta_max + s, (unsigned long long)__double_as_longlong(m));
    }
    __syncthreads();
    if (threadIdx.x < kDykBlk && blk + threadIdx.x < kDykMax && cta_max[threadIdx.x] != 0ull)
      atomicMax(slots + blk + threadIdx.x, cta_max[threadIdx.x]);
    grid.sync();
    const int it1 = min(blk + kDykBlk, kDykMax);
    for (int it = blk; it < it1; ++it) {
      const double g = __longlong_as_double((long long)*((volatile unsigned long long*)(slots + it)));
      if (g < 1e-13) { K = it; break; }
    }
    if (K >= 0) { blk0 = blk; break; }
  }
  if (!active) return;
  if (K >= 0) {  // restart K's block, stop after sweep K
#pragma unroll
    for (int i = 0; i < kDykCU; ++i) {
      x[i] = xs[i];
      inc[i] = is[i];
    }
#pragma unroll 1
    for (int s = 0; s < K + 1 - blk0; ++s) (void)sweep();
  }
  double y[kDykCU];
  project_row(y);
#pragma unroll
  for (int i = 0; i < kDykCU; ++i)
    if (i < n) uf[(size_t)e * c.NUP + ui[i]] = y[i];
}

// The same per-(edge, junction row) Dykstra in two passes, for grids too large to be
// co-resident (SMPC8: 178k components): pass 1 runs every component's sweeps and
// records which sweeps change some flow by >= 1e-13 (the stopping criterion needs no
// more than that).  Pass 2 reads the
// stopping sweep K (the first whose maximum is < 1e-13) and reruns every component
// from its start for K + 1 sweeps (all 200 when none stops) before the final affine
// projection.  Per element the operations are those of gap_dykstra_comp_kernel, so
// the result is bitwise the same.
namespace {
struct DykItem {
  int n, emask, pmask;
  int ui[kDykCU];
  double x[kDykCU], inc[kDykCU], lo[kDykCU], hi[kDykCU], ce[kDykCU], cp[kDykCU];
  double tg;
};
__device__ __forceinline__ void dyk_item_load(const EdgeCtx& c, const DykComp& q, int e,
                                              const double* __restrict__ u0, DykItem& it) {
  it.n = q.n;
  it.emask = q.emask;
  it.pmask = q.pmask;
  it.tg = c.jrhs[(size_t)e * c.ne + q.row];
#pragma unroll
  for (int i = 0; i < kDykCU; ++i) {
    it.ui[i] = i < it.n ? q.u[i] : 0;
    it.ce[i] = q.e[i];
    it.cp[i] = q.p[i];
    it.x[i] = i < it.n ? u0[(size_t)e * c.NUP + it.ui[i]] : 0.0;
    it.lo[i] = c.u_min[it.ui[i]];
    it.hi[i] = c.u_max[it.ui[i]];
    it.inc[i] = 0.0;
  }
}
__device__ __forceinline__ void dyk_item_project(const DykItem& it, double* y) {
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < kDykCU; ++i)
    if (i < it.n && (it.emask >> i & 1)) s = fma(it.x[i], it.ce[i], s);
  const double rr = s - it.tg;
#pragma unroll
  for (int i = 0; i < kDykCU; ++i) y[i] = it.x[i] - ((it.pmask >> i & 1) ? fma(rr, it.cp[i], 0.0) : 0.0);
}
// one sweep; returns the largest flow change.  *fixed: this sweep and every later one
// leave the flows unchanged, because with y = P(x) (the same in every later sweep
// while x does not move) each flow satisfies one of
//   interior:  y == x, inc == 0, lo <= x <= hi   ->  t = x, x' = x, inc' = 0
//   at hi:     x == hi, y >= hi, inc >= 0        ->  t = y + inc >= hi, x' = hi, inc' >= 0
//   at lo:     x == lo, y <= lo, inc <= 0        ->  t <= lo, x' = lo, inc' <= 0
// (IEEE rounding is monotone, so the inequalities survive y + inc and t - x').
__device__ __forceinline__ double dyk_item_sweep(DykItem& it, bool* fixed) {
  double y[kDykCU], mx = 0.0;
  bool fx = true;
  dyk_item_project(it, y);
#pragma unroll
  for (int i = 0; i < kDykCU; ++i)
    if (i < it.n) {
      const double x = it.x[i], c = it.inc[i];
      fx = fx && ((y[i] == x && c == 0.0 && it.lo[i] <= x && x <= it.hi[i]) ||
                  (x == it.hi[i] && y[i] >= x && c >= 0.0) || (x == it.lo[i] && y[i] <= x && c <= 0.0));
      const double t = y[i] + c;
      const double xn = clip(t, it.lo[i], it.hi[i]);
      it.inc[i] = t - xn;
      mx = fmax(mx, fabs(xn - x));
      it.x[i] = xn;
    }
  *fixed = fx;
  return mx;
}
}  // namespace

// Pass 1 records only which sweeps have a change >= 1e-13 somewhere (a bit per sweep,
// OR-reduced per warp every 32 sweeps, then per CTA, then globally in the words after
// the value slots): the stopping sweep K is the first sweep without one, exactly the
// first whose maximum over all edges is < 1e-13.
constexpr int kDykWords = (kDykMax + 31) / 32;
__global__ void __launch_bounds__(256) gap_dykstra_comp_pass1_kernel(EdgeCtx c, const DykComp* __restrict__ comps,
                                                                     int ncomp, const int* __restrict__ free_u,
                                                                     int nfree, const double* __restrict__ u0,
                                                                     unsigned long long* slots, double* uf) {
  __shared__ unsigned cta_bits[kDykWords];
  unsigned* gbits = reinterpret_cast<unsigned*>(slots + kDykMax);
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kDykWords; i += blockDim.x) cta_bits[i] = 0u;
  __syncthreads();
  {  // flows no junction touches: clip(x0) after one sweep (sweep 0 only)
    double m0 = 0.0;
    for (int i = tid; i < c.E * nfree; i += nth) {
      const int e = i / nfree, j = free_u[i - e * nfree];
      const double x0 = u0[(size_t)e * c.NUP + j];
      const double t = (x0 - 0.0) + 0.0;
      const double xn = clip(t, c.u_min[j], c.u_max[j]);
      m0 = fmax(m0, fabs(xn - x0));
      uf[(size_t)e * c.NUP + j] = xn - 0.0;
    }
    if (__any_sync(0xffffffffu, m0 >= 1e-13) && lane == 0) atomicOr(cta_bits, 1u);
  }
  const long long total = (long long)c.E * ncomp;
  // warp-uniform trip count: every lane of a warp runs the same number of items
  const long long warp0 = (long long)(tid - lane), nwarps_th = nth;
  for (long long base = warp0; base < total; base += nwarps_th) {
    const long long item = base + lane;
    const bool active = item < total;
    DykItem it;
    it.n = 0;
    if (active) {
      const int e = (int)(item / ncomp);
      dyk_item_load(c, comps[item - (long long)e * ncomp], e, u0, it);
    }
    unsigned bits = 0u;
#pragma unroll 1
    for (int s = 0; s < kDykMax; ++s) {
      bool fixed;
      const double mx = active ? dyk_item_sweep(it, &fixed) : 0.0;
      if (mx >= 1e-13) bits |= 1u << (s & 31);
      if ((s & 31) == 31 || s == kDykMax - 1) {
        const unsigned w = __reduce_or_sync(0xffffffffu, bits);
        if (lane == 0 && w) atomicOr(cta_bits + (s >> 5), w);
        bits = 0u;
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kDykWords; i += blockDim.x)
    if (cta_bits[i]) atomicOr(gbits + i, cta_bits[i]);
}

__global__ void __launch_bounds__(256) gap_dykstra_comp_pass2_kernel(EdgeCtx c, const DykComp* __restrict__ comps,
                                                                     int ncomp, const double* __restrict__ u0,
                                                                     const unsigned long long* __restrict__ slots,
                                                                     double* uf) {
  __shared__ int s_sweeps;
  if (threadIdx.x == 0) {
    const unsigned* gbits = reinterpret_cast<const unsigned*>(slots + kDykMax);
    int K = -1;
    for (int it = 0; it < kDykMax && K < 0; ++it)
      if (!((gbits[it >> 5] >> (it & 31)) & 1u)) K = it;
    s_sweeps = K >= 0 ? K + 1 : kDykMax;
  }
  __syncthreads();
  const int nsw = s_sweeps;
  const long long total = (long long)c.E * ncomp;
  for (long long item = blockIdx.x * (long long)blockDim.x + threadIdx.x; item < total;
       item += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(item / ncomp);
    DykItem it;
    dyk_item_load(c, comps[item - (long long)e * ncomp], e, u0, it);
    bool fixed;
#pragma unroll 1
    for (int s = 0; s < nsw; ++s) (void)dyk_item_sweep(it, &fixed);
    double y[kDykCU];
    dyk_item_project(it, y);
#pragma unroll
    for (int i = 0; i < kDykCU; ++i)
      if (i < it.n) uf[(size_t)e * c.NUP + it.ui[i]] = y[i];
  }
}

// ub_e = u_feas_e B'   (E x NXP)
__global__ void gap_ub_kernel(EdgeCtx c, const double* __restrict__ uf, double* ub) {
  __shared__ double shm[8][128];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int e = gw; e < c.E; e += nw) {
    for (int j = lane; j < c.nu; j += 32) shm[wl][j] = uf[(size_t)e * c.NUP + j];
    __syncwarp();
    for (int i = lane; i < c.nx; i += 32) {
      double s = 0.0;  // non-zeros of row i of B, ascending columns
      for (int q = c.bq_ptr[i]; q < c.bq_ptr[i + 1]; ++q) s = fma(shm[wl][c.bq_idx[q]], c.bq_val[q], s);
      ub[(size_t)e * c.NXP + i] = s;
    }
    __syncwarp();
  }
}

// one stage of x_feas propagation (engine.py:422-432): x = (x_anc A' + u B') + Gd d
__global__ void gap_propagate_stage_kernel(EdgeCtx c, int n0, int n1, double* xf,
                                           const double* __restrict__ ub) {
  const int total = (n1 - n0) * c.nx;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
    const int n = n0 + k / c.nx, i = k % c.nx;
    const int an = c.anc[n];
    double s;
    if (c.a_diag) {
      s = xf[(size_t)an * c.NXP + i] * c.a_diag[i];
    } else {
      s = 0.0;
      for (int j = 0; j < c.nx; ++j) s = fma(xf[(size_t)an * c.NXP + j], c.A[(size_t)i * c.nx + j], s);
    }
    const size_t oe = (size_t)(n - 1) * c.NXP + i;
    xf[(size_t)n * c.NXP + i] = (s + ub[oe]) + c.gdd[oe];
  }
}

// All stages at once when A is diagonal: each (node, component) replays its root
// path top-down with the operations of gap_propagate_stage_kernel, in the same
// order (identical values), so one launch replaces N stage launches.
__global__ void gap_propagate_paths_kernel(EdgeCtx c, int n_nodes, double* xf, const double* __restrict__ ub) {
  const int total = (n_nodes - 1) * c.nx;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
    const int n = 1 + k / c.nx, i = k % c.nx;
    int path[kPropMaxDepth];
    int m = 0;
    for (int v = n; v > 0 && m < kPropMaxDepth; v = c.anc[v]) path[m++] = v;
    const double a = c.a_diag[i];
    double x = xf[i];  // root row (the initial state)
    for (int j = m - 1; j >= 0; --j) {
      const size_t oe = (size_t)(path[j] - 1) * c.NXP + i;
      x = (x * a + ub[oe]) + c.gdd[oe];
    }
    xf[(size_t)n * c.NXP + i] = x;
  }
}

// Primal side, part 2: smooth cost of u_feas and soft state cost (engine.py:347-364).
__global__ void gap_primal_terms_kernel(EdgeCtx c, const double* __restrict__ uf,
                                        const double* __restrict__ xf, double* cols) {
  __shared__ double shm[8][128];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int e = gw; e < c.E; e += nw) {
    const double k0 = smooth_term(c, e, uf, c.NUP, shm[wl]);
    double b = 0, o = 0;
    for (int i = lane; i < c.nx; i += 32) {
      const double x = xf[(size_t)(e + 1) * c.NXP + i];
      const double below = fmax(c.x_s[i] - x, 0.0);
      const double out = x - clip(x, c.x_min[i], c.x_max[i]);
      b = fma(below, below, b);
      o = fma(out, out, o);
    }
    b = sqrt(warp_sum(b));
    o = sqrt(warp_sum(o));
    if (lane == 0) {
      cols[10 * (size_t)e + 0] = k0;
      cols[10 * (size_t)e + 1] = b;
      cols[10 * (size_t)e + 2] = o;
    }
  }
}

}  // namespace tsmpc
