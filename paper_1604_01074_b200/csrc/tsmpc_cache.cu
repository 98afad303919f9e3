// tsmpc_cache.cu — per-forecast stage cache on the device (reference
// pkg/src/treesmpc/elimination.py:114-158 build_stage_cache and tree.py:319-331
// node_demands).  Per forecast only the stage forecast dhat (N x n_d), the stage
// prices (N x n_u), the reduced prices alpha_bar (N x n_v) and q go up; the
// per-edge vectors are built in HBM:
//
//   d_e    = dhat[stage(e)] + eps_{e+1}                       (node_demands)
//   uhat_e = part_map d_e            e_e = B uhat_e + Gd d_e
//   beta_e = p_e abar[stage(e)] + 2 Rhat' (pbar_e uhat_e - p_e uhat_pa(e) - sum_c p_c uhat_c)
//
// plus the duality-gap inputs jrhs_e = -Ed d_e and gdd_e = Gd d_e.  One CTA per
// edge row (grid-strided); the operands of a row are staged in shared memory.
#include "tsmpc_cache.cuh"

namespace tsmpc {

__global__ void __launch_bounds__(128) cache_rows_kernel(CacheArgs a) {
  extern __shared__ double sm[];
  double* d = sm;               // n_d
  double* uh = sm + a.nd;       // n_u
  for (int e = blockIdx.x; e < a.E; e += gridDim.x) {
    const int st = a.edge_stage[e];
    for (int k = threadIdx.x; k < a.nd; k += blockDim.x)
      d[k] = __dadd_rn(a.dhat[(size_t)st * a.nd + k], a.eps[(size_t)e * a.nd + k]);
    __syncthreads();
    for (int j = threadIdx.x; j < a.nu; j += blockDim.x) {
      double s = 0.0;
      const double* pm = a.part_map + (size_t)j * a.nd;
      for (int k = 0; k < a.nd; ++k) s = fma(pm[k], d[k], s);
      uh[j] = s;
      a.uhat[(size_t)e * a.NUP + j] = s;
    }
    for (int r = threadIdx.x; r < a.ne; r += blockDim.x) {
      double s = 0.0;
      const double* ed = a.Ed + (size_t)r * a.nd;
      for (int k = 0; k < a.nd; ++k) s = fma(ed[k], d[k], s);
      a.jrhs[(size_t)e * a.ne + r] = -s;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < a.nx; i += blockDim.x) {
      double bu = 0.0, gd = 0.0;
      const double* b = a.B + (size_t)i * a.nu;
      for (int j = 0; j < a.nu; ++j) bu = fma(b[j], uh[j], bu);
      const double* g = a.Gd + (size_t)i * a.nd;
      for (int k = 0; k < a.nd; ++k) gd = fma(g[k], d[k], gd);
      a.evec[(size_t)e * a.NXP + i] = __dadd_rn(bu, gd);
      a.gdd[(size_t)e * a.NXP + i] = gd;
    }
    __syncthreads();
  }
}

// The same rows with the operators in CSR (a water network's part_map, Ed, B, Gd
// have a few entries per row): a CTA per edge row, skipped zeros only drop
// fma(0, d, s) = s terms (the dense kernel's results, bitwise).
__global__ void __launch_bounds__(128) cache_rows_sparse_kernel(CacheArgs a) {
  extern __shared__ double sm[];
  double* d = sm;               // n_d
  double* uh = sm + a.nd;       // n_u
  for (int e = blockIdx.x; e < a.E; e += gridDim.x) {
    const int st = a.edge_stage[e];
    for (int k = threadIdx.x; k < a.nd; k += blockDim.x)
      d[k] = __dadd_rn(a.dhat[(size_t)st * a.nd + k], a.eps[(size_t)e * a.nd + k]);
    __syncthreads();
    for (int j = threadIdx.x; j < a.nu; j += blockDim.x) {
      double s = 0.0;
      for (int q = a.pm_ptr[j]; q < a.pm_ptr[j + 1]; ++q) s = fma(a.pm_val[q], d[a.pm_idx[q]], s);
      uh[j] = s;
      a.uhat[(size_t)e * a.NUP + j] = s;
    }
    for (int r = threadIdx.x; r < a.ne; r += blockDim.x) {
      double s = 0.0;
      for (int q = a.ed_ptr[r]; q < a.ed_ptr[r + 1]; ++q) s = fma(a.ed_val[q], d[a.ed_idx[q]], s);
      a.jrhs[(size_t)e * a.ne + r] = -s;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < a.nx; i += blockDim.x) {
      double bu = 0.0, gd = 0.0;
      for (int q = a.b_ptr[i]; q < a.b_ptr[i + 1]; ++q) bu = fma(a.b_val[q], uh[a.b_idx[q]], bu);
      for (int q = a.gd_ptr[i]; q < a.gd_ptr[i + 1]; ++q) gd = fma(a.gd_val[q], d[a.gd_idx[q]], gd);
      a.evec[(size_t)e * a.NXP + i] = __dadd_rn(bu, gd);
      a.gdd[(size_t)e * a.NXP + i] = gd;
    }
    __syncthreads();
  }
}

// beta_e = p_e abar[stage] + 2 Rhat' (pbar_e uhat_e - p_e uhat_pa(e) - sum_c p_c uhat_c),
// kCB edges per pass of a CTA: their combos in shared memory, each thread's column
// of Rhat read once for all of them (independent accumulations, each in the
// ascending-j order of the single-edge product).
__global__ void __launch_bounds__(128) cache_beta_kernel(CacheArgs a) {
  extern __shared__ double sm[];
  double* combo = sm;  // kCB x n_u
  for (int e0 = blockIdx.x * kCB; e0 < a.E; e0 += gridDim.x * kCB) {
    const int ne = min(kCB, a.E - e0);
    for (int idx = threadIdx.x; idx < ne * a.nu; idx += blockDim.x) {
      const int b = idx / a.nu, j = idx - b * a.nu, e = e0 + b;
      const int node = e + 1;
      const int pa = a.anc[node] - 1;
      const int c0 = a.child_start[node] - 1, c1 = a.child_stop[node] - 1;
      const double pe = a.prob_edge[e], pb = a.pbar[e];
      const double up = pa >= 0 ? a.uhat[(size_t)pa * a.NUP + j] : a.q[j];
      double cs = 0.0;  // sum over children in node order (np.add.at order)
      for (int c = c0; c < c1; ++c) cs = __dadd_rn(cs, __dmul_rn(a.prob_edge[c], a.uhat[(size_t)c * a.NUP + j]));
      combo[b * a.nu + j] = __dsub_rn(__dsub_rn(__dmul_rn(pb, a.uhat[(size_t)e * a.NUP + j]), __dmul_rn(pe, up)), cs);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < a.nv; k += blockDim.x) {
      double s[kCB];
#pragma unroll
      for (int b = 0; b < kCB; ++b) s[b] = 0.0;
      for (int j = 0; j < a.nu; ++j) {
        const double r = a.Rhat[(size_t)j * a.nv + k];
#pragma unroll
        for (int b = 0; b < kCB; ++b)
          if (b < ne) s[b] = fma(combo[b * a.nu + j], r, s[b]);
      }
#pragma unroll
      for (int b = 0; b < kCB; ++b)
        if (b < ne) {
          const int e = e0 + b;
          a.beta[(size_t)e * a.NVP + k] = __dadd_rn(__dmul_rn(a.prob_edge[e], a.abar[(size_t)a.edge_stage[e] * a.nv + k]),
                                                    __dmul_rn(2.0, s[b]));
        }
    }
    __syncthreads();
  }
}

}  // namespace tsmpc
