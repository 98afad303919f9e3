// tsmpc_aux.cuh — declarations of the per-edge helper kernels (tsmpc_aux.cu).
#pragma once
#include "tsmpc_kernels.cuh"

namespace tsmpc {

// Read-only per-edge context shared by the helper kernels.
struct EdgeCtx {
  int nx, nu, ne, E, NXP, NUP;
  double Wx, gamma_d, W_alpha;
  const int* edge_stage;
  const int* anc;
  const double *sig_stage, *zeta_stage, *psi_stage;  // null -> identity
  const double *x_s, *x_min, *x_max, *u_min, *u_max;
  const double* prob_edge;  // E
  const double* prices;     // N*nu
  const double* q;          // nu
  const double* Wu;         // nu*nu
  const double* Emat;       // ne*nu (junction matrix)
  const double* Ej;         // row 0 of E (ne == 1)
  const double* EpinvT;     // ne*nu
  const double* jrhs;       // E*ne
  const double* gdd;        // E*NXP
  const double* B;          // nx*nu
  const double* a_diag;     // NXP or null
  const double* A;          // nx*nx
  // sparse junction operators for the Dykstra projection: E by row (CSR) and
  // E_pinv^T by column (CSC), ascending order = the dense summation order
  const int *er_ptr, *er_idx, *pc_ptr, *pc_idx;
  const double *er_val, *pc_val;
  int er_nnz, pc_nnz;
  const int *wu_ptr, *wu_idx;   // Wu by row (CSR): the smooth cost's quadratic form
  const double* wu_val;
  const int *bq_ptr, *bq_idx;   // B by row (CSR): ub = u B'
  const double* bq_val;
};

struct ProxArgs {
  int rows, nx, nu;
  double lam, Wx, gamma_d;
  const int* edge_stage;  // null -> unscaled
  const double *sig_stage, *zeta_stage, *psi_stage;  // compact (N, N, N*nu) or null
  const double *x_s, *x_min, *x_max, *u_min, *u_max;
  const double *t_sig, *t_zeta, *t_psi;
  double *o_sig, *o_zeta, *o_psi;
};

__global__ void reduce_cols_kernel(const double* vals, int n, int ncols, double* out);
__global__ void prox_kernel(ProxArgs a);
__global__ void dual_sq_rows_kernel(EdgeCtx c, const double* y, double* rows);
__global__ void dual_normalize_kernel(EdgeCtx c, double* y, const double* sq);
__global__ void dual_apply_kernel(EdgeCtx c, double* y, const double* X, const double* U,
                                  const double* Z0X, const double* Z0U, double* rows);
__global__ void gap_dual_project_kernel(EdgeCtx c, const double* y, double* what, double* cols);
__global__ void gap_dual_terms_kernel(EdgeCtx c, const double* what, const double* X,
                                      const double* U, double* cols);
__global__ void gap_project_bisect_kernel(EdgeCtx c, const double* uavg, double* uf);
__global__ void gap_project_dykstra_kernel(EdgeCtx c, double* xit, double* inc, double* uf,
                                           unsigned long long* slots);
__global__ void gap_dykstra_pass_kernel(EdgeCtx c, const double* __restrict__ u0,
                                        unsigned long long* slots, int pass, double* uf);
// One junction row of the gap's Dykstra projection with the flows it touches
// (E row k and the E_pinv^T entries of row k), when the junction rows have
// disjoint flow supports (gap_dykstra_comp_kernel).
constexpr int kDykCU = 4;
struct DykComp {
  int n, row, emask, pmask;  // flows, junction row, which E / E_pinv^T entries exist
  int u[kDykCU];             // flow indices, ascending
  double e[kDykCU];          // E[row, u[i]]
  double p[kDykCU];          // E_pinv^T[row, u[i]]
};
__global__ void gap_dykstra_comp_kernel(EdgeCtx c, const DykComp* __restrict__ comps, int ncomp,
                                        const int* __restrict__ free_u, int nfree,
                                        const double* __restrict__ u0, unsigned long long* slots,
                                        double* uf);
__global__ void gap_dykstra_comp_pass1_kernel(EdgeCtx c, const DykComp* __restrict__ comps, int ncomp,
                                              const int* __restrict__ free_u, int nfree,
                                              const double* __restrict__ u0, unsigned long long* slots,
                                              double* uf);
__global__ void gap_dykstra_comp_pass2_kernel(EdgeCtx c, const DykComp* __restrict__ comps, int ncomp,
                                              const double* __restrict__ u0,
                                              const unsigned long long* __restrict__ slots, double* uf);
__global__ void gap_dykstra_coop_kernel(EdgeCtx c, const double* __restrict__ u0,
                                        unsigned long long* slots, double* st, double* uf);
__global__ void gap_ub_kernel(EdgeCtx c, const double* uf, double* ub);
__global__ void gap_propagate_stage_kernel(EdgeCtx c, int n0, int n1, double* xf, const double* ub);
constexpr int kPropMaxDepth = 64;  // deepest tree for gap_propagate_paths_kernel
__global__ void gap_propagate_paths_kernel(EdgeCtx c, int n_nodes, double* xf, const double* ub);
__global__ void gap_primal_terms_kernel(EdgeCtx c, const double* uf, const double* xf, double* cols);

__global__ void apg_persistent_kernel(const __grid_constant__ Params P);
__global__ void apg_sparse_kernel(LaunchWin win);
// copies S to the kernel's constant parameter block and launches (cooperative)
cudaError_t sparse_launch(const SParams& S, LaunchWin w, int ctas, size_t smem, cudaStream_t stream);
cudaError_t sparse_params_upload(const SParams& S, cudaStream_t stream);
cudaError_t sparse_note_launch(cudaStream_t stream);
const void* sparse_kernel_fn(int wide, int nx, bool fg);
__global__ void beta_rotate_kernel(const double* __restrict__ beta, const int* __restrict__ mc,
                                   const double* __restrict__ mv, double* out, int E, int nv, int NVP);

}  // namespace tsmpc
