// tsmpc_cache.cuh — device stage cache (tsmpc_cache.cu).
#pragma once
#include <cuda_runtime.h>

namespace tsmpc {

struct CacheArgs {
  int E, nx, nu, nv, nd, ne, NXP, NUP, NVP;
  // tree
  const int *edge_stage, *anc, *child_start, *child_stop;
  const double *prob_edge, *pbar;  // E
  const double* eps;               // E x nd (edge e <-> node e+1)
  // model / basis
  const double* part_map;          // nu x nd
  const double* B;                 // nx x nu
  const double* Gd;                // nx x nd
  const double* Ed;                // ne x nd
  const double* Rhat;              // nu x nv  (Wu L)
  // per forecast
  const double* dhat;              // N x nd
  const double* abar;              // N x nv
  const double* q;                 // nu
  // outputs
  double *uhat, *evec, *beta, *jrhs, *gdd;
  // the same operators by row without their zeros (CSR, ascending columns: the
  // dense summation order), used by cache_rows_sparse_kernel
  const int *pm_ptr, *pm_idx, *ed_ptr, *ed_idx, *b_ptr, *b_idx, *gd_ptr, *gd_idx;
  const double *pm_val, *ed_val, *b_val, *gd_val;
};

#ifndef TSMPC_CB
#define TSMPC_CB 4
#endif
constexpr int kCB = TSMPC_CB;  // edges per pass of cache_beta_kernel

__global__ void cache_rows_kernel(CacheArgs a);
__global__ void cache_rows_sparse_kernel(CacheArgs a);
__global__ void cache_beta_kernel(CacheArgs a);

}  // namespace tsmpc
