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
};

__global__ void cache_rows_kernel(CacheArgs a);
__global__ void cache_beta_kernel(CacheArgs a);

}  // namespace tsmpc
