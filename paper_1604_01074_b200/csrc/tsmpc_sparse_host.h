// tsmpc_sparse_host.h — host planner of the structured-basis kernel
// (tsmpc_sparse.cu): chain tiles, CTA assignment, trunk schedule, shared-memory
// layout.  Pure host code; tsmpc_capi.cu owns the device buffers.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "tsmpc_kernels.cuh"

namespace tsmpc {

struct SparseTreeIn {
  int N, n_nodes;
  const int64_t* stage_starts;  // N + 2
  const int64_t* anc;           // n_nodes
  const int64_t* child_start;   // n_nodes
  const int64_t* child_stop;    // n_nodes
  const double* prob;           // n_nodes
};

struct SparseOpsIn {
  int nx, nu, nv;
  const double* B;    // nx * nu
  const double* Ls;   // nu * nv
  const double* lam;  // nv
};

struct SparseHostPlan {
  bool ok = false;
  std::string why;                  // reason when !ok
  int n_ctas = 0, n_chains = 0, n_trunk = 0, n_tiles = 0;
  int resident_ctas = 0, max_rows = 0, max_needs = 0;
  size_t smem = 0;
  std::vector<int> meta, meta_ptr;  // per-CTA plans
  std::vector<int> tsched;          // trunk schedule
  std::vector<int> trunk_edge;      // trunk position -> edge
  std::vector<int> spi;             // sparse index pool
  std::vector<double> spv;          // sparse value pool
  // split mode: trunk forward operators on a KY row [K | Yx | Ypsi] (pitch KY_LD),
  // du = M1 KY and B du = M2 KY, CSR by row: tpi = [M1 ptr (nu+1) | M1 col | M2 ptr
  // (nx+1) | M2 col], tpv = [M1 val | M2 val] (offsets in SParams)
  std::vector<int> tpi;
  std::vector<double> tpv;
  // sharding (rank of world): chains owned, per trunk position ownership of the heads
  int rank = 0, world = 1, owned_rows = 0, total_chains = 0;
  std::vector<unsigned char> towned;
  std::vector<int> owned_edges;     // edges of the owned chains (ascending)
  // cut exchange (world > 1): role of every trunk position on this rank (kRole*,
  // tsmpc_kernels.cuh) and the rows of the per-iteration exchange buffer: one per
  // mixed position (its chain-head sums) and one per cut position (a single-rank
  // subtree hanging from a mixed position: its bottom-up sums)
  std::vector<signed char> trole;
  std::vector<int> txrow;           // exchange row of each trunk position, -1 if none
  int n_xch = 0;
  bool cut = false;                 // false: whole trunk replicated, XCH = every position's head sums
  std::vector<int> result_edges;    // edges whose rows this rank computes (chains + own / mixed trunk)
  // filled layout / pool offsets (device pointers are set by the caller)
  SParams S{};
};

// Build the plan.  smem_limit: opt-in shared memory per block (bytes);
// max_ctas: SMs available for the cooperative launch.
// sharded: split the leaf chains across `world` ranks by the trunk node they hang
// from (all chain heads of a node go to one rank), keep this rank's share, stream
// every tile (state lives in HBM between the two launches of an iteration).
// allow_split: use split mode (SParams::split) when every chain gets its own CTA
// and enough CTAs are left for the trunk.
// wide: wide mode (SParams::wide, apg_wide_kernel): tiles of up to kTileW rows,
// dual / ergodic rows in HBM, no split mode; chains up to kTileW edges.
SparseHostPlan plan_sparse(const SparseTreeIn& t, const SparseOpsIn& ops, int NXP, int NUP, int NVP,
                           int max_ctas, size_t smem_limit, bool sharded = false, int rank = 0,
                           int world = 1, bool psi_in_smem = true, bool allow_split = true,
                           bool wide = false);

}  // namespace tsmpc
