// tsmpc_nccl.h — minimal runtime binding of NCCL for the sharded solve.
//
// libtsmpc does not link NCCL: the sharded plan resolves the handful of entry
// points it needs with dlopen/dlsym at plan creation, preferring the libnccl that
// is already loaded in the process (PyTorch's), so one NCCL instance serves both
// torch.distributed and the solver.  Types mirror nccl.h (NCCL 2.x ABI).
#pragma once
#include <cuda_runtime.h>

#include <string>

namespace tsmpc {

struct NcclApi {
  using Comm = void*;
  struct UniqueId { char internal[128]; };
  int (*GetUniqueId)(UniqueId*) = nullptr;
  int (*CommInitRank)(Comm*, int, UniqueId, int) = nullptr;
  int (*CommDestroy)(Comm) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  int (*CommInitAll)(Comm*, int, const int*) = nullptr;  // single-process multi-GPU
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  static constexpr int kUint64 = 5, kFloat64 = 8, kSum = 0, kMax = 2;
};

// Resolve the NCCL entry points (once per process).  Returns nullptr and sets
// `why` if no libnccl can be loaded.
const NcclApi* nccl_api(std::string& why);

}  // namespace tsmpc
