// tsmpc_capi.cu — host runtime behind include/tsmpc.h: tree planning (segments,
// levels, tiles), HBM layout, uploads, launches and the C ABI.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tsmpc.h"
#include "tsmpc_aux.cuh"
#include "tsmpc_cache.cuh"
#include "tsmpc_nccl.h"
#include "tsmpc_sparse_host.h"

using namespace tsmpc;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(TSMPC_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                    \
  } while (0)

inline int r4(int v) { return (v + 3) / 4 * 4; }
constexpr size_t kArenaPad = 0;  // TSMPC_ARENA_PAD overrides (bytes)
inline int r8(int v) { return (v + 7) / 8 * 8; }

}  // namespace

struct tsmpc_plan {
  int device = 0;
  int nx, nu, nv, nd, ne, N, n_nodes, E;
  int NXP, NUP, NVP;
  int sm_count = 0;
  size_t smem = 0;
  Params base{};
  EdgeCtx ctx{};
  cudaStream_t stream = nullptr;
  cudaStream_t stream2 = nullptr;   // result read-back, overlapping the duality gap
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev_out = nullptr;
  long long launches = 0;  // kernels launched by the current API call
  std::vector<void*> allocs;
  std::vector<int64_t> stage_starts;
  bool has_cache = false;
  bool has_op = false;
  // device buffers
  double *Y0, *Y1, *WB, *PY;
  double *XAVG, *UAVG, *X, *U, *XL, *UL, *T, *GG, *XIQG;
  double *BETA, *BETA0, *UHAT, *EVEC, *GDD, *JRHS, *PRICES, *Q, *P;
  double *Z0X, *Z0U, *UF, *XIT, *INC, *UB, *XF, *COLS, *ROWS, *RED;
  double *THETA, *COEF;
  int theta_cap = 0;
  unsigned long long* RESID = nullptr;
  int resid_cap = 0;
  unsigned long long* DYK = nullptr;
  // residual stopping test (tsmpc_set_stopping; sparse kernel only)
  double tol = 0.0;
  int check_every = 25;
  unsigned long long* RCHK = nullptr;
  int rchk_cap = 0;
  int* ITERS = nullptr;
  unsigned long long* TIMERS = nullptr;
  // compact scaling copies for tsmpc_prox
  double *sig_c = nullptr, *zeta_c = nullptr, *psi_c = nullptr;
  // structured-basis kernel (tsmpc_sparse.cu); used by tsmpc_solve when available
  bool use_sparse = false;
  SParams sbase{};
  int sp_ctas = 0, sp_resident = 0, sp_tiles = 0, sp_trunk = 0;
  size_t sp_smem = 0;
  double *BETA_S = nullptr, *TG = nullptr, *FG = nullptr, *KY_S = nullptr, *MS = nullptr;
  int* MSC = nullptr;  // the basis rotation M by column without zeros: [ptr (nv+1) | rows], values in MS
  std::string sp_why;
  // device stage cache (tsmpc_set_cache_operators / tsmpc_set_forecast)
  bool has_cache_ops = false;
  int nd_c = 0;
  double *PART_MAP = nullptr, *GD = nullptr, *ED = nullptr, *RHAT = nullptr, *EPS = nullptr, *PBAR = nullptr;
  // the stage cache operators part_map, Ed, B, Gd in CSR (device): ints, values, offsets
  int* CSR_I = nullptr;
  double* CSR_V = nullptr;
  int csr_oi[8] = {0}, csr_ov[4] = {0};
  double *DHAT = nullptr, *ABAR = nullptr;
  double* last_y = nullptr;  // final dual of the last solve (device warm start)
  int *d_est_c = nullptr, *d_anc_c = nullptr, *d_cs_c = nullptr, *d_ce_c = nullptr;
  double *d_pe_c = nullptr, *d_B_c = nullptr;
  // subtree sharding across GPUs (tsmpc_plan_create_shard)
  bool sharded = false;
  int rank = 0, world = 1, total_chains = 0;
  const NcclApi* nccl = nullptr;
  void* comm = nullptr;
  double* HS = nullptr;
  double* XCH = nullptr;            // shard plans: the cut exchange rows (summed across ranks)
  // shard plans: the cut exchange over peer memory inside the kernel (SParams::peer_rx)
  double* RX = nullptr;                 // 2 x world x n_xch x XCH_LD receive rows
  unsigned long long* RXCNT = nullptr;  // arrival counter
  std::vector<void*> ipc_mapped;        // other ranks' buffers opened with cudaIpcOpenMemHandle
  bool peer_on = false;
  unsigned long long xgen = 0;          // exchange generations run so far (the same on every rank)
  double* TR = nullptr;            // split mode: [du | B du | x] per trunk position
  unsigned int* SUBCTR = nullptr;  // split mode: trunk-CTA barrier counter
  unsigned int* ABORT = nullptr;   // raised by a sparse-kernel spin-wait that timed out
  double* GTR = nullptr;           // per-iteration gap reductions (TSMPC_GAP_TRACE), iters x 10
  int gtr_cap = 0;
  double* DYKST = nullptr;  // lockstep Dykstra state (2 x E x [x | inc])
  DykComp* DYKC = nullptr;  // per-junction-row components (disjoint flow supports)
  int* DYKF = nullptr;      // flows no junction touches
  int dyk_ncomp = -1, dyk_nfree = 0;  // dyk_ncomp < 0: components not usable
  bool dyk_warp = std::getenv("TSMPC_DYKSTRA_WARP") != nullptr;
  bool dyk_two_pass = std::getenv("TSMPC_DYKSTRA_TWO_PASS") != nullptr;
  std::vector<int> owned_edges, trunk_edges;
  std::vector<int> result_edges;    // shard plans: rows this rank computes (chains + own / mixed trunk)
  std::vector<int> zero_edges;      // shard plans: rows zeroed before the cross-rank assembly
  int* d_zero = nullptr;
  bool multi = false;               // one of the plans of tsmpc_plans_create_multi
  cudaGraphExec_t gexec = nullptr;  // sharded solve: the captured launches + all-reduces
  int g_iters = 0;
  std::string graph_why;
  // plan stats
  int n_levels = 0, n_tiles = 0, n_segs = 0, n_ctas = 0, n_trunk = 0;
  int dyk_blocks = 0;

  template <class T>
  int alloc(T** p, size_t count) {
    void* d = nullptr;
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc(&d, count * sizeof(T));
    if (e != cudaSuccess)
      return fail(TSMPC_ERR_CUDA, "cudaMalloc(%zu bytes): %s", count * sizeof(T), cudaGetErrorString(e));
    allocs.push_back(d);
    *p = static_cast<T*>(d);
    e = cudaMemsetAsync(d, 0, count * sizeof(T), stream);
    if (e != cudaSuccess) return fail(TSMPC_ERR_CUDA, "cudaMemset: %s", cudaGetErrorString(e));
    return TSMPC_OK;
  }
  template <class T>
  int upload(T** p, const T* host, size_t count) {
    int rc = alloc(p, count);
    if (rc) return rc;
    CU(cudaMemcpyAsync(*p, host, count * sizeof(T), cudaMemcpyHostToDevice, stream));
    return TSMPC_OK;
  }
  // host rows of `w` doubles -> device rows of pitch `ld` doubles
  int put_rows(double* dst, int ld, const double* src, int w, int rows) {
    if (rows == 0 || w == 0) return TSMPC_OK;
    CU(cudaMemcpy2DAsync(dst, ld * sizeof(double), src, w * sizeof(double), w * sizeof(double), rows,
                         cudaMemcpyHostToDevice, stream));
    return TSMPC_OK;
  }
  int get_rows(double* dst, int w, const double* src, int ld, int rows, cudaStream_t s = nullptr) {
    if (rows == 0 || w == 0 || dst == nullptr) return TSMPC_OK;
    CU(cudaMemcpy2DAsync(dst, w * sizeof(double), src, ld * sizeof(double), w * sizeof(double), rows,
                         cudaMemcpyDeviceToHost, s ? s : stream));
    return TSMPC_OK;
  }
  ~tsmpc_plan() {
    if (stream) cudaStreamSynchronize(stream);
    if (gexec) cudaGraphExecDestroy(gexec);
    if (comm && nccl) nccl->CommDestroy(comm);
    for (void* p : ipc_mapped) cudaIpcCloseMemHandle(p);
    for (void* p : allocs) cudaFree(p);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (ev2) cudaEventDestroy(ev2);
    if (ev_out) cudaEventDestroy(ev_out);
    if (stream2) {
      cudaStreamSynchronize(stream2);
      cudaStreamDestroy(stream2);
    }
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

// ---------------------------------------------------------------- planning
// The structured-basis plan: split / resident / slot-streamed (apg_sparse_kernel),
// or wide mode (apg_wide_kernel) when some CTA would stream its rows through a
// tile slot, when a leaf chain is longer than a slot tile, and for shards
// (TSMPC_NO_WIDE keeps the slot-streaming plan).
SparseHostPlan choose_sparse_plan(const SparseTreeIn& ti, const SparseOpsIn& oi, int NXP, int NUP, int NVP,
                                  int ctas, size_t smem_plain, size_t smem_wide, bool shard, int rank, int world) {
  SparseHostPlan hp = plan_sparse(ti, oi, NXP, NUP, NVP, ctas, smem_plain, shard, rank, world);
  if (!std::getenv("TSMPC_NO_WIDE") && oi.nx <= 128 && (!hp.ok || hp.resident_ctas < hp.n_ctas || shard)) {
    SparseHostPlan hw = plan_sparse(ti, oi, NXP, NUP, NVP, ctas, smem_wide, shard, rank, world, true, true, true);
    if (hw.ok) return hw;
    if (!hp.ok) hp.why += std::string("; wide mode: ") + hw.why;
  }
  return hp;
}

struct Decomposition {
  int n_levels = 0;
  std::vector<int> lvl_tiles, tile_seg, seg_row, row_edge;
  int n_ctas = 0;
  // collapsed-trunk mode
  bool collapsed = false;
  std::vector<int> trunk_edge, trunk_stage_ptr, trunk_pos, path_ptr, path_list, trunk_child0,
      trunk_parent;
};

// Cut the tree into segments (maximal only-child chains of <= kMaxSeg edges),
// group them by segment depth, balance each level's rows over the CTAs and pack
// every CTA's share into tiles of <= kTileM rows.
int decompose(const tsmpc_problem* pb, int max_ctas, bool collapse, Decomposition& out) {
  const int n_nodes = pb->n_nodes, E = n_nodes - 1;
  std::vector<int> nch(n_nodes);
  for (int n = 0; n < n_nodes; ++n) nch[n] = (int)(pb->child_stop[n] - pb->child_start[n]);
  std::vector<char> head(E, 0);
  for (int e = 0; e < E; ++e) {
    const int p = (int)pb->anc[e + 1];
    head[e] = (p == 0 || nch[p] != 1) ? 1 : 0;
  }
  std::vector<std::vector<int>> segs;
  std::vector<int> seg_of(E, -1);
  for (int e = 0; e < E; ++e) {
    if (!head[e] || seg_of[e] >= 0) continue;
    int cur = e;
    while (cur >= 0) {  // one segment per pass; long chains continue in a new segment
      std::vector<int> s{cur};
      seg_of[cur] = (int)segs.size();
      int x = cur;
      int next = -1;
      while (nch[x + 1] == 1) {
        const int c = (int)pb->child_start[x + 1] - 1;
        if ((int)s.size() == kMaxSeg) { next = c; break; }
        s.push_back(c);
        seg_of[c] = (int)segs.size();
        x = c;
      }
      segs.push_back(std::move(s));
      cur = next;
    }
  }
  for (int e = 0; e < E; ++e)
    if (seg_of[e] < 0) return fail(TSMPC_ERR_VALIDATION, "tree decomposition missed edge %d", e);
  // segment order by head edge id => parents before children
  std::vector<int> order(segs.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return segs[a][0] < segs[b][0]; });
  std::vector<int> level(segs.size(), 0);
  int D = 0;
  for (int s : order) {
    const int h = segs[s][0];
    const int pn = (int)pb->anc[h + 1];
    level[s] = pn == 0 ? 0 : level[seg_of[pn - 1]] + 1;
    D = std::max(D, level[s] + 1);
  }
  std::vector<std::vector<int>> by_level(D);
  for (int s : order) by_level[level[s]].push_back(s);
  out.collapsed = collapse;
  if (collapse) {
    // leaf segments (tail is a leaf) form the single tile level; every other edge
    // is a trunk edge handled by the collapsed sweep + GEMM
    std::vector<int> leaf_segs;
    std::vector<char> in_leaf(E, 0);
    for (int s : order) {
      if (nch[segs[s].back() + 1] == 0) {
        leaf_segs.push_back(s);
        for (int e : segs[s]) in_leaf[e] = 1;
      }
    }
    out.trunk_pos.assign(E, -1);
    out.trunk_edge.clear();
    for (int e = 0; e < E; ++e)
      if (!in_leaf[e]) {
        out.trunk_pos[e] = (int)out.trunk_edge.size();
        out.trunk_edge.push_back(e);
      }
    const int N = pb->N;
    out.trunk_stage_ptr.assign(N + 1, 0);
    {
      int k = 0;
      for (int st = 0; st < N; ++st) {
        out.trunk_stage_ptr[st] = k;
        const int e_end = (int)pb->stage_starts[st + 2] - 1;  // edges into stage st+1
        while (k < (int)out.trunk_edge.size() && out.trunk_edge[k] < e_end) ++k;
      }
      out.trunk_stage_ptr[N] = k;
    }
    out.trunk_parent.assign(out.trunk_edge.size(), -1);
    for (size_t t = 0; t < out.trunk_edge.size(); ++t) {
      const int pa = (int)pb->anc[out.trunk_edge[t] + 1] - 1;
      out.trunk_parent[t] = pa >= 0 ? out.trunk_pos[pa] : -1;
    }
    out.trunk_child0.assign(out.trunk_edge.size(), -1);
    for (size_t t = 0; t < out.trunk_edge.size(); ++t) {
      const int node = out.trunk_edge[t] + 1;
      int n_tr = 0, n = 0;
      for (int64_t ch = pb->child_start[node] - 1; ch < pb->child_stop[node] - 1; ++ch, ++n)
        n_tr += out.trunk_pos[ch] >= 0;
      out.trunk_child0[t] = n_tr == 0 ? -1 : (n_tr == n ? out.trunk_pos[pb->child_start[node] - 1] : -2);
    }
    out.path_ptr.assign(out.trunk_edge.size() + 1, 0);
    out.path_list.clear();
    for (size_t t = 0; t < out.trunk_edge.size(); ++t) {
      std::vector<int> path;
      for (int e = out.trunk_edge[t]; e >= 0; e = (int)pb->anc[e + 1] - 1) path.push_back(out.trunk_pos[e]);
      for (auto it = path.rbegin(); it != path.rend(); ++it) out.path_list.push_back(*it);
      out.path_ptr[t + 1] = (int)out.path_list.size();
    }
    by_level.assign(1, leaf_segs);
    D = 1;
  }
  size_t widest = 0;
  for (auto& v : by_level) widest = std::max(widest, v.size());
  int C = std::max(1, std::min<int>(max_ctas, (int)widest));
  if (collapse && !out.trunk_edge.empty()) C = std::max(1, max_ctas);

  out.n_levels = D;
  out.n_ctas = C;
  out.lvl_tiles.assign((size_t)D * C + 1, 0);
  out.tile_seg.clear();
  out.seg_row.clear();
  out.row_edge.clear();
  int tiles = 0;
  for (int l = 0; l < D; ++l) {
    const auto& v = by_level[l];
    long long R = 0;
    for (int s : v) R += (long long)segs[s].size();
    std::vector<std::vector<int>> share(C);
    long long pre = 0;
    for (int s : v) {
      const long long mid2 = 2 * pre + (long long)segs[s].size();  // 2 x segment midpoint
      int c = (int)((mid2 * C) / (2 * std::max<long long>(R, 1)));
      c = std::min(std::max(c, 0), C - 1);
      share[c].push_back(s);
      pre += (long long)segs[s].size();
    }
    for (int c = 0; c < C; ++c) {
      out.lvl_tiles[(size_t)l * C + c] = tiles;
      int rows_in_tile = kTileM + 1;
      for (int s : share[c]) {
        const int len = (int)segs[s].size();
        if (rows_in_tile + len > kTileM) {  // open a new tile
          out.tile_seg.push_back((int)out.seg_row.size());
          ++tiles;
          rows_in_tile = 0;
        }
        out.seg_row.push_back((int)out.row_edge.size());
        for (int e : segs[s]) out.row_edge.push_back(e);
        rows_in_tile += len;
      }
    }
  }
  out.lvl_tiles[(size_t)D * C] = tiles;
  out.tile_seg.push_back((int)out.seg_row.size());
  out.seg_row.push_back((int)out.row_edge.size());
  return TSMPC_OK;
}

int launch_apg(tsmpc_plan* pl, const Params& P) {
  void* args[] = {const_cast<Params*>(&P)};
  CU(cudaLaunchCooperativeKernel((void*)apg_persistent_kernel, dim3(pl->n_ctas), dim3(kThreads), args,
                                 pl->smem, pl->stream));
  ++pl->launches;
  return TSMPC_OK;
}

int grid_for(int E) {  // warp-per-edge helper kernels, 256 threads = 8 warps per block
  return std::max(1, std::min((E + 7) / 8, 148 * 16));
}

}  // namespace

extern "C" {

const char* tsmpc_last_error(void) { return g_err.c_str(); }

const char* tsmpc_plan_path(const tsmpc_plan* pl) {
  if (!pl) return "";
  static thread_local std::string s;
  s = !pl->use_sparse ? "dense: " + pl->sp_why
                      : pl->sbase.wide ? "sparse (wide)" : pl->sbase.split ? "sparse (split)" : "sparse";
  return s.c_str();
}

void* tsmpc_host_alloc(int64_t bytes) {
  void* p = nullptr;
  if (bytes <= 0 || cudaHostAlloc(&p, (size_t)bytes, cudaHostAllocPortable) != cudaSuccess) {
    fail(TSMPC_ERR_CUDA, "cudaHostAlloc(%lld bytes) failed", (long long)bytes);
    return nullptr;
  }
  return p;
}

void tsmpc_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int tsmpc_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

static tsmpc_plan* plan_create_impl(const tsmpc_problem* pb, int device, int srank, int sworld,
                                    const void* nccl_id) {
  const bool shard = srank >= 0;
  if (!pb) { fail(TSMPC_ERR_ARGUMENT, "null problem"); return nullptr; }
  const int nx = pb->n_x, nu = pb->n_u, nv = pb->n_v, ne = pb->n_e, N = pb->N, n_nodes = pb->n_nodes;
  if (nx < 1 || nu < 1 || nv < 1 || ne < 1 || N < 1 || n_nodes < 2) {
    fail(TSMPC_ERR_DIMENSION, "invalid dimensions n_x=%d n_u=%d n_v=%d n_e=%d N=%d n_nodes=%d", nx, nu, nv, ne,
         N, n_nodes);
    return nullptr;
  }
  if (nx > 128 || nu > 128 || ne > 64) {
    fail(TSMPC_ERR_DIMENSION, "dimension above the supported limit (n_x, n_u <= 128, n_e <= 64)");
    return nullptr;
  }
  if (!pb->A || !pb->B || !pb->L || !pb->Bbar || !pb->Phi || !pb->Psi || !pb->Wu || !pb->E ||
      !pb->E_pinvT || !pb->u_min || !pb->u_max || !pb->x_min || !pb->x_max || !pb->x_s ||
      !pb->stage_starts || !pb->anc || !pb->child_start || !pb->child_stop || !pb->prob) {
    fail(TSMPC_ERR_ARGUMENT, "null array in tsmpc_problem");
    return nullptr;
  }
  if (pb->stage_starts[0] != 0 || pb->stage_starts[N + 1] != n_nodes || pb->stage_starts[1] != 1) {
    fail(TSMPC_ERR_VALIDATION, "stage offsets do not cover the node arrays");
    return nullptr;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    fail(TSMPC_ERR_CUDA, "no CUDA device available");
    return nullptr;
  }
  if (device < 0 || device >= ndev) {
    fail(TSMPC_ERR_ARGUMENT, "device %d out of range (%d devices)", device, ndev);
    return nullptr;
  }
  auto* pl = new tsmpc_plan();
  auto bail = [&](int) -> tsmpc_plan* { delete pl; return nullptr; };
  pl->device = device;
  if (cudaSetDevice(device) != cudaSuccess) { fail(TSMPC_ERR_CUDA, "cudaSetDevice failed"); return bail(0); }
  if (cudaStreamCreateWithFlags(&pl->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&pl->stream2, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&pl->ev0) != cudaSuccess || cudaEventCreate(&pl->ev1) != cudaSuccess ||
      cudaEventCreate(&pl->ev2) != cudaSuccess ||
      cudaEventCreateWithFlags(&pl->ev_out, cudaEventDisableTiming) != cudaSuccess) {
    fail(TSMPC_ERR_CUDA, "stream/event creation failed");
    return bail(0);
  }
  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, device);
  pl->sm_count = prop.multiProcessorCount;

  const int E = n_nodes - 1;
  pl->nx = nx; pl->nu = nu; pl->nv = nv; pl->nd = pb->n_d; pl->ne = ne; pl->N = N;
  pl->n_nodes = n_nodes; pl->E = E;
  const int NXP = r4(nx), NUP = r4(nu), NVP = r4(nv);
  pl->NXP = NXP; pl->NUP = NUP; pl->NVP = NVP;
  pl->stage_starts.assign(pb->stage_starts, pb->stage_starts + N + 2);

  Params& P = pl->base;
  P.nx = nx; P.nu = nu; P.nv = nv; P.N = N; P.n_nodes = n_nodes; P.n_edges = E;
  P.NXP = NXP; P.NUP = NUP; P.NVP = NVP;
  const int K1 = NXP + NUP;
  P.KS1 = K1 / 4;
  P.NT1 = (nv + 7) / 8;
  P.KS2 = NVP / 4;
  P.NU8 = r8(nu);
  P.NT2 = (P.NU8 + r8(nx)) / 8;
  // shared-memory tile layout: A leading dims = 4 mod 16 doubles (conflict-free
  // DMMA fragment loads); C holds h (backward) / [u | bv + e] (forward)
  auto lda_of = [](int k) { while (k % 16 != 4) ++k; return k; };
  P.LDA1 = lda_of(K1);
  P.LDB1 = std::max(P.NT1 * 8, r8(nx));          // dense-A child sums reuse C
  P.LDA2 = lda_of(std::max(NVP, NXP));           // S, then x
  P.LDB2 = P.NT2 * 8;
  // the trunk GEMM reduces kWarps x 4 m-tile partials through the tile region
  const int region = std::max({kTileM * (P.LDA1 + P.LDB1), kTileM * (P.LDA2 + P.LDB2), kWarps * 4 * 64});
  P.META_OFF = region;
  P.Wx = pb->Wx; P.gamma_d = pb->gamma_d;
  // + metadata ints (<= 160 doubles) + per-row inv2p (kTileM doubles) + model bounds
  pl->smem = sizeof(double) * ((size_t)region + 160 + kTileM + 3 * NXP + 2 * NUP);
  if (pl->smem > (size_t)prop.sharedMemPerBlockOptin) {
    fail(TSMPC_ERR_DIMENSION, "tile needs %zu bytes of shared memory (limit %zu)", pl->smem,
         (size_t)prop.sharedMemPerBlockOptin);
    return bail(0);
  }
  cudaFuncAttributes fp{};
  cudaFuncGetAttributes(&fp, apg_persistent_kernel);
  if (cudaFuncSetAttribute(apg_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(prop.sharedMemPerBlockOptin - fp.sharedSizeBytes)) != cudaSuccess) {
    fail(TSMPC_ERR_CUDA, "cannot reserve %zu bytes of shared memory", pl->smem);
    return bail(0);
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, apg_persistent_kernel, kThreads, pl->smem);
  if (occ < 1) { fail(TSMPC_ERR_CUDA, "persistent kernel does not fit on an SM"); return bail(0); }

  bool diag = true;
  for (int i = 0; i < nx && diag; ++i)
    for (int j = 0; j < nx; ++j)
      if (i != j && pb->A[(size_t)i * nx + j] != 0.0) { diag = false; break; }
  const char* env_mode = getenv("TSMPC_LEVEL_MODE");  // force the level-synchronous path
  const bool collapse = diag && !(env_mode && env_mode[0] == '1');

  Decomposition dec;
  if (decompose(pb, pl->sm_count * std::min(occ, 1), collapse, dec)) return bail(0);
  pl->n_levels = dec.n_levels;
  pl->n_ctas = dec.n_ctas;
  pl->n_tiles = (int)dec.tile_seg.size() - 1;
  pl->n_segs = (int)dec.seg_row.size() - 1;
  pl->n_trunk = (int)dec.trunk_edge.size();
  P.n_levels = dec.n_levels;
  P.n_ctas = dec.n_ctas;
  P.collapsed = dec.collapsed ? 1 : 0;
  P.n_trunk = pl->n_trunk;

  // ---- operator blocks in DMMA fragment order
  std::vector<double> W1((size_t)K1 * P.NT1 * 8, 0.0), W2((size_t)P.KS2 * 4 * P.NT2 * 8, 0.0);
  const int n1 = P.NT1 * 8, n2 = P.NT2 * 8;
  for (int i = 0; i < nx; ++i)
    for (int n = 0; n < nv; ++n) W1[(size_t)i * n1 + n] = pb->Bbar[(size_t)i * nv + n];
  for (int j = 0; j < nu; ++j)
    for (int n = 0; n < nv; ++n) W1[(size_t)(NXP + j) * n1 + n] = pb->L[(size_t)j * nv + n];
  for (int k = 0; k < nv; ++k) {
    for (int j = 0; j < nu; ++j) W2[(size_t)k * n2 + j] = pb->Psi[(size_t)k * nu + j];
    for (int i = 0; i < nx; ++i) W2[(size_t)k * n2 + P.NU8 + i] = pb->Phi[(size_t)k * nx + i];
  }
  auto frag = [](const std::vector<double>& W, int KS, int NT) {
    std::vector<double> f((size_t)NT * KS * 32);
    const int ld = NT * 8;
    for (int nt = 0; nt < NT; ++nt)
      for (int ks = 0; ks < KS; ++ks)
        for (int l = 0; l < 32; ++l)
          f[((size_t)nt * KS + ks) * 32 + l] = W[(size_t)(4 * ks + (l & 3)) * ld + nt * 8 + (l >> 2)];
    return f;
  };
  const auto W1f = frag(W1, P.KS1, P.NT1), W2f = frag(W2, P.KS2, P.NT2);

  // ---- fused trunk operator MT = [[I, W2], [W1, W1 W2]] (rows [K | Yx | Ypsi],
  //      columns [S | u | bv]) for the collapsed trunk GEMM
  const int NTS = P.NT1;                 // S column tiles
  P.KY_LD = NVP + NXP + NUP;
  P.KSK = P.KY_LD / 4;
  P.U_OFF = NTS * 8;
  P.X_OFF = P.U_OFF + P.NU8;
  P.OUT_LD = P.X_OFF + r8(nx);
  P.NTT = P.OUT_LD / 8;
  std::vector<double> MTf;
  if (dec.collapsed && pl->n_trunk > 0) {
    const int ld = P.OUT_LD;
    std::vector<double> MT((size_t)P.KY_LD * ld, 0.0);
    // W1 rows: r < nx -> Bbar[r], NXP + j -> L[j] (row index into the Y block)
    auto w1 = [&](int yr, int v) -> double {
      if (yr < NXP) return yr < nx ? pb->Bbar[(size_t)yr * nv + v] : 0.0;
      const int j = yr - NXP;
      return j < nu ? pb->L[(size_t)j * nv + v] : 0.0;
    };
    auto w2 = [&](int v, int col) -> double {  // col in [U_OFF, OUT_LD)
      if (col < P.X_OFF) { const int j = col - P.U_OFF; return j < nu ? pb->Psi[(size_t)v * nu + j] : 0.0; }
      const int i = col - P.X_OFF;
      return i < nx ? pb->Phi[(size_t)v * nx + i] : 0.0;
    };
    for (int k = 0; k < nv; ++k) {           // K block: identity on S, W2 on [u | bv]
      MT[(size_t)k * ld + k] = 1.0;
      for (int col = P.U_OFF; col < ld; ++col) MT[(size_t)k * ld + col] = w2(k, col);
    }
    for (int yr = 0; yr < NXP + NUP; ++yr) {  // Y block: W1 on S, W1 W2 on [u | bv]
      double* row = &MT[(size_t)(NVP + yr) * ld];
      for (int v = 0; v < nv; ++v) row[v] = w1(yr, v);
      for (int col = P.U_OFF; col < ld; ++col) {
        double s = 0.0;
        for (int v = 0; v < nv; ++v) s += w1(yr, v) * w2(v, col);
        row[col] = s;
      }
    }
    MTf = frag(MT, P.KSK, P.NTT);
  }

  // ---- model vectors (padded)
  auto padv = [](const double* v, int n, int np) {
    std::vector<double> o(np, 0.0);
    std::copy(v, v + n, o.begin());
    return o;
  };
  std::vector<double> adiag(NXP, 0.0);
  for (int i = 0; i < nx; ++i) adiag[i] = pb->A[(size_t)i * nx + i];
  P.diagA = diag ? 1 : 0;

  // ---- tree arrays
  std::vector<int> anc(n_nodes), cs(n_nodes), ce(n_nodes), est(E);
  std::vector<double> inv2p(E), pe(E);
  for (int n = 0; n < n_nodes; ++n) {
    anc[n] = (int)pb->anc[n];
    cs[n] = (int)pb->child_start[n];
    ce[n] = (int)pb->child_stop[n];
  }
  for (int j = 0; j < N; ++j)
    for (int64_t n = pb->stage_starts[j + 1]; n < pb->stage_starts[j + 2]; ++n) est[n - 1] = j;
  for (int e = 0; e < E; ++e) {
    pe[e] = pb->prob[e + 1];
    inv2p[e] = 1.0 / (2.0 * pb->prob[e + 1]);
  }

  // ---- scaling
  const bool scaled = pb->sig_stage && pb->zeta_stage && pb->psi_stage;
  std::vector<double> sig(N, 1.0), zeta(N, 1.0), psi((size_t)N * NUP, 1.0), psi_c((size_t)N * nu, 1.0);
  if (scaled) {
    for (int j = 0; j < N; ++j) {
      sig[j] = pb->sig_stage[j];
      zeta[j] = pb->zeta_stage[j];
      for (int k = 0; k < nu; ++k) psi[(size_t)j * NUP + k] = psi_c[(size_t)j * nu + k] = pb->psi_stage[(size_t)j * nu + k];
    }
  }
  P.scaled = scaled ? 1 : 0;

  int rc = 0;
  double *d_W1f, *d_W2f, *d_adiag, *d_A, *d_xs, *d_xmin, *d_xmax, *d_umin, *d_umax, *d_sig, *d_zeta, *d_psi,
      *d_inv2p, *d_pe, *d_Wu, *d_E, *d_EpinvT, *d_B;
  int *d_anc, *d_cs, *d_ce, *d_est, *d_lt, *d_ts, *d_sr, *d_re;
  rc |= pl->upload(&d_W1f, W1f.data(), W1f.size());
  rc |= pl->upload(&d_W2f, W2f.data(), W2f.size());
  rc |= pl->upload(&d_adiag, adiag.data(), adiag.size());
  rc |= pl->upload(&d_A, pb->A, (size_t)nx * nx);
  rc |= pl->upload(&d_B, pb->B, (size_t)nx * nu);
  const auto xs = padv(pb->x_s, nx, NXP), xmn = padv(pb->x_min, nx, NXP), xmx = padv(pb->x_max, nx, NXP);
  const auto umn = padv(pb->u_min, nu, NUP), umx = padv(pb->u_max, nu, NUP);
  rc |= pl->upload(&d_xs, xs.data(), xs.size());
  rc |= pl->upload(&d_xmin, xmn.data(), xmn.size());
  rc |= pl->upload(&d_xmax, xmx.data(), xmx.size());
  rc |= pl->upload(&d_umin, umn.data(), umn.size());
  rc |= pl->upload(&d_umax, umx.data(), umx.size());
  rc |= pl->upload(&d_sig, sig.data(), sig.size());
  rc |= pl->upload(&d_zeta, zeta.data(), zeta.size());
  rc |= pl->upload(&d_psi, psi.data(), psi.size());
  rc |= pl->upload(&pl->psi_c, psi_c.data(), psi_c.size());
  pl->sig_c = d_sig;
  pl->zeta_c = d_zeta;
  {  // reciprocal scaling tables for the epilogue's quotients
    std::vector<double> rs(N), rz(N), rp(psi.size());
    for (int j = 0; j < N; ++j) { rs[j] = 1.0 / sig[j]; rz[j] = 1.0 / zeta[j]; }
    for (size_t k = 0; k < psi.size(); ++k) rp[k] = 1.0 / psi[k];
    double *d_rs, *d_rz, *d_rp;
    rc |= pl->upload(&d_rs, rs.data(), rs.size());
    rc |= pl->upload(&d_rz, rz.data(), rz.size());
    rc |= pl->upload(&d_rp, rp.data(), rp.size());
    P.sig_rcp = d_rs; P.zeta_rcp = d_rz; P.psi_rcp = d_rp;
  }
  rc |= pl->upload(&d_inv2p, inv2p.data(), inv2p.size());
  rc |= pl->upload(&d_pe, pe.data(), pe.size());
  rc |= pl->upload(&d_Wu, pb->Wu, (size_t)nu * nu);
  rc |= pl->upload(&d_E, pb->E, (size_t)ne * nu);
  rc |= pl->upload(&d_EpinvT, pb->E_pinvT, (size_t)ne * nu);
  rc |= pl->upload(&d_anc, anc.data(), anc.size());
  rc |= pl->upload(&d_cs, cs.data(), cs.size());
  rc |= pl->upload(&d_ce, ce.data(), ce.size());
  rc |= pl->upload(&d_est, est.data(), est.size());
  rc |= pl->upload(&d_lt, dec.lvl_tiles.data(), dec.lvl_tiles.size());
  rc |= pl->upload(&d_ts, dec.tile_seg.data(), dec.tile_seg.size());
  rc |= pl->upload(&d_sr, dec.seg_row.data(), dec.seg_row.size());
  rc |= pl->upload(&d_re, dec.row_edge.data(), dec.row_edge.size());
  // state.  The buffers the persistent kernels touch every iteration (both dual
  // slots, the ergodic averages, the static per-edge vectors) come from one arena
  // with a skew between consecutive buffers: the kernel reads the same row of
  // several of them back to back, and buffer bases that map those rows onto the
  // same L2 sets / DRAM banks measurably slow it down (identical SMPC8 plans at
  // different cudaMalloc addresses ran 58-67 us/iteration; tools/layout_probe.py)
  const size_t yblk = 2 * (size_t)E * NXP + (size_t)E * NUP;
  {
    const char* pe = std::getenv("TSMPC_ARENA_PAD");
    // bytes, skew per buffer (a multiple of 16: the epilogues use 16-byte accesses)
    const size_t pad = ((pe ? (size_t)std::atoll(pe) : kArenaPad) + 15) / 16 * 16;
    const size_t sizes[] = {yblk, yblk, (size_t)n_nodes * NXP, (size_t)E * NUP, (size_t)E * NUP,
                            (size_t)E * NXP, (size_t)E * NVP};
    double** dst[] = {&pl->Y0, &pl->Y1, &pl->XAVG, &pl->UAVG, &pl->UHAT, &pl->EVEC, &pl->BETA_S};
    size_t total = 0;
    std::vector<size_t> off;
    for (size_t i = 0; i < sizeof(sizes) / sizeof(sizes[0]); ++i) {
      off.push_back(total);
      total += ((sizes[i] * sizeof(double) + 255) / 256) * 256 + (i + 1) * pad;
    }
    char* arena = nullptr;
    rc |= pl->alloc(&arena, total);
    if (rc) return bail(0);
    for (size_t i = 0; i < off.size(); ++i) *dst[i] = reinterpret_cast<double*>(arena + off[i] + (i + 1) * pad);
  }
  rc |= pl->alloc(&pl->WB, yblk);
  rc |= pl->alloc(&pl->PY, yblk);
  rc |= pl->alloc(&pl->X, (size_t)n_nodes * NXP);
  rc |= pl->alloc(&pl->XL, (size_t)n_nodes * NXP);
  rc |= pl->alloc(&pl->XF, (size_t)n_nodes * NXP);
  rc |= pl->alloc(&pl->Z0X, (size_t)n_nodes * NXP);
  rc |= pl->alloc(&pl->U, (size_t)E * NUP);
  rc |= pl->alloc(&pl->UL, (size_t)E * NUP);
  rc |= pl->alloc(&pl->Z0U, (size_t)E * NUP);
  rc |= pl->alloc(&pl->UF, (size_t)E * NUP);
  rc |= pl->alloc(&pl->XIT, (size_t)E * NUP);
  rc |= pl->alloc(&pl->INC, (size_t)E * NUP);
  rc |= pl->alloc(&pl->T, (size_t)E * NVP);
  rc |= pl->alloc(&pl->GG, (size_t)E * NVP);
  rc |= pl->alloc(&pl->BETA, (size_t)E * NVP);
  rc |= pl->alloc(&pl->BETA0, (size_t)E * NVP);
  rc |= pl->alloc(&pl->XIQG, (size_t)E * NXP);
  rc |= pl->alloc(&pl->GDD, (size_t)E * NXP);
  rc |= pl->alloc(&pl->UB, (size_t)E * NXP);
  rc |= pl->alloc(&pl->JRHS, (size_t)E * ne);
  rc |= pl->alloc(&pl->PRICES, (size_t)N * nu);
  rc |= pl->alloc(&pl->Q, (size_t)nu);
  rc |= pl->alloc(&pl->P, (size_t)NXP);
  rc |= pl->alloc(&pl->COLS, (size_t)E * 10);
  rc |= pl->alloc(&pl->ROWS, (size_t)E * 6);
  rc |= pl->alloc(&pl->RED, 16);
  rc |= pl->alloc(&pl->ABORT, 1);
  rc |= pl->alloc(&pl->DYK, 256);
  rc |= pl->alloc(&pl->TIMERS, 16 + 8 * 256);  // phase timers + timeline stamps (timer builds)
  int *d_te = nullptr, *d_tsp = nullptr, *d_tpos = nullptr, *d_pp = nullptr, *d_pl = nullptr,
      *d_tc0 = nullptr, *d_tpar = nullptr;
  double *d_MTf = nullptr, *d_KY = nullptr, *d_OUT = nullptr;
  if (dec.collapsed) {
    const size_t T = std::max<size_t>(1, dec.trunk_edge.size());
    rc |= pl->upload(&d_tpos, dec.trunk_pos.data(), dec.trunk_pos.size());
    rc |= pl->upload(&d_tsp, dec.trunk_stage_ptr.data(), dec.trunk_stage_ptr.size());
    if (!dec.trunk_edge.empty()) {
      rc |= pl->upload(&d_te, dec.trunk_edge.data(), dec.trunk_edge.size());
      rc |= pl->upload(&d_tc0, dec.trunk_child0.data(), dec.trunk_child0.size());
      rc |= pl->upload(&d_tpar, dec.trunk_parent.data(), dec.trunk_parent.size());
      rc |= pl->upload(&d_pp, dec.path_ptr.data(), dec.path_ptr.size());
      rc |= pl->upload(&d_pl, dec.path_list.data(), dec.path_list.size());
      rc |= pl->upload(&d_MTf, MTf.data(), MTf.size());
    }
    rc |= pl->alloc(&d_KY, T * P.KY_LD);
    rc |= pl->alloc(&d_OUT, T * P.OUT_LD);
  }
  if (rc) return bail(0);
  P.trunk_edge = d_te; P.trunk_stage_ptr = d_tsp; P.trunk_pos = d_tpos; P.trunk_child0 = d_tc0;
  P.trunk_parent = d_tpar;
  {  // the component sweep stages 2 x T x (components per CTA) doubles in the tile region
    const long long per_cta = (nv + nx + nu + dec.n_ctas - 1) / dec.n_ctas;
    P.trunk_smem = (2LL * pl->n_trunk * per_cta <= (long long)P.META_OFF) ? 1 : 0;
  }
  P.path_ptr = d_pp; P.path_list = d_pl; P.MTf = d_MTf; P.KY = d_KY; P.OUT = d_OUT;

  P.a_diag = d_adiag; P.A = d_A; P.W1f = d_W1f; P.W2f = d_W2f;
  P.x_s = d_xs; P.x_min = d_xmin; P.x_max = d_xmax; P.u_min = d_umin; P.u_max = d_umax;
  P.sig_stage = d_sig; P.zeta_stage = d_zeta; P.psi_stage = d_psi;
  P.anc = d_anc; P.child_start = d_cs; P.child_stop = d_ce; P.edge_stage = d_est; P.inv2p = d_inv2p;
  P.lvl_tiles = d_lt; P.tile_seg = d_ts; P.seg_row = d_sr; P.row_edge = d_re;
  P.xavg = pl->XAVG; P.uavg = pl->UAVG; P.X = pl->X; P.U = pl->U; P.T = pl->T;
  P.XIQG = pl->XIQG; P.GG = pl->GG; P.p = pl->P;
  P.timers = pl->TIMERS;
  P.timer_cta = std::getenv("TSMPC_TIMER_CTA") ? std::atoi(std::getenv("TSMPC_TIMER_CTA")) : 0;

  pl->d_est_c = d_est; pl->d_anc_c = d_anc; pl->d_cs_c = d_cs; pl->d_ce_c = d_ce;
  pl->d_pe_c = d_pe; pl->d_B_c = d_B;
  EdgeCtx& c = pl->ctx;
  c.nx = nx; c.nu = nu; c.ne = ne; c.E = E; c.NXP = NXP; c.NUP = NUP;
  c.Wx = pb->Wx; c.gamma_d = pb->gamma_d; c.W_alpha = pb->W_alpha;
  c.edge_stage = d_est; c.anc = d_anc;
  c.sig_stage = scaled ? d_sig : nullptr;
  c.zeta_stage = scaled ? d_zeta : nullptr;
  c.psi_stage = scaled ? d_psi : nullptr;
  c.x_s = d_xs; c.x_min = d_xmin; c.x_max = d_xmax; c.u_min = d_umin; c.u_max = d_umax;
  c.prob_edge = d_pe; c.prices = pl->PRICES; c.q = pl->Q; c.Wu = d_Wu; c.Emat = d_E; c.Ej = d_E;
  c.EpinvT = d_EpinvT; c.jrhs = pl->JRHS; c.gdd = pl->GDD; c.B = d_B;
  c.a_diag = diag ? d_adiag : nullptr; c.A = d_A;

  // ---- structured-basis (sparse) kernel plan
  {
    const char* force = getenv("TSMPC_FORCE_DENSE");
    if (!diag) pl->sp_why = "A is not diagonal";
    else if (!pb->Ls || !pb->lam_s || !pb->Ms) pl->sp_why = "no structured basis supplied";
    else if (force && force[0] == '1') pl->sp_why = "disabled by TSMPC_FORCE_DENSE";
    else {
      SparseTreeIn ti{N, n_nodes, pb->stage_starts, pb->anc, pb->child_start, pb->child_stop, pb->prob};
      SparseOpsIn oi{nx, nu, nv, pb->B, pb->Ls, pb->lam_s};
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, apg_sparse_kernel);  // static shared memory counts against the opt-in limit
      cudaFuncAttributes fw{}, fw2{};
      cudaFuncGetAttributes(&fw, sparse_kernel_fn(1, nx, false));
      cudaFuncGetAttributes(&fw2, sparse_kernel_fn(1, nx, true));
      fw.sharedSizeBytes = std::max(fw.sharedSizeBytes, fw2.sharedSizeBytes);
      SparseHostPlan hp = choose_sparse_plan(ti, oi, NXP, NUP, NVP, pl->sm_count,
                                             (size_t)prop.sharedMemPerBlockOptin - fa.sharedSizeBytes,
                                             (size_t)prop.sharedMemPerBlockOptin - fw.sharedSizeBytes, shard,
                                             shard ? srank : 0, shard ? sworld : 1);
      // fill rows through HBM (FG) for multi-tile / sharded wide CTAs: the kernel variant
      // compiled with them (the others keep the one-tile code as it was)
      if (!hp.S.wide || (std::getenv("TSMPC_NO_FG") && !hp.S.rows_window)) hp.S.FL = 0;
      const void* kfn = sparse_kernel_fn(hp.S.wide, nx, hp.S.FL > 0);
      int occ_s = 0;
      if (hp.ok) {
        // the attribute is per kernel, shared by every plan of the process: the
        // opt-in maximum (not this plan's size, which a plan needing more would trip on)
        cudaFuncAttributes fk{};
        cudaFuncGetAttributes(&fk, kfn);
        const int smem_max = (int)(prop.sharedMemPerBlockOptin - fk.sharedSizeBytes);
        if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max) != cudaSuccess) {
          hp.ok = false;
          hp.why = "cannot reserve shared memory for the sparse kernel";
          cudaGetLastError();
        } else {
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, kfn, kThreadsS, hp.smem);
          if (occ_s < 1) { hp.ok = false; hp.why = "sparse kernel does not fit on an SM"; }
        }
      }
      if (hp.ok) {
        int *d_meta, *d_mptr, *d_ts, *d_spi;
        double* d_spv;
        rc |= pl->upload(&d_meta, hp.meta.data(), hp.meta.size());
        rc |= pl->upload(&d_mptr, hp.meta_ptr.data(), hp.meta_ptr.size());
        rc |= pl->upload(&d_ts, hp.tsched.data(), hp.tsched.size());
        rc |= pl->upload(&d_spi, hp.spi.data(), hp.spi.size());
        rc |= pl->upload(&d_spv, hp.spv.data(), hp.spv.size());
        {  // M (structured basis = L M) by column, zeros dropped: beta_s = beta M per edge
          std::vector<int> mc(1, 0), mr;
          std::vector<double> mv;
          for (int k = 0; k < nv; ++k) {
            for (int j = 0; j < nv; ++j)
              if (pb->Ms[(size_t)j * nv + k] != 0.0) {
                mr.push_back(j);
                mv.push_back(pb->Ms[(size_t)j * nv + k]);
              }
            mc.push_back((int)mr.size());
          }
          mc.insert(mc.end(), mr.begin(), mr.end());
          rc |= pl->upload(&pl->MSC, mc.data(), mc.size());
          rc |= pl->upload(&pl->MS, mv.data(), std::max<size_t>(1, mv.size()));
        }
        rc |= pl->alloc(&pl->TG, (size_t)E * NVP);
        if (hp.S.FL > 0) rc |= pl->alloc(&pl->FG, (size_t)E * hp.S.FL);
        rc |= pl->alloc(&pl->KY_S, (size_t)std::max(1, hp.n_trunk) * P.KY_LD);
        if (rc) return bail(0);
        SParams& S = pl->sbase;
        S = hp.S;
        S.spi = d_spi; S.spv = d_spv; S.meta = d_meta; S.meta_ptr = d_mptr; S.tsched = d_ts;
        S.beta_s = pl->BETA_S; S.TG = pl->TG; S.FG = pl->FG;
        S.a_unit = 1;
        for (int i = 0; i < nx; ++i)
          if (pb->A[(size_t)i * nx + i] != 1.0) S.a_unit = 0;
        S.HS_LD = NVP + NXP;
        S.abort_flag = pl->ABORT;
        if (S.split) {
          int* d_tpi;
          double* d_tpv;
          rc |= pl->upload(&d_tpi, hp.tpi.data(), hp.tpi.size());
          rc |= pl->upload(&d_tpv, hp.tpv.data(), hp.tpv.size());
          S.tpi = d_tpi;
          S.tpv = d_tpv;
          rc |= pl->alloc(&pl->TR, (size_t)std::max(1, hp.n_trunk) * S.TR_LD);
          rc |= pl->alloc(&pl->SUBCTR, 4);
          S.split_flags = std::getenv("TSMPC_SPLIT_GRID") ? 0 : 1;
          if (rc) return bail(0);
          S.TR = pl->TR;
          S.sub_ctr = pl->SUBCTR;
        }
        if (shard) {
          unsigned char* d_tow;
          rc |= pl->upload(&d_tow, hp.towned.data(), std::max<size_t>(1, hp.towned.size()));
          rc |= pl->alloc(&pl->HS, (size_t)std::max(1, hp.n_trunk) * S.HS_LD);
          S.cut = hp.cut ? 1 : 0;
          S.n_xch = hp.n_xch;
          S.XCH_LD = hp.cut ? P.KY_LD + NXP : S.HS_LD;
          if (hp.cut) rc |= pl->alloc(&pl->XCH, (size_t)std::max(1, hp.n_xch) * S.XCH_LD);
          else pl->XCH = pl->HS;  // every position's head sums, exchanged in place
          // receive rows and arrival counter of the in-kernel exchange (own allocations:
          // other ranks map them through CUDA IPC handles)
          rc |= pl->alloc(&pl->RX, 2 * (size_t)sworld * std::max(1, hp.n_xch) * S.XCH_LD);
          rc |= pl->alloc(&pl->RXCNT, 1);
          if (rc) return bail(0);
          S.RX = pl->RX;
          S.RXCNT = pl->RXCNT;
          S.rank = srank;
          S.world = sworld;
          S.sharded = 1;
          S.HS = pl->HS;
          S.XCH = pl->XCH;
          S.towned = d_tow;
          pl->sharded = true;
          pl->rank = srank;
          pl->world = sworld;
          pl->total_chains = hp.total_chains;
          pl->owned_edges = hp.owned_edges;
          pl->trunk_edges = hp.trunk_edge;
          pl->result_edges = hp.result_edges;
          // rows another rank computes (or, replicated, rank 0 counts): zeroed before
          // the cross-rank assembly of the averages and the dual
          {
            std::vector<char> keep(E, 0);
            for (int e : hp.result_edges) keep[e] = 1;
            if (srank != 0)
              for (size_t tp = 0; tp < hp.trunk_edge.size(); ++tp)
                if (hp.trole[tp] == kRoleMixed) keep[hp.trunk_edge[tp]] = 0;
            for (int e = 0; e < E; ++e)
              if (!keep[e]) pl->zero_edges.push_back(e);
          }
          if (pl->zero_edges.empty()) pl->zero_edges.push_back(-1);  // (a valid upload; never read)
          rc |= pl->upload(&pl->d_zero, pl->zero_edges.data(), pl->zero_edges.size());
          if (pl->zero_edges[0] < 0) pl->zero_edges.clear();
          if (rc) return bail(0);
        }
        pl->use_sparse = true;
        pl->sp_ctas = hp.n_ctas;
        pl->sp_smem = hp.smem;
        pl->sp_resident = hp.resident_ctas;
        pl->sp_tiles = hp.n_tiles;
        pl->sp_trunk = hp.n_trunk;
      } else {
        pl->sp_why = hp.why;
      }
    }
  }

  if (shard && !pl->use_sparse) {
    fail(TSMPC_ERR_VALIDATION, "subtree sharding needs the structured-basis kernel (%s)", pl->sp_why.c_str());
    return bail(0);
  }
  if (shard && nccl_id) {  // without an id: a local shard plan for tsmpc_solve_group
    std::string why;
    pl->nccl = nccl_api(why);
    if (!pl->nccl) { fail(TSMPC_ERR_NCCL, "%s", why.c_str()); return bail(0); }
    NcclApi::UniqueId id;
    std::memcpy(id.internal, nccl_id, sizeof(id.internal));
    const int nr = pl->nccl->CommInitRank(&pl->comm, sworld, id, srank);
    if (nr != 0) {
      pl->comm = nullptr;
      fail(TSMPC_ERR_NCCL, "ncclCommInitRank(rank %d of %d): %s", srank, sworld, pl->nccl->GetErrorString(nr));
      return bail(0);
    }
  }

  cudaFuncSetAttribute(gap_dykstra_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(sizeof(double) * (2 * 64 * 128 + 8 * 448 + 1) + sizeof(int) * (2 * 64 * 128 + 200)));
  cudaFuncSetAttribute(gap_dykstra_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(sizeof(double) * (2 * 64 * 128 + 8 * 448 + 1) + sizeof(int) * (2 * 64 * 128 + 200)));
  {  // sparse junction operators for the gap's Dykstra projection
    std::vector<int> erp{0}, eri, pcp{0}, pci;
    std::vector<double> erv, pcv;
    for (int k = 0; k < ne; ++k) {
      for (int j = 0; j < nu; ++j)
        if (pb->E[(size_t)k * nu + j] != 0.0) { eri.push_back(j); erv.push_back(pb->E[(size_t)k * nu + j]); }
      erp.push_back((int)eri.size());
    }
    for (int j = 0; j < nu; ++j) {
      for (int k = 0; k < ne; ++k)
        if (pb->E_pinvT[(size_t)k * nu + j] != 0.0) { pci.push_back(k); pcv.push_back(pb->E_pinvT[(size_t)k * nu + j]); }
      pcp.push_back((int)pci.size());
    }
    int *d_erp, *d_eri, *d_pcp, *d_pci;
    double *d_erv, *d_pcv;
    rc |= pl->upload(&d_erp, erp.data(), erp.size());
    rc |= pl->upload(&d_eri, eri.data(), std::max<size_t>(1, eri.size()));
    rc |= pl->upload(&d_erv, erv.data(), std::max<size_t>(1, erv.size()));
    rc |= pl->upload(&d_pcp, pcp.data(), pcp.size());
    rc |= pl->upload(&d_pci, pci.data(), std::max<size_t>(1, pci.size()));
    rc |= pl->upload(&d_pcv, pcv.data(), std::max<size_t>(1, pcv.size()));
    if (rc) return bail(0);
    c.er_ptr = d_erp; c.er_idx = d_eri; c.er_val = d_erv; c.er_nnz = (int)eri.size();
    c.pc_ptr = d_pcp; c.pc_idx = d_pci; c.pc_val = d_pcv; c.pc_nnz = (int)pci.size();
    {  // Wu by row for the gap's smooth cost
      std::vector<int> wp{0}, wi;
      std::vector<double> wv;
      for (int j = 0; j < nu; ++j) {
        for (int k = 0; k < nu; ++k)
          if (pb->Wu[(size_t)j * nu + k] != 0.0) { wi.push_back(k); wv.push_back(pb->Wu[(size_t)j * nu + k]); }
        wp.push_back((int)wi.size());
      }
      if (wi.empty()) { wi.push_back(0); wv.push_back(0.0); }
      int *d_wp, *d_wi;
      double* d_wv;
      rc |= pl->upload(&d_wp, wp.data(), wp.size());
      rc |= pl->upload(&d_wi, wi.data(), wi.size());
      rc |= pl->upload(&d_wv, wv.data(), wv.size());
      if (rc) return bail(0);
      c.wu_ptr = d_wp; c.wu_idx = d_wi; c.wu_val = d_wv;
    }
    {  // B by row for the gap's ub = u B'
      std::vector<int> bp{0}, bi;
      std::vector<double> bv;
      for (int i = 0; i < nx; ++i) {
        for (int j = 0; j < nu; ++j)
          if (pb->B[(size_t)i * nu + j] != 0.0) { bi.push_back(j); bv.push_back(pb->B[(size_t)i * nu + j]); }
        bp.push_back((int)bi.size());
      }
      if (bi.empty()) { bi.push_back(0); bv.push_back(0.0); }
      int *d_bp, *d_bi;
      double* d_bv;
      rc |= pl->upload(&d_bp, bp.data(), bp.size());
      rc |= pl->upload(&d_bi, bi.data(), bi.size());
      rc |= pl->upload(&d_bv, bv.data(), bv.size());
      if (rc) return bail(0);
      c.bq_ptr = d_bp; c.bq_idx = d_bi; c.bq_val = d_bv;
    }
    // junction rows with disjoint flow supports -> one Dykstra component per row
    std::vector<int> owner(nu, -1);
    bool disjoint = ne > 0;
    for (int k = 0; k < ne && disjoint; ++k)
      for (int j = 0; j < nu; ++j)
        if (pb->E[(size_t)k * nu + j] != 0.0 || pb->E_pinvT[(size_t)k * nu + j] != 0.0) {
          if (owner[j] >= 0 && owner[j] != k) disjoint = false;
          owner[j] = k;
        }
    std::vector<DykComp> comps;
    std::vector<int> freeu;
    for (int k = 0; k < ne && disjoint; ++k) {
      DykComp q{};
      q.row = k;
      for (int j = 0; j < nu; ++j) {
        if (owner[j] != k) continue;
        if (q.n == kDykCU) { disjoint = false; break; }
        q.u[q.n] = j;
        q.e[q.n] = pb->E[(size_t)k * nu + j];
        q.p[q.n] = pb->E_pinvT[(size_t)k * nu + j];
        if (q.e[q.n] != 0.0) q.emask |= 1 << q.n;
        if (q.p[q.n] != 0.0) q.pmask |= 1 << q.n;
        ++q.n;
      }
      if (q.n > 0) comps.push_back(q);
    }
    for (int j = 0; j < nu; ++j)
      if (owner[j] < 0) freeu.push_back(j);
    if (disjoint && !comps.empty()) {
      const int nfree = (int)freeu.size();
      if (freeu.empty()) freeu.push_back(0);  // keep the device array non-empty
      rc |= pl->alloc(&pl->DYKC, comps.size());
      rc |= pl->upload(&pl->DYKF, freeu.data(), freeu.size());
      if (rc) return bail(0);
      if (cudaMemcpyAsync(pl->DYKC, comps.data(), sizeof(DykComp) * comps.size(), cudaMemcpyHostToDevice,
                          pl->stream) != cudaSuccess) {
        fail(TSMPC_ERR_CUDA, "upload of the Dykstra components failed");
        return bail(0);
      }
      pl->dyk_ncomp = (int)comps.size();
      pl->dyk_nfree = nfree;
    }
  }

  int occ_d = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_d, gap_project_dykstra_kernel, 256, 0);
  pl->dyk_blocks = std::max(1, std::min(occ_d, 4)) * pl->sm_count;
  if (cudaStreamSynchronize(pl->stream) != cudaSuccess) {
    fail(TSMPC_ERR_CUDA, "plan upload failed: %s", cudaGetErrorString(cudaGetLastError()));
    return bail(0);
  }
  return pl;
}

tsmpc_plan* tsmpc_plan_create(const tsmpc_problem* pb, int device) {
  return plan_create_impl(pb, device, -1, 1, nullptr);
}

int tsmpc_nccl_unique_id(uint8_t* out) {
  if (!out) return fail(TSMPC_ERR_ARGUMENT, "null argument");
  std::string why;
  const NcclApi* api = nccl_api(why);
  if (!api) return fail(TSMPC_ERR_NCCL, "%s", why.c_str());
  NcclApi::UniqueId id;
  const int r = api->GetUniqueId(&id);
  if (r != 0) return fail(TSMPC_ERR_NCCL, "ncclGetUniqueId: %s", api->GetErrorString(r));
  std::memcpy(out, id.internal, sizeof(id.internal));
  return TSMPC_OK;
}

tsmpc_plan* tsmpc_plan_create_shard(const tsmpc_problem* pb, int device, int32_t rank, int32_t world,
                                    const uint8_t* nccl_id) {
  if (world < 1 || rank < 0 || rank >= world) {
    fail(TSMPC_ERR_ARGUMENT, "invalid shard arguments (rank %d of %d)", rank, world);
    return nullptr;
  }
  return plan_create_impl(pb, device, rank, world, nccl_id);
}

// ---------------------------------------------------------------- peer exchange
namespace {
// the ranks' receive rows / arrival counters as this device sees them -> SParams
int peer_setup(tsmpc_plan* pl, const std::vector<double*>& rx, const std::vector<unsigned long long*>& cnt,
               unsigned long long expect) {
  CU(cudaSetDevice(pl->device));
  double** d_rx = nullptr;
  unsigned long long** d_cnt = nullptr;
  int rc = pl->upload(&d_rx, rx.data(), rx.size());
  rc |= pl->upload(&d_cnt, cnt.data(), cnt.size());
  if (rc) return rc;
  CU(cudaStreamSynchronize(pl->stream));
  pl->sbase.peer_rx = d_rx;
  pl->sbase.peer_cnt = d_cnt;
  pl->sbase.xch_expect = expect;
  pl->peer_on = true;
  return TSMPC_OK;
}
// peer exchange blob: [RX handle | RXCNT handle | ctas, rank, world, fg | exchange doubles |
// exchange generations run so far (the ranks' arrival counters must agree)]
struct PeerBlob {
  cudaIpcMemHandle_t rx, cnt;
  int32_t ctas, rank, world, fg;
  int64_t xn;
  uint64_t xgen;
};
static_assert(sizeof(PeerBlob) <= TSMPC_PEER_BLOB_BYTES, "peer blob size");
bool peer_capable(const tsmpc_plan* pl) {
  return pl->sharded && pl->use_sparse && pl->sbase.wide && pl->sbase.FL > 0 && pl->RX && pl->RXCNT;
}
}  // namespace

int tsmpc_plan_peer_handles(const tsmpc_plan* pl, uint8_t* blob) {
  if (!pl || !blob) return fail(TSMPC_ERR_ARGUMENT, "null argument");
  if (!peer_capable(pl)) return fail(TSMPC_ERR_VALIDATION, "not a wide shard plan: no in-kernel exchange");
  CU(cudaSetDevice(pl->device));
  PeerBlob b{};
  CU(cudaIpcGetMemHandle(&b.rx, pl->RX));
  CU(cudaIpcGetMemHandle(&b.cnt, pl->RXCNT));
  b.ctas = pl->sp_ctas;
  b.rank = pl->rank;
  b.world = pl->world;
  b.fg = pl->sbase.FL > 0 ? 1 : 0;
  b.xn = (int64_t)pl->sbase.n_xch * pl->sbase.XCH_LD;
  b.xgen = pl->xgen;
  std::memset(blob, 0, TSMPC_PEER_BLOB_BYTES);
  std::memcpy(blob, &b, sizeof b);
  return TSMPC_OK;
}

int tsmpc_plan_peer_open(tsmpc_plan* pl, const uint8_t* blobs, int32_t world) {
  if (!pl || !blobs) return fail(TSMPC_ERR_ARGUMENT, "null argument");
  if (!peer_capable(pl)) return fail(TSMPC_ERR_VALIDATION, "not a wide shard plan: no in-kernel exchange");
  if (world != pl->world) return fail(TSMPC_ERR_ARGUMENT, "%d blobs for a world of %d", world, pl->world);
  if (pl->peer_on) return TSMPC_OK;
  CU(cudaSetDevice(pl->device));
  std::vector<double*> rx(world);
  std::vector<unsigned long long*> cnt(world);
  std::vector<void*> opened;
  auto undo = [&]() {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    cudaGetLastError();
  };
  const int64_t xn = (int64_t)pl->sbase.n_xch * pl->sbase.XCH_LD;
  for (int p = 0; p < world; ++p) {
    PeerBlob b;
    std::memcpy(&b, blobs + (size_t)p * TSMPC_PEER_BLOB_BYTES, sizeof b);
    if (b.rank != p || b.world != world || b.ctas != pl->sp_ctas || b.xn != xn || !b.fg || b.xgen != pl->xgen) {
      undo();
      return fail(TSMPC_ERR_VALIDATION,
                  "peer %d: plan mismatch (rank %d, world %d, %d CTAs, %lld exchange doubles, generation %llu)", p,
                  b.rank, b.world, b.ctas, (long long)b.xn, (unsigned long long)b.xgen);
    }
    if (p == pl->rank) {
      rx[p] = pl->RX;
      cnt[p] = pl->RXCNT;
      continue;
    }
    void* a = nullptr;
    void* c = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&a, b.rx, cudaIpcMemLazyEnablePeerAccess);
    if (e == cudaSuccess) {
      opened.push_back(a);
      e = cudaIpcOpenMemHandle(&c, b.cnt, cudaIpcMemLazyEnablePeerAccess);
      if (e == cudaSuccess) opened.push_back(c);
    }
    if (e != cudaSuccess) {
      undo();
      return fail(TSMPC_ERR_CUDA, "cudaIpcOpenMemHandle (rank %d's exchange buffers): %s", p, cudaGetErrorString(e));
    }
    rx[p] = static_cast<double*>(a);
    cnt[p] = static_cast<unsigned long long*>(c);
  }
  const int rc = peer_setup(pl, rx, cnt, (unsigned long long)world * pl->sp_ctas);
  if (rc) {
    undo();
    return rc;
  }
  pl->ipc_mapped.insert(pl->ipc_mapped.end(), opened.begin(), opened.end());
  return TSMPC_OK;
}

int tsmpc_plan_peer_close(tsmpc_plan* pl) {
  if (!pl) return fail(TSMPC_ERR_ARGUMENT, "null argument");
  pl->peer_on = false;  // back to the two launches + ncclAllReduce per iteration
  pl->sbase.peer_rx = nullptr;
  pl->sbase.peer_cnt = nullptr;
  return TSMPC_OK;
}

int tsmpc_plan_edges(const tsmpc_plan* pl, int32_t which, int64_t* out, int64_t cap) {
  if (!pl) return fail(TSMPC_ERR_ARGUMENT, "null argument");
  std::vector<int> all;
  const std::vector<int>* v = &all;
  if (which == 0) {  // edges whose results this plan computes
    if (!pl->sharded) {
      for (int e = 0; e < pl->E; ++e) all.push_back(e);
    } else {
      all = pl->result_edges;  // own chains, own and mixed trunk positions
    }
  } else if (which == 1) {
    v = &pl->trunk_edges;
  } else {
    return fail(TSMPC_ERR_ARGUMENT, "which must be 0 (owned) or 1 (trunk)");
  }
  if (out)
    for (int64_t i = 0; i < cap && i < (int64_t)v->size(); ++i) out[i] = (*v)[i];
  return (int)v->size();
}

void tsmpc_plan_destroy(tsmpc_plan* plan) { delete plan; }

int tsmpc_describe_tree(const tsmpc_problem* pb, int32_t max_ctas, int32_t collapse, int64_t* info,
                        int32_t n) {
  if (!pb || !info || !pb->anc || !pb->child_start || !pb->child_stop || !pb->stage_starts)
    return fail(TSMPC_ERR_ARGUMENT, "null argument");
  if (pb->n_nodes < 2 || pb->N < 1) return fail(TSMPC_ERR_DIMENSION, "tree too small");
  Decomposition dec;
  const int rc = decompose(pb, std::max(1, (int)max_ctas), collapse != 0, dec);
  if (rc) return rc;
  int64_t max_rows = 0, max_tiles = 0;
  for (int c = 0; c < dec.n_ctas; ++c) {
    int64_t rows = 0, tiles = 0;
    for (int l = 0; l < dec.n_levels; ++l)
      for (int t = dec.lvl_tiles[(size_t)l * dec.n_ctas + c]; t < dec.lvl_tiles[(size_t)l * dec.n_ctas + c + 1]; ++t) {
        rows += dec.seg_row[dec.tile_seg[t + 1]] - dec.seg_row[dec.tile_seg[t]];
        ++tiles;
      }
    max_rows = std::max(max_rows, rows);
    max_tiles = std::max(max_tiles, tiles);
  }
  int64_t max_path = 0;
  for (size_t t = 0; t + 1 < dec.path_ptr.size(); ++t)
    max_path = std::max<int64_t>(max_path, dec.path_ptr[t + 1] - dec.path_ptr[t]);
  const int64_t vals[] = {dec.n_levels, dec.n_ctas, (int64_t)dec.tile_seg.size() - 1,
                          (int64_t)dec.seg_row.size() - 1, (int64_t)dec.row_edge.size(),
                          (int64_t)dec.trunk_edge.size(), max_rows, max_tiles, max_path};
  for (int i = 0; i < n && i < (int)(sizeof(vals) / sizeof(vals[0])); ++i) info[i] = vals[i];
  return TSMPC_OK;
}

int tsmpc_describe_sparse(const tsmpc_problem* pb, int32_t max_ctas, int64_t smem_limit, int64_t* info,
                          int32_t n) {
  if (!pb || !info || !pb->anc || !pb->child_start || !pb->child_stop || !pb->stage_starts || !pb->prob ||
      !pb->B || !pb->Ls || !pb->lam_s)
    return fail(TSMPC_ERR_ARGUMENT, "null argument");
  SparseTreeIn ti{pb->N, pb->n_nodes, pb->stage_starts, pb->anc, pb->child_start, pb->child_stop, pb->prob};
  SparseOpsIn oi{pb->n_x, pb->n_u, pb->n_v, pb->B, pb->Ls, pb->lam_s};
  SparseHostPlan hp = choose_sparse_plan(ti, oi, r4(pb->n_x), r4(pb->n_u), r4(pb->n_v), std::max(1, (int)max_ctas),
                                         (size_t)smem_limit, (size_t)smem_limit, false, 0, 1);
  if (!hp.ok) return fail(TSMPC_ERR_VALIDATION, "%s", hp.why.c_str());
  const int64_t vals[] = {hp.n_ctas, hp.n_tiles, hp.n_chains, hp.n_trunk, hp.resident_ctas, hp.max_rows,
                          hp.max_needs, (int64_t)hp.smem, hp.S.split_n, hp.S.wide, hp.S.tile_cap};
  for (int i = 0; i < n && i < (int)(sizeof(vals) / sizeof(vals[0])); ++i) info[i] = vals[i];
  return TSMPC_OK;
}

int tsmpc_describe_shard(const tsmpc_problem* pb, int32_t max_ctas, int64_t smem_limit, int32_t rank,
                         int32_t world, int64_t* info, int32_t n, int64_t* edges, int64_t cap) {
  if (!pb || !info || !pb->anc || !pb->child_start || !pb->child_stop || !pb->stage_starts || !pb->prob ||
      !pb->B || !pb->Ls || !pb->lam_s)
    return fail(TSMPC_ERR_ARGUMENT, "null argument");
  SparseTreeIn ti{pb->N, pb->n_nodes, pb->stage_starts, pb->anc, pb->child_start, pb->child_stop, pb->prob};
  SparseOpsIn oi{pb->n_x, pb->n_u, pb->n_v, pb->B, pb->Ls, pb->lam_s};
  SparseHostPlan hp = choose_sparse_plan(ti, oi, r4(pb->n_x), r4(pb->n_u), r4(pb->n_v), std::max(1, (int)max_ctas),
                                         (size_t)smem_limit, (size_t)smem_limit, true, rank, world);
  if (!hp.ok) return fail(TSMPC_ERR_VALIDATION, "%s", hp.why.c_str());
  int64_t owned_heads = 0;
  for (unsigned char t : hp.towned) owned_heads += t;
  int64_t own_trunk = 0, mixed = 0, cut = 0;
  for (signed char r : hp.trole) {
    own_trunk += r == kRoleOwn || r == kRoleCutOwn;
    mixed += r == kRoleMixed;
    cut += r == kRoleCutOwn || r == kRoleCutForeign;
  }
  const int64_t xld = hp.cut ? r4(pb->n_x) * 2 + r4(pb->n_v) + r4(pb->n_u) : r4(pb->n_x) + r4(pb->n_v);
  const int64_t vals[] = {hp.n_ctas, hp.n_chains, hp.owned_rows, hp.n_trunk, hp.total_chains, owned_heads,
                          (int64_t)hp.smem, own_trunk, mixed, cut, hp.n_xch,
                          hp.n_xch * xld,
                          (int64_t)hp.result_edges.size()};
  for (int i = 0; i < n && i < (int)(sizeof(vals) / sizeof(vals[0])); ++i) info[i] = vals[i];
  if (edges)
    for (int64_t i = 0; i < cap && i < (int64_t)hp.result_edges.size(); ++i) edges[i] = hp.result_edges[i];
  return TSMPC_OK;
}

int tsmpc_plan_info(const tsmpc_plan* pl, int64_t* info, int32_t n) {
  if (!pl || !info) return fail(TSMPC_ERR_ARGUMENT, "null argument");
  const bool sp = pl->use_sparse;
  const int64_t vals[] = {pl->n_levels, sp ? pl->sp_ctas : pl->n_ctas, sp ? pl->sp_tiles : pl->n_tiles,
                          pl->n_segs, (int64_t)(sp ? pl->sp_smem : pl->smem), pl->base.diagA,
                          sp ? kThreadsS : kThreads, sp ? pl->sbase.tile_cap : kTileM, pl->sm_count, pl->base.collapsed,
                          sp ? pl->sp_trunk : pl->n_trunk, sp ? 1 : 0, pl->sp_resident,
                          pl->sharded ? 1 : 0, pl->rank, pl->world, (int64_t)pl->owned_edges.size(),
                          pl->total_chains, sp ? pl->sbase.split_n : 0, sp ? pl->sbase.wide : 0,
                          pl->sharded ? (int64_t)pl->sbase.n_xch * pl->sbase.XCH_LD : 0,
                          sp && pl->sbase.FG ? 1 : 0, pl->peer_on ? 1 : 0};
  for (int i = 0; i < n && i < (int)(sizeof(vals) / sizeof(vals[0])); ++i) info[i] = vals[i];
  return TSMPC_OK;
}

int tsmpc_debug_timers(tsmpc_plan* pl, uint64_t* out, int32_t n) {
  if (!pl || !out) return fail(TSMPC_ERR_ARGUMENT, "null argument");
  std::vector<unsigned long long> t(16 + 8 * 256);
  CU(cudaMemcpy(t.data(), pl->TIMERS, t.size() * sizeof(t[0]), cudaMemcpyDeviceToHost));
  CU(cudaMemset(pl->TIMERS, 0, t.size() * sizeof(t[0])));
  for (int i = 0; i < n && i < (int)t.size(); ++i) out[i] = t[i];
  return TSMPC_OK;
}

int tsmpc_set_cache(tsmpc_plan* pl, const double* beta, const double* uhat, const double* evec,
                    const double* q, const double* prices, const double* jrhs, const double* gdd) {
  if (!pl || !beta || !uhat || !evec || !q) return fail(TSMPC_ERR_ARGUMENT, "null cache array");
  CU(cudaSetDevice(pl->device));
  const int E = pl->E;
  int rc = 0;
  rc |= pl->put_rows(pl->BETA, pl->NVP, beta, pl->nv, E);
  rc |= pl->put_rows(pl->UHAT, pl->NUP, uhat, pl->nu, E);
  rc |= pl->put_rows(pl->EVEC, pl->NXP, evec, pl->nx, E);
  if (rc) return rc;
  if (pl->use_sparse) {
    beta_rotate_kernel<<<std::max(1, std::min((pl->E * pl->nv + 255) / 256, pl->sm_count * 16)), 256, 0,
                         pl->stream>>>(pl->BETA, pl->MSC, pl->MS, pl->BETA_S, pl->E, pl->nv, pl->NVP);
    CU(cudaGetLastError());
  }
  CU(cudaMemcpyAsync(pl->Q, q, sizeof(double) * pl->nu, cudaMemcpyHostToDevice, pl->stream));
  if (prices)
    CU(cudaMemcpyAsync(pl->PRICES, prices, sizeof(double) * pl->N * pl->nu, cudaMemcpyHostToDevice, pl->stream));
  if (jrhs)
    CU(cudaMemcpyAsync(pl->JRHS, jrhs, sizeof(double) * (size_t)E * pl->ne, cudaMemcpyHostToDevice, pl->stream));
  if (gdd && pl->put_rows(pl->GDD, pl->NXP, gdd, pl->nx, E)) return TSMPC_ERR_CUDA;
  CU(cudaStreamSynchronize(pl->stream));
  pl->has_cache = true;
  return TSMPC_OK;
}

int tsmpc_set_cache_operators(tsmpc_plan* pl, int32_t n_d, const double* part_map, const double* Gd,
                              const double* Ed, const double* Rhat, const double* eps_edge, const double* pbar) {
  if (!pl || !part_map || !Gd || !Ed || !Rhat || !eps_edge || !pbar) return fail(TSMPC_ERR_ARGUMENT, "null argument");
  if (n_d < 1) return fail(TSMPC_ERR_DIMENSION, "n_d must be >= 1");
  CU(cudaSetDevice(pl->device));
  if (pl->has_cache_ops) {
    if (n_d != pl->nd_c) return fail(TSMPC_ERR_DIMENSION, "n_d changed (%d -> %d)", pl->nd_c, n_d);
  } else {
    int rc = 0;
    rc |= pl->alloc(&pl->PART_MAP, (size_t)pl->nu * n_d);
    rc |= pl->alloc(&pl->GD, (size_t)pl->nx * n_d);
    rc |= pl->alloc(&pl->ED, (size_t)pl->ne * n_d);
    rc |= pl->alloc(&pl->RHAT, (size_t)pl->nu * pl->nv);
    rc |= pl->alloc(&pl->EPS, (size_t)pl->E * n_d);
    rc |= pl->alloc(&pl->PBAR, (size_t)pl->E);
    rc |= pl->alloc(&pl->DHAT, (size_t)pl->N * n_d);
    rc |= pl->alloc(&pl->ABAR, (size_t)pl->N * pl->nv);
    if (rc) return rc;
  }
  pl->nd_c = n_d;
  auto up = [&](double* dst, const double* src, size_t n) {
    return cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyHostToDevice, pl->stream);
  };
  CU(up(pl->PART_MAP, part_map, (size_t)pl->nu * n_d));
  CU(up(pl->GD, Gd, (size_t)pl->nx * n_d));
  CU(up(pl->ED, Ed, (size_t)pl->ne * n_d));
  CU(up(pl->RHAT, Rhat, (size_t)pl->nu * pl->nv));
  CU(up(pl->EPS, eps_edge, (size_t)pl->E * n_d));
  CU(up(pl->PBAR, pbar, (size_t)pl->E));
  {
    // CSR of part_map (nu x nd), Ed (ne x nd), B (nx x nu), Gd (nx x nd), rows in order
    std::vector<double> Bh((size_t)pl->nx * pl->nu);
    CU(cudaMemcpyAsync(Bh.data(), pl->d_B_c, Bh.size() * sizeof(double), cudaMemcpyDeviceToHost, pl->stream));
    CU(cudaStreamSynchronize(pl->stream));
    std::vector<int> ci;
    std::vector<double> cv;
    auto csr = [&](const double* M, int rows, int cols, int slot) {
      pl->csr_oi[2 * slot] = (int)ci.size();
      std::vector<int> ptr(rows + 1, 0), idx;
      for (int r = 0; r < rows; ++r) {
        for (int k = 0; k < cols; ++k)
          if (M[(size_t)r * cols + k] != 0.0) {
            idx.push_back(k);
            cv.push_back(M[(size_t)r * cols + k]);
          }
        ptr[r + 1] = (int)idx.size();
      }
      pl->csr_ov[slot] = (int)cv.size() - (int)idx.size();
      ci.insert(ci.end(), ptr.begin(), ptr.end());
      pl->csr_oi[2 * slot + 1] = (int)ci.size();
      ci.insert(ci.end(), idx.begin(), idx.end());
    };
    csr(part_map, pl->nu, n_d, 0);
    csr(Ed, pl->ne, n_d, 1);
    csr(Bh.data(), pl->nx, pl->nu, 2);
    csr(Gd, pl->nx, n_d, 3);
    // (a new upload each call: an earlier pattern may have been smaller)
    int rc = pl->upload(&pl->CSR_I, ci.data(), ci.size());
    rc |= pl->upload(&pl->CSR_V, cv.data(), std::max<size_t>(1, cv.size()));
    if (rc) return rc;
  }
  CU(cudaStreamSynchronize(pl->stream));
  pl->has_cache_ops = true;
  return TSMPC_OK;
}

int tsmpc_set_forecast(tsmpc_plan* pl, const double* dhat, const double* q, const double* prices,
                       const double* abar) {
  if (!pl || !dhat || !q || !prices || !abar) return fail(TSMPC_ERR_ARGUMENT, "null argument");
  if (!pl->has_cache_ops) return fail(TSMPC_ERR_VALIDATION, "no cache operators (tsmpc_set_cache_operators)");
  CU(cudaSetDevice(pl->device));
  const int N = pl->N, nd = pl->nd_c;
  CU(cudaMemcpyAsync(pl->DHAT, dhat, sizeof(double) * N * nd, cudaMemcpyHostToDevice, pl->stream));
  CU(cudaMemcpyAsync(pl->ABAR, abar, sizeof(double) * N * pl->nv, cudaMemcpyHostToDevice, pl->stream));
  CU(cudaMemcpyAsync(pl->Q, q, sizeof(double) * pl->nu, cudaMemcpyHostToDevice, pl->stream));
  CU(cudaMemcpyAsync(pl->PRICES, prices, sizeof(double) * N * pl->nu, cudaMemcpyHostToDevice, pl->stream));
  CacheArgs a{};
  a.E = pl->E; a.nx = pl->nx; a.nu = pl->nu; a.nv = pl->nv; a.nd = nd; a.ne = pl->ne;
  a.NXP = pl->NXP; a.NUP = pl->NUP; a.NVP = pl->NVP;
  a.edge_stage = pl->d_est_c; a.anc = pl->d_anc_c; a.child_start = pl->d_cs_c; a.child_stop = pl->d_ce_c;
  a.prob_edge = pl->d_pe_c; a.pbar = pl->PBAR; a.eps = pl->EPS;
  a.part_map = pl->PART_MAP; a.B = pl->d_B_c; a.Gd = pl->GD; a.Ed = pl->ED; a.Rhat = pl->RHAT;
  a.dhat = pl->DHAT; a.abar = pl->ABAR; a.q = pl->Q;
  a.uhat = pl->UHAT; a.evec = pl->EVEC; a.beta = pl->BETA; a.jrhs = pl->JRHS; a.gdd = pl->GDD;
  const int grid = std::max(1, std::min(pl->E, pl->sm_count * 8));
  if (pl->CSR_I && !std::getenv("TSMPC_DENSE_CACHE")) {
    const int* I = pl->CSR_I;
    const double* V = pl->CSR_V;
    a.pm_ptr = I + pl->csr_oi[0]; a.pm_idx = I + pl->csr_oi[1]; a.pm_val = V + pl->csr_ov[0];
    a.ed_ptr = I + pl->csr_oi[2]; a.ed_idx = I + pl->csr_oi[3]; a.ed_val = V + pl->csr_ov[1];
    a.b_ptr = I + pl->csr_oi[4]; a.b_idx = I + pl->csr_oi[5]; a.b_val = V + pl->csr_ov[2];
    a.gd_ptr = I + pl->csr_oi[6]; a.gd_idx = I + pl->csr_oi[7]; a.gd_val = V + pl->csr_ov[3];
    const int grid_s = std::max(1, std::min(pl->E, pl->sm_count * 16));
    cache_rows_sparse_kernel<<<grid_s, 128, sizeof(double) * (nd + pl->nu), pl->stream>>>(a);
  } else {
    cache_rows_kernel<<<grid, 128, sizeof(double) * (nd + pl->nu), pl->stream>>>(a);
  }
  CU(cudaGetLastError());
  cache_beta_kernel<<<std::max(1, std::min((pl->E + kCB - 1) / kCB, pl->sm_count * 8)), 128,
                      sizeof(double) * kCB * pl->nu, pl->stream>>>(a);
  CU(cudaGetLastError());
  if (pl->use_sparse) {
    beta_rotate_kernel<<<std::max(1, std::min((pl->E * pl->nv + 255) / 256, pl->sm_count * 16)), 256, 0,
                         pl->stream>>>(pl->BETA, pl->MSC, pl->MS, pl->BETA_S, pl->E, pl->nv, pl->NVP);
    CU(cudaGetLastError());
  }
  // no host wait: the solve that reads the cache is queued behind it on the same
  // stream (the pageable inputs are staged before cudaMemcpyAsync returns)
  pl->has_cache = true;
  return TSMPC_OK;
}

int tsmpc_get_cache(tsmpc_plan* pl, double* beta, double* uhat, double* evec) {
  if (!pl) return fail(TSMPC_ERR_ARGUMENT, "null argument");
  if (!pl->has_cache) return fail(TSMPC_ERR_VALIDATION, "no stage cache on the device");
  CU(cudaSetDevice(pl->device));
  if (pl->get_rows(beta, pl->nv, pl->BETA, pl->NVP, pl->E) || pl->get_rows(uhat, pl->nu, pl->UHAT, pl->NUP, pl->E) ||
      pl->get_rows(evec, pl->nx, pl->EVEC, pl->NXP, pl->E))
    return TSMPC_ERR_CUDA;
  CU(cudaStreamSynchronize(pl->stream));
  return TSMPC_OK;
}

static int set_root(tsmpc_plan* pl, const double* p) {
  std::vector<double> pp(pl->NXP, 0.0);
  if (p) std::copy(p, p + pl->nx, pp.begin());
  CU(cudaMemcpyAsync(pl->P, pp.data(), sizeof(double) * pl->NXP, cudaMemcpyHostToDevice, pl->stream));
  CU(cudaMemcpyAsync(pl->X, pl->P, sizeof(double) * pl->NXP, cudaMemcpyDeviceToDevice, pl->stream));
  CU(cudaStreamSynchronize(pl->stream));  // pp is a stack buffer
  return TSMPC_OK;
}

// One solve step (mode STEP) on the dual stored in `w` (three blocks).
static int run_step(tsmpc_plan* pl, double* w, int scaled, const double* beta, const double* uhat,
                    const double* evec) {
  Params P = pl->base;
  P.mode = kModeStep;
  P.iters = 1;
  P.scaled = scaled && pl->base.scaled;
  P.slot0 = 0;
  P.ybuf[0] = P.ybuf[1] = w;
  P.beta = beta;
  P.uhat = uhat;
  P.evec = evec;
  P.record_all = 0;
  P.lam = 1.0;
  P.theta = P.coef = nullptr;
  P.resid = nullptr;
  return launch_apg(pl, P);
}

// duality gap (engine.py:458-480) from the 10 reduced terms of compute_gap_terms
static double gap_from_terms(const tsmpc_plan* pl, const double* k) {
  const double primal = k[0] + (pl->ctx.Wx * k[1] + pl->ctx.gamma_d * k[2]);
  const double pairing = (k[3] + k[4]) + k[5];
  const double conj = (k[7] + k[8]) + k[9];
  return primal - ((pairing + k[6]) - conj);
}

// the gap's kernels for the dual `yfinal` (scaled) and the ergodic averages in
// XAVG / UAVG; the 10 reduced terms go to `terms` (device, no host sync)
static int compute_gap_terms(tsmpc_plan* pl, const double* yfinal, double* terms) {
  EdgeCtx c = pl->ctx;
  const int E = pl->E, G = grid_for(E);
  CU(cudaMemsetAsync(pl->COLS, 0, sizeof(double) * (size_t)E * 10, pl->stream));
  gap_dual_project_kernel<<<G, 256, 0, pl->stream>>>(c, yfinal, pl->WB, pl->COLS);
  CU(cudaGetLastError());
  pl->launches += 6 + pl->N;  // project, terms, projection, ub, N stages, primal terms, reduce (+ step)
  if (run_step(pl, pl->WB, 0, pl->BETA, pl->UHAT, pl->EVEC)) return TSMPC_ERR_CUDA;
  gap_dual_terms_kernel<<<G, 256, 0, pl->stream>>>(c, pl->WB, pl->X, pl->U, pl->COLS);
  CU(cudaGetLastError());
  if (pl->ne == 1) {
    gap_project_bisect_kernel<<<G, 256, 0, pl->stream>>>(c, pl->UAVG, pl->UF);
    CU(cudaGetLastError());
  } else {
    CU(cudaMemsetAsync(pl->DYK, 0, sizeof(unsigned long long) * 256, pl->stream));
    const size_t dsm = sizeof(double) * ((size_t)c.er_nnz + c.pc_nnz + 1 + 8 * 448) +
                       sizeof(int) * ((size_t)pl->ne + 1 + c.er_nnz + pl->nu + 1 + c.pc_nnz);
    // lockstep cooperative Dykstra when its grid is co-resident: a thread per (edge,
    // junction row) when the rows have disjoint flows, else a warp per edge; else
    // the two-pass form
    int occ = 0, occ_c = 0;
    const bool comp_coresident =
        pl->dyk_ncomp > 0 &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_c, gap_dykstra_comp_kernel, 256, 0) == cudaSuccess &&
        (long long)E * pl->dyk_ncomp <= (long long)occ_c * pl->sm_count * 256;
    if (!pl->dyk_warp && pl->dyk_ncomp > 0 && !pl->dyk_two_pass &&
        (!comp_coresident || std::getenv("TSMPC_DYKSTRA_COMP2")) && !std::getenv("TSMPC_DYKSTRA_LOCKSTEP")) {
      // a thread per (edge, junction row) in two passes, when the lockstep grid of
      // one thread per component cannot be co-resident (SMPC8: 178k components)
      const long long items = (long long)E * pl->dyk_ncomp;
      const int gblk = (int)std::max(1LL, std::min((items + 255) / 256, (long long)pl->sm_count * 16));
      gap_dykstra_comp_pass1_kernel<<<gblk, 256, 0, pl->stream>>>(c, pl->DYKC, pl->dyk_ncomp, pl->DYKF,
                                                                  pl->dyk_nfree, pl->UAVG, pl->DYK, pl->UF);
      CU(cudaGetLastError());
      gap_dykstra_comp_pass2_kernel<<<gblk, 256, 0, pl->stream>>>(c, pl->DYKC, pl->dyk_ncomp, pl->UAVG, pl->DYK,
                                                                  pl->UF);
      CU(cudaGetLastError());
      pl->launches += 1;
    } else if (!pl->dyk_two_pass && !pl->dyk_warp && comp_coresident) {
      const int gblk = std::max(1, (int)(((long long)E * pl->dyk_ncomp + 255) / 256));
      const DykComp* comps = pl->DYKC;
      int ncomp = pl->dyk_ncomp, nfree = pl->dyk_nfree;
      const int* freeu = pl->DYKF;
      double* u0 = pl->UAVG;
      unsigned long long* slots = pl->DYK;
      double* uf = pl->UF;
      void* args[] = {&c, &comps, &ncomp, &freeu, &nfree, &u0, &slots, &uf};
      CU(cudaLaunchCooperativeKernel((void*)gap_dykstra_comp_kernel, dim3(gblk), dim3(256), args, 0, pl->stream));
    } else if (!pl->dyk_two_pass &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gap_dykstra_coop_kernel, 256, dsm) == cudaSuccess &&
        occ > 0) {
      if (!pl->DYKST && pl->alloc(&pl->DYKST, 4 * (size_t)E * pl->NUP)) return TSMPC_ERR_CUDA;
      const int gblk = std::max(1, std::min((E + 7) / 8, occ * pl->sm_count));
      double* u0 = pl->UAVG;
      unsigned long long* slots = pl->DYK;
      double* st = pl->DYKST;
      double* uf = pl->UF;
      void* args[] = {&c, &u0, &slots, &st, &uf};
      CU(cudaLaunchCooperativeKernel((void*)gap_dykstra_coop_kernel, dim3(gblk), dim3(256), args, dsm, pl->stream));
      if (std::getenv("TSMPC_DEBUG_DYKSTRA")) {
        std::vector<unsigned long long> sl(200);
        CU(cudaMemcpyAsync(sl.data(), pl->DYK, sizeof(unsigned long long) * 200, cudaMemcpyDeviceToHost, pl->stream));
        CU(cudaStreamSynchronize(pl->stream));
        int K = -1;
        for (int it = 0; it < 200 && K < 0; ++it) {
          double g;
          std::memcpy(&g, &sl[it], sizeof g);
          if (g < 1e-13) K = it;
        }
        std::fprintf(stderr, "[tsmpc] dykstra: grid %d x 256 (occupancy %d/SM), stopping sweep K = %d\n", gblk, occ, K);
      }
    } else {
      const int gblk = std::max(1, std::min((E + 7) / 8, pl->sm_count * 8));
      gap_dykstra_pass_kernel<<<gblk, 256, dsm, pl->stream>>>(c, pl->UAVG, pl->DYK, 1, pl->UF);
      CU(cudaGetLastError());
      gap_dykstra_pass_kernel<<<gblk, 256, dsm, pl->stream>>>(c, pl->UAVG, pl->DYK, 2, pl->UF);
      CU(cudaGetLastError());
      pl->launches += 1;
    }
  }
  gap_ub_kernel<<<G, 256, 0, pl->stream>>>(c, pl->UF, pl->UB);
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(pl->XF, pl->P, sizeof(double) * pl->NXP, cudaMemcpyDeviceToDevice, pl->stream));
  if (c.a_diag && pl->N <= kPropMaxDepth) {  // every stage in one launch (root paths)
    const int total = (pl->n_nodes - 1) * pl->nx;
    gap_propagate_paths_kernel<<<std::max(1, std::min((total + 255) / 256, 4096)), 256, 0, pl->stream>>>(
        c, pl->n_nodes, pl->XF, pl->UB);
    pl->launches -= pl->N - 1;
  } else {
    for (int j = 0; j < pl->N; ++j) {
      const int n0 = (int)pl->stage_starts[j + 1], n1 = (int)pl->stage_starts[j + 2];
      const int total = (n1 - n0) * pl->nx;
      gap_propagate_stage_kernel<<<std::max(1, std::min((total + 255) / 256, 4096)), 256, 0, pl->stream>>>(
          c, n0, n1, pl->XF, pl->UB);
    }
  }
  CU(cudaGetLastError());
  gap_primal_terms_kernel<<<G, 256, 0, pl->stream>>>(c, pl->UF, pl->XF, pl->COLS);
  CU(cudaGetLastError());
  reduce_cols_kernel<<<1, 1024, 0, pl->stream>>>(pl->COLS, E, 10, terms);
  CU(cudaGetLastError());
  return TSMPC_OK;
}

static int compute_gap(tsmpc_plan* pl, const double* yfinal, double* gap) {
  int rc = compute_gap_terms(pl, yfinal, pl->RED);
  if (rc) return rc;
  double k[10];
  CU(cudaMemcpyAsync(k, pl->RED, sizeof(k), cudaMemcpyDeviceToHost, pl->stream));
  CU(cudaStreamSynchronize(pl->stream));
  *gap = gap_from_terms(pl, k);
  return TSMPC_OK;
}

namespace {

// One solve split in three so that tsmpc_solve_group can interleave several
// shard plans: prepare (tables, dual start, root), the launches, finish (stopping
// bookkeeping, gap, read-back).
struct SolveState {
  int iters = 0, nres = 1;
  bool record = false, stopping = false;
  Params P{};
};

int solve_prepare(tsmpc_plan* pl, const double* p, int32_t iters, double lam, const double* warm_sig,
                  const double* warm_zeta, const double* warm_psi, const double* theta, const double* coef,
                  int32_t flags, SolveState& st) {
  if (!pl || !p) return fail(TSMPC_ERR_ARGUMENT, "null argument");
  if (iters < 1) return fail(TSMPC_ERR_VALIDATION, "max_iters must be >= 1");
  if (!(lam > 0.0)) return fail(TSMPC_ERR_VALIDATION, "step size must be positive");
  if (!pl->has_cache) return fail(TSMPC_ERR_VALIDATION, "no stage cache uploaded (tsmpc_set_cache)");
  CU(cudaSetDevice(pl->device));
  pl->launches = 0;
  const int E = pl->E, NXP = pl->NXP, NUP = pl->NUP, nx = pl->nx, nu = pl->nu;
  const bool record = flags & (TSMPC_RECORD_RESIDUALS | TSMPC_GAP_TRACE);
  if ((flags & TSMPC_GAP_TRACE) && (!pl->use_sparse || pl->sharded))
    return fail(TSMPC_ERR_VALIDATION, "the per-iteration duality gap needs a single-GPU structured-basis plan");
  if ((flags & TSMPC_GAP_TRACE) && pl->tol > 0.0)
    return fail(TSMPC_ERR_VALIDATION, "the per-iteration duality gap runs the fixed iteration count (no tol)");
  if ((flags & TSMPC_GAP_TRACE) && (flags & TSMPC_SKIP_GAP))
    return fail(TSMPC_ERR_VALIDATION, "TSMPC_GAP_TRACE and TSMPC_SKIP_GAP exclude each other");
  CU(cudaMemsetAsync(pl->ABORT, 0, sizeof(unsigned int), pl->stream));
  // momentum tables
  if (pl->theta_cap < iters) {
    int rc = pl->alloc(&pl->THETA, iters) | pl->alloc(&pl->COEF, iters);
    if (rc) return rc;
    pl->theta_cap = iters;
  }
  std::vector<double> th(iters), cf(iters);
  if (theta && coef) {
    std::copy(theta, theta + iters, th.begin());
    std::copy(coef, coef + iters, cf.begin());
  } else {
    double t = 1.0, tp = 1.0;
    for (int k = 0; k < iters; ++k) {
      th[k] = t;
      cf[k] = t * (1.0 / tp - 1.0);
      tp = t;
      t = 0.5 * (std::sqrt(std::pow(t, 4.0) + 4.0 * (t * t)) - t * t);
    }
  }
  CU(cudaMemcpyAsync(pl->THETA, th.data(), sizeof(double) * iters, cudaMemcpyHostToDevice, pl->stream));
  CU(cudaMemcpyAsync(pl->COEF, cf.data(), sizeof(double) * iters, cudaMemcpyHostToDevice, pl->stream));
  const int nres = record ? iters : 1;
  if (pl->resid_cap < nres) {
    if (pl->alloc(&pl->RESID, nres)) return TSMPC_ERR_CUDA;
    pl->resid_cap = nres;
  }
  CU(cudaMemsetAsync(pl->RESID, 0, sizeof(unsigned long long) * nres, pl->stream));
  // dual start
  const size_t yblk = 2 * (size_t)E * NXP + (size_t)E * NUP;
  if ((flags & TSMPC_WARM_DEVICE) && pl->last_y) {
    // warm start from the previous solve's final dual, still resident in HBM
    if (pl->last_y != pl->Y0)
      CU(cudaMemcpyAsync(pl->Y0, pl->last_y, sizeof(double) * yblk, cudaMemcpyDeviceToDevice, pl->stream));
    CU(cudaMemcpyAsync(pl->Y1, pl->Y0, sizeof(double) * yblk, cudaMemcpyDeviceToDevice, pl->stream));
  } else if (warm_sig && warm_zeta && warm_psi) {
    if (pl->put_rows(pl->Y0, NXP, warm_sig, nx, E) || pl->put_rows(pl->Y0 + (size_t)E * NXP, NXP, warm_zeta, nx, E) ||
        pl->put_rows(pl->Y0 + 2 * (size_t)E * NXP, NUP, warm_psi, nu, E))
      return TSMPC_ERR_CUDA;
    CU(cudaMemcpyAsync(pl->Y1, pl->Y0, sizeof(double) * yblk, cudaMemcpyDeviceToDevice, pl->stream));
  } else {
    CU(cudaMemsetAsync(pl->Y0, 0, sizeof(double) * yblk, pl->stream));
    CU(cudaMemsetAsync(pl->Y1, 0, sizeof(double) * yblk, pl->stream));
  }
  CU(cudaMemsetAsync(pl->XAVG, 0, sizeof(double) * (size_t)pl->n_nodes * NXP, pl->stream));
  CU(cudaMemsetAsync(pl->UAVG, 0, sizeof(double) * (size_t)E * NUP, pl->stream));
  if (set_root(pl, p)) return TSMPC_ERR_CUDA;

  const bool stopping = pl->tol > 0.0 && pl->use_sparse && !pl->sharded;
  if (stopping) {
    const int nchk = iters / std::max(1, pl->check_every) + 1;
    if (pl->rchk_cap < nchk) {
      if (pl->alloc(&pl->RCHK, nchk)) return TSMPC_ERR_CUDA;
      pl->rchk_cap = nchk;
    }
    if (!pl->ITERS && pl->alloc(&pl->ITERS, 1)) return TSMPC_ERR_CUDA;
    CU(cudaMemsetAsync(pl->RCHK, 0, sizeof(unsigned long long) * nchk, pl->stream));
  }
  Params P = pl->base;
  P.mode = kModeApg;
  P.iters = iters;
  P.tol = stopping ? pl->tol : 0.0;
  P.check_every = std::max(1, pl->check_every);
  P.resid_chk = pl->RCHK;
  P.iters_done = pl->ITERS;
  P.slot0 = 0;
  P.ybuf[0] = pl->Y0;
  P.ybuf[1] = pl->Y1;
  P.beta = pl->BETA;
  P.uhat = pl->UHAT;
  P.evec = pl->EVEC;
  P.lam = lam;
  P.inv_lam = 1.0 / lam;
  P.theta = pl->THETA;
  P.coef = pl->COEF;
  P.record_all = record ? 1 : 0;
  P.resid = pl->RESID;
  st.iters = iters;
  st.nres = nres;
  st.record = record;
  st.stopping = stopping;
  st.P = P;
  return TSMPC_OK;
}

// Shard plans hold the rows of their own chains, of the trunk positions with
// only their chains below, and of the mixed (replicated) trunk positions; the other
// rows hold zeros or a warm start.  Before the duality gap every rank assembles the
// full ergodic averages and final dual by a sum over ranks, after zeroing the rows
// it does not count (another rank's; mixed rows and the root's x_avg on ranks != 0):
// exact, each entry has one non-zero contributor.
__global__ void zero_rows_kernel(const int* rows, int n, bool root, int E, int NXP, int NUP, double* xavg,
                                 double* uavg, double* y) {
  const int b = blockIdx.x;
  if (b == n) {
    if (root)
      for (int i = threadIdx.x; i < NXP; i += blockDim.x) xavg[i] = 0.0;
    return;
  }
  const size_t e = (size_t)rows[b];
  for (int i = threadIdx.x; i < NXP; i += blockDim.x) {
    xavg[(e + 1) * NXP + i] = 0.0;
    y[e * NXP + i] = 0.0;
    y[(size_t)E * NXP + e * NXP + i] = 0.0;
  }
  for (int j = threadIdx.x; j < NUP; j += blockDim.x) {
    uavg[e * NUP + j] = 0.0;
    y[2 * (size_t)E * NXP + e * NUP + j] = 0.0;
  }
}

int zero_replicated_rows(tsmpc_plan* pl, double* yfin, cudaStream_t s) {
  const int n = (int)pl->zero_edges.size();
  zero_rows_kernel<<<n + 1, 128, 0, s>>>(pl->d_zero, n, pl->rank != 0, pl->E, pl->NXP, pl->NUP, pl->XAVG, pl->UAVG,
                                         yfin);
  CU(cudaGetLastError());
  return TSMPC_OK;
}

int assemble_shard_state(tsmpc_plan* pl, double* yfin) {
  if (zero_replicated_rows(pl, yfin, pl->stream)) return TSMPC_ERR_CUDA;
  const size_t yblk = 2 * (size_t)pl->E * pl->NXP + (size_t)pl->E * pl->NUP;
  struct { double* p; size_t n; } bufs[] = {{pl->XAVG, (size_t)pl->n_nodes * pl->NXP},
                                            {pl->UAVG, (size_t)pl->E * pl->NUP}, {yfin, yblk}};
  for (auto& b : bufs) {
    const int nr = pl->nccl->AllReduce(b.p, b.p, b.n, NcclApi::kFloat64, NcclApi::kSum, pl->comm, pl->stream);
    if (nr != 0) return fail(TSMPC_ERR_NCCL, "ncclAllReduce: %s", pl->nccl->GetErrorString(nr));
  }
  return TSMPC_OK;
}

SParams sparse_params(const tsmpc_plan* pl, const Params& P) {
  SParams S = pl->sbase;
  S.P = P;
  S.P.KY = pl->KY_S;
  S.P.n_trunk = pl->sp_trunk;
  return S;
}

int solve_finish(tsmpc_plan* pl, const SolveState& st, int32_t flags, tsmpc_result* out,
                 bool assembled = false) {
  CU(cudaSetDevice(pl->device));
  const int E = pl->E, NXP = pl->NXP, NUP = pl->NUP, nx = pl->nx, nu = pl->nu;
  const int iters = st.iters, nres = st.nres;
  const bool record = st.record, stopping = st.stopping;
  int done = iters;
  unsigned int aborted = 0;
  CU(cudaMemcpyAsync(&aborted, pl->ABORT, sizeof(aborted), cudaMemcpyDeviceToHost, pl->stream));
  unsigned long long stop_bits = 0;  // residual of the check that stopped the solve
  if (stopping) {
    CU(cudaMemcpyAsync(&done, pl->ITERS, sizeof(int), cudaMemcpyDeviceToHost, pl->stream));
    CU(cudaStreamSynchronize(pl->stream));
    if (done < 1 || done > iters) done = iters;
    if (done < iters) {
      CU(cudaMemcpyAsync(&stop_bits, pl->RCHK + done / pl->check_every - 1, sizeof(stop_bits),
                         cudaMemcpyDeviceToHost, pl->stream));
    }
  }
  CU(cudaStreamSynchronize(pl->stream));
  if (aborted)
    return fail(TSMPC_ERR_CUDA, "sparse kernel: a chain/trunk signal wait timed out (launch results discarded)");
  double* yfin = ((done & 1) == 0) ? pl->Y0 : pl->Y1;
  pl->last_y = yfin;
  const bool want_gap = !(flags & TSMPC_SKIP_GAP) && (!pl->sharded || pl->comm || assembled);
  if (want_gap && pl->sharded && pl->comm && !assembled) {
    int rc = assemble_shard_state(pl, yfin);
    if (rc) return rc;
  }
  // keep the last iterate before the gap's solve step reuses X / U
  CU(cudaMemcpyAsync(pl->XL, pl->X, sizeof(double) * (size_t)pl->n_nodes * NXP, cudaMemcpyDeviceToDevice, pl->stream));
  CU(cudaMemcpyAsync(pl->UL, pl->U, sizeof(double) * (size_t)E * NUP, cudaMemcpyDeviceToDevice, pl->stream));
  // the results are final here (the gap only reads them): read them back on the
  // copy stream while the gap runs
  CU(cudaEventRecord(pl->ev_out, pl->stream));
  CU(cudaStreamWaitEvent(pl->stream2, pl->ev_out, 0));
  cudaStream_t cs = pl->stream2;
  std::vector<unsigned long long> rbits(nres);
  CU(cudaMemcpyAsync(rbits.data(), pl->RESID, sizeof(unsigned long long) * nres, cudaMemcpyDeviceToHost, cs));
  if (pl->get_rows(out->u0, nu, pl->UAVG, NUP, 1, cs)) return TSMPC_ERR_CUDA;
  if (!(flags & TSMPC_KEEP_DEVICE)) {
    int rc = 0;
    rc |= pl->get_rows(out->x, nx, pl->XL, NXP, pl->n_nodes, cs);
    rc |= pl->get_rows(out->u, nu, pl->UL, NUP, E, cs);
    rc |= pl->get_rows(out->x_avg, nx, pl->XAVG, NXP, pl->n_nodes, cs);
    rc |= pl->get_rows(out->u_avg, nu, pl->UAVG, NUP, E, cs);
    rc |= pl->get_rows(out->dual_sig, nx, yfin, NXP, E, cs);
    rc |= pl->get_rows(out->dual_zeta, nx, yfin + (size_t)E * NXP, NXP, E, cs);
    rc |= pl->get_rows(out->dual_psi, nu, yfin + 2 * (size_t)E * NXP, NUP, E, cs);
    if (rc) return rc;
  }
  double gap = NAN;
  if (want_gap) {
    int rc = compute_gap(pl, yfin, &gap);
    if (rc) {
      cudaStreamSynchronize(cs);
      return rc;
    }
  }
  CU(cudaEventRecord(pl->ev2, pl->stream));
  out->gap = gap;
  out->iterations = done;
  if ((flags & TSMPC_GAP_TRACE) && out->gap_trace) {
    std::vector<double> terms((size_t)std::max(0, iters - 1) * 10);
    if (!terms.empty())
      CU(cudaMemcpyAsync(terms.data(), pl->GTR, sizeof(double) * terms.size(), cudaMemcpyDeviceToHost, pl->stream));
    CU(cudaStreamSynchronize(pl->stream));
    for (int k = 0; k + 1 < iters; ++k) out->gap_trace[k] = gap_from_terms(pl, terms.data() + (size_t)k * 10);
    out->gap_trace[iters - 1] = gap;
  }
  CU(cudaStreamSynchronize(cs));
  CU(cudaStreamSynchronize(pl->stream));
  float ms = 0.f;
  CU(cudaEventElapsedTime(&ms, pl->ev0, pl->ev1));
  out->device_ms = ms;
  CU(cudaEventElapsedTime(&ms, pl->ev0, pl->ev2));
  out->device_total_ms = ms;
  out->kernel_launches = pl->launches;
  auto as_d = [](unsigned long long b) { double d; std::memcpy(&d, &b, sizeof d); return d; };
  // residual_inf: the last iteration run (record: its trace slot; a stopped solve
  // without a trace: the residual of the check that stopped it)
  out->residual_inf = record ? as_d(rbits[done - 1]) : (stop_bits ? as_d(stop_bits) : as_d(rbits[0]));
  if (record && out->resid_trace)
    for (int k = 0; k < iters; ++k) out->resid_trace[k] = k < done ? as_d(rbits[k]) : NAN;
  return TSMPC_OK;
}

}  // namespace

int tsmpc_solve(tsmpc_plan* pl, const double* p, int32_t iters, double lam, const double* warm_sig,
                const double* warm_zeta, const double* warm_psi, const double* theta, const double* coef,
                int32_t flags, tsmpc_result* out) {
  if (!pl || !p || !out) return fail(TSMPC_ERR_ARGUMENT, "null argument");
  if (pl->sharded && !pl->comm && pl->world > 1)
    return fail(TSMPC_ERR_VALIDATION, "shard plan without a communicator: run it through tsmpc_solve_group");
  if (pl->multi && pl->world > 1)
    return fail(TSMPC_ERR_VALIDATION, "plan of a multi-GPU set: run it through tsmpc_solve_multi");
  SolveState st;
  int rc = solve_prepare(pl, p, iters, lam, warm_sig, warm_zeta, warm_psi, theta, coef, flags, st);
  if (rc) return rc;
  const Params& P = st.P;
  CU(cudaEventRecord(pl->ev0, pl->stream));
  if (pl->use_sparse) {
    SParams S = sparse_params(pl, P);
    if (!pl->sharded && (flags & TSMPC_GAP_TRACE)) {
      // per-iteration duality gap (engine.py:577-582): one launch per iteration,
      // each leaving its state in HBM, then the gap's kernels on y_{nu+1} and the
      // ergodic averages; the 10 reduced terms of every iteration stay on the device
      // until the end (no host round trip per iteration)
      if (pl->gtr_cap < iters) {
        if (pl->alloc(&pl->GTR, (size_t)iters * 10)) return TSMPC_ERR_CUDA;
        pl->gtr_cap = iters;
      }
      for (int nu = 0; nu < iters; ++nu) {
        if (pl->SUBCTR) CU(cudaMemsetAsync(pl->SUBCTR, 0, 4 * sizeof(unsigned int), pl->stream));
        CU(sparse_launch(S, LaunchWin{nu, nu + 1, 3, 1}, pl->sp_ctas, pl->sp_smem, pl->stream));
        ++pl->launches;
        if (nu + 1 < iters) {  // the last one is the solve's own gap (solve_finish)
          if (compute_gap_terms(pl, ((nu + 1) & 1) ? pl->Y1 : pl->Y0, pl->GTR + (size_t)nu * 10))
            return TSMPC_ERR_CUDA;
        }
      }
    } else if (!pl->sharded) {
      if (pl->SUBCTR) CU(cudaMemsetAsync(pl->SUBCTR, 0, 4 * sizeof(unsigned int), pl->stream));
      CU(sparse_launch(S, LaunchWin{0, iters, 3, 0}, pl->sp_ctas, pl->sp_smem, pl->stream));
      ++pl->launches;
    } else {
      // per iteration: phase 1 (backward, head pre-reduction, the bottom-up sums below
      // the cut), the cross-GPU sum of the cut exchange rows XCH, phase 2 (trunk
      // sweep above the cut, needs, forward, epilogue).
      // With a communicator the 2 x iters launches and the all-reduces are captured
      // once per iteration count into a CUDA graph and replayed (the launch windows
      // are kernel arguments; the plan's parameters are uploaded before each replay)
      const size_t xn = (size_t)S.n_xch * S.XCH_LD;
      auto issue = [&]() -> int {
        for (int nu = 0; nu < iters; ++nu) {
          CU(sparse_launch(S, LaunchWin{nu, nu + 1, 1, 0}, pl->sp_ctas, pl->sp_smem, pl->stream));
          if (pl->sp_trunk > 0 && pl->comm && xn > 0) {
            const int nr = pl->nccl->AllReduce(pl->XCH, pl->XCH, xn, NcclApi::kFloat64, NcclApi::kSum, pl->comm,
                                               pl->stream);
            if (nr != 0) return fail(TSMPC_ERR_NCCL, "ncclAllReduce: %s", pl->nccl->GetErrorString(nr));
          }
          CU(sparse_launch(S, LaunchWin{nu, nu + 1, 2, 0}, pl->sp_ctas, pl->sp_smem, pl->stream));
        }
        return TSMPC_OK;
      };
      bool graphed = false;
      const bool fused = pl->peer_on && !std::getenv("TSMPC_NO_PEER");
      if (fused) {
        // both phases and the cut exchange over peer memory in one launch
        CU(sparse_launch(S, LaunchWin{0, iters, 7, 0, pl->xgen}, pl->sp_ctas, pl->sp_smem, pl->stream));
        pl->xgen += (unsigned long long)iters;
      } else if (pl->comm && !std::getenv("TSMPC_NO_GRAPH")) {
        if (pl->gexec && pl->g_iters == iters) {
          graphed = true;
        } else {
          if (pl->gexec) {
            cudaGraphExecDestroy(pl->gexec);
            pl->gexec = nullptr;
          }
          CU(sparse_params_upload(S, pl->stream));  // g_sp holds this plan's parameters
          cudaGraph_t g = nullptr;
          if (cudaStreamBeginCapture(pl->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
            const int irc = issue();
            const cudaError_t ce = cudaStreamEndCapture(pl->stream, &g);
            if (irc == TSMPC_OK && ce == cudaSuccess && g &&
                cudaGraphInstantiate(&pl->gexec, g, 0) == cudaSuccess) {
              pl->g_iters = iters;
              graphed = true;
            } else {
              pl->gexec = nullptr;
              pl->graph_why = irc != TSMPC_OK ? g_err : std::string(cudaGetErrorString(ce));
            }
            if (g) cudaGraphDestroy(g);
          }
          cudaGetLastError();  // a failed capture falls back to direct launches
        }
      }
      if (fused) {
        // (launched above)
      } else if (graphed) {
        CU(sparse_params_upload(S, pl->stream));
        CU(cudaGraphLaunch(pl->gexec, pl->stream));
        CU(sparse_note_launch(pl->stream));
      } else {
        const int irc = issue();
        if (irc) return irc;
      }
      pl->launches += fused ? 1 : 2 * (long long)iters;
      if (pl->comm) {
        // residual: max over ranks (non-negative doubles order like their bit patterns)
        const int nr = pl->nccl->AllReduce(pl->RESID, pl->RESID, (size_t)st.nres, NcclApi::kUint64, NcclApi::kMax,
                                           pl->comm, pl->stream);
        if (nr != 0) return fail(TSMPC_ERR_NCCL, "ncclAllReduce: %s", pl->nccl->GetErrorString(nr));
      }
    }
  } else if (launch_apg(pl, P)) {
    return TSMPC_ERR_CUDA;
  }
  CU(cudaEventRecord(pl->ev1, pl->stream));
  return solve_finish(pl, st, flags, out);
}

namespace {

constexpr int kMaxGroup = 8;
struct GroupBufs {
  double* hs[kMaxGroup];
  unsigned long long* res[kMaxGroup];
};

// The exchange NCCL performs between shard ranks, done in place on one device:
// every plan's head-sum buffer becomes the sum over the group.
__global__ void group_sum_kernel(GroupBufs g, int n, size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < n; ++r) s += g.hs[r][i];
    for (int r = 0; r < n; ++r) g.hs[r][i] = s;
  }
}

__global__ void group_max_kernel(GroupBufs g, int n, int count) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    unsigned long long m = 0;
    for (int r = 0; r < n; ++r) m = max(m, g.res[r][i]);
    for (int r = 0; r < n; ++r) g.res[r][i] = m;
  }
}

}  // namespace

int tsmpc_solve_group(tsmpc_plan* const* plans, int32_t n, const double* p, int32_t iters, double lam,
                      const double* theta, const double* coef, int32_t flags, tsmpc_result* outs) {
  if (!plans || !p || !outs) return fail(TSMPC_ERR_ARGUMENT, "null argument");
  if (n < 1 || n > kMaxGroup) return fail(TSMPC_ERR_ARGUMENT, "group size %d outside 1..%d", n, kMaxGroup);
  for (int r = 0; r < n; ++r) {
    const tsmpc_plan* pl = plans[r];
    if (!pl) return fail(TSMPC_ERR_ARGUMENT, "null plan in group");
    if (!pl->sharded || pl->comm || pl->world != n || pl->rank != r)
      return fail(TSMPC_ERR_VALIDATION, "group member %d must be the local shard plan of rank %d of %d", r, r, n);
    if (pl->device != plans[0]->device || pl->sp_trunk != plans[0]->sp_trunk ||
        pl->sbase.n_xch != plans[0]->sbase.n_xch || pl->E != plans[0]->E)
      return fail(TSMPC_ERR_VALIDATION, "group members must be shards of one tree on one device");
  }
  CU(cudaSetDevice(plans[0]->device));
  // all members run on the first member's stream, in the order NCCL ranks would
  std::vector<cudaStream_t> saved(n);
  for (int r = 0; r < n; ++r) saved[r] = plans[r]->stream;
  struct Restore {
    tsmpc_plan* const* pl;
    std::vector<cudaStream_t>& s;
    ~Restore() { for (size_t r = 0; r < s.size(); ++r) pl[r]->stream = s[r]; }
  } restore{plans, saved};
  cudaStream_t s0 = plans[0]->stream;
  for (int r = 0; r < n; ++r) plans[r]->stream = s0;
  std::vector<SolveState> st(n);
  std::vector<SParams> S(n);
  GroupBufs g{};
  for (int r = 0; r < n; ++r) {
    int rc = solve_prepare(plans[r], p, iters, lam, nullptr, nullptr, nullptr, theta, coef, flags, st[r]);
    if (rc) return rc;
    S[r] = sparse_params(plans[r], st[r].P);
    g.hs[r] = plans[r]->XCH;
    g.res[r] = plans[r]->RESID;
    CU(cudaEventRecord(plans[r]->ev0, s0));
  }
  const size_t hs = (size_t)S[0].n_xch * S[0].XCH_LD;
  for (int nu = 0; nu < iters; ++nu) {
    for (int r = 0; r < n; ++r) {
      CU(sparse_launch(S[r], LaunchWin{nu, nu + 1, 1, 0}, plans[r]->sp_ctas, plans[r]->sp_smem, s0));
    }
    if (plans[0]->sp_trunk > 0 && hs > 0) {
      group_sum_kernel<<<(unsigned)std::min<size_t>(256, (hs + 255) / 256), 256, 0, s0>>>(g, n, hs);
      CU(cudaGetLastError());
    }
    for (int r = 0; r < n; ++r) {
      CU(sparse_launch(S[r], LaunchWin{nu, nu + 1, 2, 0}, plans[r]->sp_ctas, plans[r]->sp_smem, s0));
      plans[r]->launches += 2;
    }
  }
  group_max_kernel<<<(st[0].nres + 255) / 256, 256, 0, s0>>>(g, n, st[0].nres);
  CU(cudaGetLastError());
  for (int r = 0; r < n; ++r) CU(cudaEventRecord(plans[r]->ev1, s0));
  const bool gap = !(flags & TSMPC_SKIP_GAP);
  if (gap) {
    // the exchange assemble_shard_state does across GPUs: every shard's averages and
    // final dual become the full arrays (replicated rows counted once)
    const size_t yblk = 2 * (size_t)plans[0]->E * plans[0]->NXP + (size_t)plans[0]->E * plans[0]->NUP;
    GroupBufs gx{}, gu{}, gy{};
    for (int r = 0; r < n; ++r) {
      double* yfin = (iters & 1) == 0 ? plans[r]->Y0 : plans[r]->Y1;
      if (zero_replicated_rows(plans[r], yfin, s0)) return TSMPC_ERR_CUDA;
      gx.hs[r] = plans[r]->XAVG;
      gu.hs[r] = plans[r]->UAVG;
      gy.hs[r] = yfin;
    }
    const size_t nx_ = (size_t)plans[0]->n_nodes * plans[0]->NXP, nu_ = (size_t)plans[0]->E * plans[0]->NUP;
    group_sum_kernel<<<(unsigned)std::min<size_t>(1024, (nx_ + 255) / 256), 256, 0, s0>>>(gx, n, nx_);
    group_sum_kernel<<<(unsigned)std::min<size_t>(1024, (nu_ + 255) / 256), 256, 0, s0>>>(gu, n, nu_);
    group_sum_kernel<<<(unsigned)std::min<size_t>(1024, (yblk + 255) / 256), 256, 0, s0>>>(gy, n, yblk);
    CU(cudaGetLastError());
  }
  for (int r = 0; r < n; ++r) {
    int rc = solve_finish(plans[r], st[r], flags, outs + r, gap);
    if (rc) return rc;
  }
  return TSMPC_OK;
}


int tsmpc_plan_trial(tsmpc_plan* pl, int32_t iters, double* ms) {
  if (!pl || !ms || iters < 1) return fail(TSMPC_ERR_ARGUMENT, "null argument or iters < 1");
  // a timing trial of the persistent kernel on whatever the plan's buffers hold
  // (zero after creation): the loop's cost does not depend on the data
  const bool had = pl->has_cache;
  const double tol = pl->tol;
  pl->has_cache = true;
  pl->tol = 0.0;
  std::vector<double> p(pl->nx, 0.0);
  SolveState st;
  int rc = solve_prepare(pl, p.data(), iters, 1.0, nullptr, nullptr, nullptr, nullptr, nullptr,
                         TSMPC_SKIP_GAP | TSMPC_KEEP_DEVICE, st);
  pl->has_cache = had;
  pl->tol = tol;
  if (rc) return rc;
  CU(cudaEventRecord(pl->ev0, pl->stream));
  if (pl->sharded && pl->sbase.FL > 0 && !std::getenv("TSMPC_NO_PEER")) {
    // this rank's share of a sharded solve in one launch (both phases per iteration,
    // as with the in-kernel exchange), without the exchange itself: the per-rank
    // compute time of a w-GPU job
    SParams S = sparse_params(pl, st.P);
    S.peer_rx = nullptr;
    S.peer_cnt = nullptr;
    CU(sparse_launch(S, LaunchWin{0, iters, 7, 0, 0}, pl->sp_ctas, pl->sp_smem, pl->stream));
  } else if (pl->sharded) {
    // this rank's share of a sharded solve: its two launches per iteration,
    // without the cross-rank exchange (the per-rank compute time of a w-GPU job)
    SParams S = sparse_params(pl, st.P);
    for (int nu = 0; nu < iters; ++nu) {
      CU(sparse_launch(S, LaunchWin{nu, nu + 1, 1, 0}, pl->sp_ctas, pl->sp_smem, pl->stream));
      CU(sparse_launch(S, LaunchWin{nu, nu + 1, 2, 0}, pl->sp_ctas, pl->sp_smem, pl->stream));
    }
  } else if (pl->use_sparse) {
    SParams S = sparse_params(pl, st.P);
    if (pl->SUBCTR) CU(cudaMemsetAsync(pl->SUBCTR, 0, 4 * sizeof(unsigned int), pl->stream));
    CU(sparse_launch(S, LaunchWin{0, iters, 3, 0}, pl->sp_ctas, pl->sp_smem, pl->stream));
  } else if (launch_apg(pl, st.P)) {
    return TSMPC_ERR_CUDA;
  }
  CU(cudaEventRecord(pl->ev1, pl->stream));
  CU(cudaEventSynchronize(pl->ev1));
  float f = 0.f;
  CU(cudaEventElapsedTime(&f, pl->ev0, pl->ev1));
  *ms = f;
  return TSMPC_OK;
}

int tsmpc_set_stopping(tsmpc_plan* pl, double tol, int32_t check_every) {
  if (!pl) return fail(TSMPC_ERR_ARGUMENT, "null argument");
  if (check_every < 1) return fail(TSMPC_ERR_VALIDATION, "check_every must be >= 1");
  if (tol > 0.0 && (!pl->use_sparse || pl->sharded))
    return fail(TSMPC_ERR_VALIDATION, "the residual stopping test needs a single-GPU structured-basis plan "
                                      "(this plan runs the %s kernel)", pl->use_sparse ? "sharded" : "dense");
  pl->tol = tol > 0.0 ? tol : 0.0;
  pl->check_every = check_every;
  return TSMPC_OK;
}

int tsmpc_solve_step(tsmpc_plan* pl, const double* w_sig, const double* w_zeta, const double* w_psi,
                     const double* p, double* x_out, double* u_out) {
  if (!pl || !w_sig || !w_zeta || !w_psi || !p) return fail(TSMPC_ERR_ARGUMENT, "null argument");
  if (!pl->has_cache) return fail(TSMPC_ERR_VALIDATION, "no stage cache uploaded (tsmpc_set_cache)");
  CU(cudaSetDevice(pl->device));
  const int E = pl->E, NXP = pl->NXP, NUP = pl->NUP;
  if (pl->put_rows(pl->WB, NXP, w_sig, pl->nx, E) || pl->put_rows(pl->WB + (size_t)E * NXP, NXP, w_zeta, pl->nx, E) ||
      pl->put_rows(pl->WB + 2 * (size_t)E * NXP, NUP, w_psi, pl->nu, E))
    return TSMPC_ERR_CUDA;
  if (set_root(pl, p)) return TSMPC_ERR_CUDA;
  if (run_step(pl, pl->WB, 0, pl->BETA, pl->UHAT, pl->EVEC)) return TSMPC_ERR_CUDA;
  if (pl->get_rows(x_out, pl->nx, pl->X, NXP, pl->n_nodes) || pl->get_rows(u_out, pl->nu, pl->U, NUP, E))
    return TSMPC_ERR_CUDA;
  CU(cudaStreamSynchronize(pl->stream));
  return TSMPC_OK;
}

int tsmpc_prox(tsmpc_plan* pl, int32_t rows, const double* t_sig, const double* t_zeta, const double* t_psi,
               double lam, int32_t use_scaling, double* o_sig, double* o_zeta, double* o_psi) {
  if (!pl || !t_sig || !t_zeta || !t_psi || !o_sig || !o_zeta || !o_psi) return fail(TSMPC_ERR_ARGUMENT, "null argument");
  if (!(lam > 0.0)) return fail(TSMPC_ERR_VALIDATION, "prox parameter must be positive");
  if (use_scaling && rows != pl->E) return fail(TSMPC_ERR_DIMENSION, "scaled prox needs one row per edge");
  if (rows < 1) return TSMPC_OK;
  CU(cudaSetDevice(pl->device));
  const int nx = pl->nx, nu = pl->nu;
  double *d_ts, *d_tz, *d_tp, *d_os, *d_oz, *d_op;
  const size_t nxr = (size_t)rows * nx, nur = (size_t)rows * nu;
  CU(cudaMallocAsync((void**)&d_ts, sizeof(double) * (4 * nxr + 2 * nur), pl->stream));
  d_tz = d_ts + nxr; d_os = d_tz + nxr; d_oz = d_os + nxr; d_tp = d_oz + nxr; d_op = d_tp + nur;
  CU(cudaMemcpyAsync(d_ts, t_sig, sizeof(double) * nxr, cudaMemcpyHostToDevice, pl->stream));
  CU(cudaMemcpyAsync(d_tz, t_zeta, sizeof(double) * nxr, cudaMemcpyHostToDevice, pl->stream));
  CU(cudaMemcpyAsync(d_tp, t_psi, sizeof(double) * nur, cudaMemcpyHostToDevice, pl->stream));
  ProxArgs a{};
  a.rows = rows; a.nx = nx; a.nu = nu; a.lam = lam; a.Wx = pl->ctx.Wx; a.gamma_d = pl->ctx.gamma_d;
  const bool sc = use_scaling && pl->base.scaled;
  a.edge_stage = sc ? pl->base.edge_stage : nullptr;
  a.sig_stage = sc ? pl->sig_c : nullptr;
  a.zeta_stage = sc ? pl->zeta_c : nullptr;
  a.psi_stage = sc ? pl->psi_c : nullptr;
  a.x_s = pl->base.x_s; a.x_min = pl->base.x_min; a.x_max = pl->base.x_max;
  a.u_min = pl->base.u_min; a.u_max = pl->base.u_max;
  a.t_sig = d_ts; a.t_zeta = d_tz; a.t_psi = d_tp; a.o_sig = d_os; a.o_zeta = d_oz; a.o_psi = d_op;
  prox_kernel<<<grid_for(rows), 256, 0, pl->stream>>>(a);
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(o_sig, d_os, sizeof(double) * nxr, cudaMemcpyDeviceToHost, pl->stream));
  CU(cudaMemcpyAsync(o_zeta, d_oz, sizeof(double) * nxr, cudaMemcpyDeviceToHost, pl->stream));
  CU(cudaMemcpyAsync(o_psi, d_op, sizeof(double) * nur, cudaMemcpyDeviceToHost, pl->stream));
  CU(cudaFreeAsync(d_ts, pl->stream));
  CU(cudaStreamSynchronize(pl->stream));
  return TSMPC_OK;
}

int tsmpc_dual_operator_begin(tsmpc_plan* pl, const double* beta0) {
  if (!pl || !beta0) return fail(TSMPC_ERR_ARGUMENT, "null argument");
  CU(cudaSetDevice(pl->device));
  const int E = pl->E;
  if (pl->put_rows(pl->BETA0, pl->NVP, beta0, pl->nv, E)) return TSMPC_ERR_CUDA;
  const size_t yblk = 2 * (size_t)E * pl->NXP + (size_t)E * pl->NUP;
  CU(cudaMemsetAsync(pl->PY, 0, sizeof(double) * yblk, pl->stream));
  if (set_root(pl, nullptr)) return TSMPC_ERR_CUDA;
  if (run_step(pl, pl->PY, 1, pl->BETA0, nullptr, nullptr)) return TSMPC_ERR_CUDA;
  CU(cudaMemcpyAsync(pl->Z0X, pl->X, sizeof(double) * (size_t)pl->n_nodes * pl->NXP, cudaMemcpyDeviceToDevice, pl->stream));
  CU(cudaMemcpyAsync(pl->Z0U, pl->U, sizeof(double) * (size_t)E * pl->NUP, cudaMemcpyDeviceToDevice, pl->stream));
  CU(cudaStreamSynchronize(pl->stream));
  pl->has_op = true;
  return TSMPC_OK;
}

int tsmpc_dual_operator_set_ones(tsmpc_plan* pl) {
  if (!pl || !pl->has_op) return fail(TSMPC_ERR_ARGUMENT, "dual operator not initialised");
  const int E = pl->E;
  std::vector<double> ones((size_t)E * std::max(pl->nx, pl->nu), 1.0);
  if (pl->put_rows(pl->PY, pl->NXP, ones.data(), pl->nx, E) ||
      pl->put_rows(pl->PY + (size_t)E * pl->NXP, pl->NXP, ones.data(), pl->nx, E) ||
      pl->put_rows(pl->PY + 2 * (size_t)E * pl->NXP, pl->NUP, ones.data(), pl->nu, E))
    return TSMPC_ERR_CUDA;
  CU(cudaStreamSynchronize(pl->stream));
  return TSMPC_OK;
}

int tsmpc_dual_operator_step(tsmpc_plan* pl, double* y_dot_dy, double* dy_dot_dy, double* y_dot_y) {
  if (!pl || !pl->has_op) return fail(TSMPC_ERR_ARGUMENT, "dual operator not initialised");
  CU(cudaSetDevice(pl->device));
  EdgeCtx c = pl->ctx;
  if (!pl->base.scaled) { c.sig_stage = c.zeta_stage = c.psi_stage = nullptr; }
  const int E = pl->E, G = grid_for(E);
  dual_sq_rows_kernel<<<G, 256, 0, pl->stream>>>(c, pl->PY, pl->ROWS);
  reduce_cols_kernel<<<1, 1024, 0, pl->stream>>>(pl->ROWS, E, 3, pl->RED);
  double sq[3];
  CU(cudaMemcpyAsync(sq, pl->RED, sizeof(sq), cudaMemcpyDeviceToHost, pl->stream));
  CU(cudaStreamSynchronize(pl->stream));
  const double yy = (sq[0] + sq[1]) + sq[2];
  if (y_dot_y) *y_dot_y = yy;
  if (!(yy > 0.0)) return fail(TSMPC_ERR_VALIDATION, "dual operator vanished during power iteration");
  dual_normalize_kernel<<<G, 256, 0, pl->stream>>>(c, pl->PY, pl->RED);
  CU(cudaGetLastError());
  if (set_root(pl, nullptr)) return TSMPC_ERR_CUDA;
  if (run_step(pl, pl->PY, 1, pl->BETA0, nullptr, nullptr)) return TSMPC_ERR_CUDA;
  dual_apply_kernel<<<G, 256, 0, pl->stream>>>(c, pl->PY, pl->X, pl->U, pl->Z0X, pl->Z0U, pl->ROWS);
  reduce_cols_kernel<<<1, 1024, 0, pl->stream>>>(pl->ROWS, E, 6, pl->RED);
  CU(cudaGetLastError());
  double d[6];
  CU(cudaMemcpyAsync(d, pl->RED, sizeof(d), cudaMemcpyDeviceToHost, pl->stream));
  CU(cudaStreamSynchronize(pl->stream));
  if (y_dot_dy) *y_dot_dy = (d[0] + d[1]) + d[2];
  if (dy_dot_dy) *dy_dot_dy = (d[3] + d[4]) + d[5];
  return TSMPC_OK;
}

}  // extern "C"

int tsmpc_plans_create_multi(const tsmpc_problem* pb, const int32_t* devices, int32_t n, tsmpc_plan** out) {
  if (!pb || !devices || !out) return fail(TSMPC_ERR_ARGUMENT, "null argument");
  if (n < 1 || n > 64) return fail(TSMPC_ERR_ARGUMENT, "device count %d outside 1..64", n);
  std::string why;
  const NcclApi* api = nccl_api(why);
  if (!api) return fail(TSMPC_ERR_NCCL, "%s", why.c_str());
  std::vector<tsmpc_plan*> plans(n, nullptr);
  auto cleanup = [&]() {
    for (tsmpc_plan* p : plans) delete p;
  };
  for (int r = 0; r < n; ++r) {
    plans[r] = plan_create_impl(pb, devices[r], r, n, nullptr);  // local shard plan of rank r
    if (!plans[r]) {
      const std::string e = g_err;
      cleanup();
      return fail(TSMPC_ERR_VALIDATION, "rank %d: %s", r, e.c_str());
    }
  }
  std::vector<NcclApi::Comm> comms(n, nullptr);
  std::vector<int> devs(devices, devices + n);
  const int nr = api->CommInitAll(comms.data(), n, devs.data());
  if (nr != 0) {
    cleanup();
    return fail(TSMPC_ERR_NCCL, "ncclCommInitAll(%d devices): %s", n, api->GetErrorString(nr));
  }
  for (int r = 0; r < n; ++r) {
    plans[r]->nccl = api;
    plans[r]->comm = comms[r];
    plans[r]->multi = true;
    out[r] = plans[r];
  }
  // the in-kernel cut exchange when every pair of devices can map each other's memory
  bool peers = !std::getenv("TSMPC_NO_PEER");
  for (int r = 0; r < n && peers; ++r) peers = peer_capable(plans[r]) && plans[r]->sp_ctas == plans[0]->sp_ctas;
  for (int r = 0; r < n && peers; ++r)
    for (int q = 0; q < n && peers; ++q) {
      if (q == r || devices[q] == devices[r]) {
        peers = q == r;
        continue;
      }
      int ok = 0;
      if (cudaDeviceCanAccessPeer(&ok, devices[r], devices[q]) != cudaSuccess || !ok) {
        peers = false;
        break;
      }
      cudaSetDevice(devices[r]);
      const cudaError_t e = cudaDeviceEnablePeerAccess(devices[q], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) peers = false;
      cudaGetLastError();
    }
  if (peers) {
    std::vector<double*> rx(n);
    std::vector<unsigned long long*> cnt(n);
    for (int r = 0; r < n; ++r) {
      rx[r] = plans[r]->RX;
      cnt[r] = plans[r]->RXCNT;
    }
    for (int r = 0; r < n; ++r)
      if (peer_setup(plans[r], rx, cnt, (unsigned long long)n * plans[r]->sp_ctas)) {
        for (int q = 0; q < n; ++q) tsmpc_plan_peer_close(plans[q]);
        cudaGetLastError();
        break;
      }
  }
  return TSMPC_OK;
}

int tsmpc_solve_multi(tsmpc_plan* const* plans, int32_t n, const double* p, int32_t iters, double lam,
                      const double* theta, const double* coef, int32_t flags, tsmpc_result* outs) {
  if (!plans || !p || !outs) return fail(TSMPC_ERR_ARGUMENT, "null argument");
  if (n < 1 || n > 64) return fail(TSMPC_ERR_ARGUMENT, "plan count %d outside 1..64", n);
  for (int r = 0; r < n; ++r) {
    const tsmpc_plan* pl = plans[r];
    if (!pl || !pl->multi || pl->world != n || pl->rank != r || !pl->comm)
      return fail(TSMPC_ERR_VALIDATION, "member %d must be rank %d of a tsmpc_plans_create_multi set of %d", r, r, n);
  }
  if (flags & TSMPC_GAP_TRACE) return fail(TSMPC_ERR_VALIDATION, "no per-iteration gap on multi-GPU solves");
  const NcclApi* api = plans[0]->nccl;
  std::vector<SolveState> st(n);
  std::vector<SParams> S(n);
  for (int r = 0; r < n; ++r) {
    int rc = solve_prepare(plans[r], p, iters, lam, nullptr, nullptr, nullptr, theta, coef, flags, st[r]);
    if (rc) return rc;
    S[r] = sparse_params(plans[r], st[r].P);
    CU(cudaEventRecord(plans[r]->ev0, plans[r]->stream));
  }
  auto nccl = [&](int nr) -> int {
    return nr == 0 ? TSMPC_OK : fail(TSMPC_ERR_NCCL, "NCCL: %s", api->GetErrorString(nr));
  };
  const size_t hs = (size_t)S[0].n_xch * S[0].XCH_LD;
  bool fused = !std::getenv("TSMPC_NO_PEER");
  for (int r = 0; r < n; ++r) fused = fused && plans[r]->peer_on;
  if (fused) {  // every GPU: both phases and the cut exchange over peer memory, one launch
    for (int r = 0; r < n; ++r) {
      CU(cudaSetDevice(plans[r]->device));
      CU(sparse_launch(S[r], LaunchWin{0, iters, 7, 0, plans[r]->xgen}, plans[r]->sp_ctas, plans[r]->sp_smem,
                       plans[r]->stream));
      plans[r]->xgen += (unsigned long long)iters;
      plans[r]->launches += 1;
    }
  }
  for (int nu = 0; nu < iters && !fused; ++nu) {
    for (int r = 0; r < n; ++r) {
      CU(cudaSetDevice(plans[r]->device));
      CU(sparse_launch(S[r], LaunchWin{nu, nu + 1, 1, 0}, plans[r]->sp_ctas, plans[r]->sp_smem, plans[r]->stream));
    }
    if (plans[0]->sp_trunk > 0 && hs > 0) {
      if (nccl(api->GroupStart())) return TSMPC_ERR_NCCL;
      for (int r = 0; r < n; ++r)
        if (nccl(api->AllReduce(plans[r]->XCH, plans[r]->XCH, hs, NcclApi::kFloat64, NcclApi::kSum, plans[r]->comm,
                                plans[r]->stream)))
          return TSMPC_ERR_NCCL;
      if (nccl(api->GroupEnd())) return TSMPC_ERR_NCCL;
    }
    for (int r = 0; r < n; ++r) {
      CU(cudaSetDevice(plans[r]->device));
      CU(sparse_launch(S[r], LaunchWin{nu, nu + 1, 2, 0}, plans[r]->sp_ctas, plans[r]->sp_smem, plans[r]->stream));
      plans[r]->launches += 2;
    }
  }
  // residual: max over ranks
  if (nccl(api->GroupStart())) return TSMPC_ERR_NCCL;
  for (int r = 0; r < n; ++r)
    if (nccl(api->AllReduce(plans[r]->RESID, plans[r]->RESID, (size_t)st[r].nres, NcclApi::kUint64, NcclApi::kMax,
                            plans[r]->comm, plans[r]->stream)))
      return TSMPC_ERR_NCCL;
  if (nccl(api->GroupEnd())) return TSMPC_ERR_NCCL;
  for (int r = 0; r < n; ++r) {
    CU(cudaSetDevice(plans[r]->device));
    CU(cudaEventRecord(plans[r]->ev1, plans[r]->stream));
  }
  const bool gap = !(flags & TSMPC_SKIP_GAP);
  if (gap) {
    // the full averages and final dual on every GPU (each row counted once)
    for (int r = 0; r < n; ++r) {
      CU(cudaSetDevice(plans[r]->device));
      double* yfin = (iters & 1) == 0 ? plans[r]->Y0 : plans[r]->Y1;
      if (zero_replicated_rows(plans[r], yfin, plans[r]->stream)) return TSMPC_ERR_CUDA;
    }
    const size_t yblk = 2 * (size_t)plans[0]->E * plans[0]->NXP + (size_t)plans[0]->E * plans[0]->NUP;
    if (nccl(api->GroupStart())) return TSMPC_ERR_NCCL;
    for (int r = 0; r < n; ++r) {
      tsmpc_plan* pl = plans[r];
      double* yfin = (iters & 1) == 0 ? pl->Y0 : pl->Y1;
      if (nccl(api->AllReduce(pl->XAVG, pl->XAVG, (size_t)pl->n_nodes * pl->NXP, NcclApi::kFloat64, NcclApi::kSum,
                              pl->comm, pl->stream)) ||
          nccl(api->AllReduce(pl->UAVG, pl->UAVG, (size_t)pl->E * pl->NUP, NcclApi::kFloat64, NcclApi::kSum, pl->comm,
                              pl->stream)) ||
          nccl(api->AllReduce(yfin, yfin, yblk, NcclApi::kFloat64, NcclApi::kSum, pl->comm, pl->stream)))
        return TSMPC_ERR_NCCL;
    }
    if (nccl(api->GroupEnd())) return TSMPC_ERR_NCCL;
  }
  for (int r = 0; r < n; ++r) {
    int rc = solve_finish(plans[r], st[r], flags, outs + r, gap);
    if (rc) return rc;
  }
  return TSMPC_OK;
}
