// tsmpc_sparse_host.cpp — host planner of the structured-basis kernel.
//
// Tree terms follow the reference's layout (tree.py:31-94): stage-major nodes,
// edge e <-> node e+1, children of a node contiguous.  A *leaf chain* is a
// maximal only-child path ending at a leaf; its first edge is the chain head,
// whose parent node has != 1 children (or is the root).  Every other edge is a
// *trunk* edge.  For the paper's trees (branching in stages <= 3, then one
// chain per scenario) the chains carry ~99% of the edges.
#include "tsmpc_sparse_host.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <queue>
#include <set>

namespace tsmpc {

namespace {

void csr(int rows, int cols, const std::vector<double>& dense, bool by_col, std::vector<int>& ptr,
         std::vector<int>& idx, std::vector<double>& val) {
  // dense is rows x cols row-major; by_col -> compressed columns
  const int outer = by_col ? cols : rows, inner = by_col ? rows : cols;
  ptr.assign(outer + 1, 0);
  idx.clear();
  val.clear();
  for (int o = 0; o < outer; ++o) {
    for (int i = 0; i < inner; ++i) {
      const double v = by_col ? dense[(size_t)i * cols + o] : dense[(size_t)o * cols + i];
      if (v != 0.0) {
        idx.push_back(i);
        val.push_back(v);
      }
    }
    ptr[o + 1] = (int)idx.size();
  }
}

}  // namespace

SparseHostPlan plan_sparse(const SparseTreeIn& t, const SparseOpsIn& ops, int NXP, int NUP, int NVP,
                           int max_ctas, size_t smem_limit, bool sharded, int rank, int world, bool psi_in_smem,
                           bool allow_split, bool wide) {
  const int tile_lim = wide ? kTileW : kTileS;
  SparseHostPlan out;
  out.rank = rank;
  out.world = world;
  if (world < 1 || rank < 0 || rank >= world) {
    out.why = "invalid shard rank/world";
    return out;
  }
  const int n_nodes = t.n_nodes, E = n_nodes - 1, N = t.N;
  const int nx = ops.nx, nu = ops.nu, nv = ops.nv;
  std::vector<int> nch(n_nodes), stage_of_edge(E);
  for (int n = 0; n < n_nodes; ++n) nch[n] = (int)(t.child_stop[n] - t.child_start[n]);
  for (int j = 0; j < N; ++j)
    for (int64_t n = t.stage_starts[j + 1]; n < t.stage_starts[j + 2]; ++n) stage_of_edge[n - 1] = j;

  // ---- leaf chains and trunk
  std::vector<std::vector<int>> chains;
  std::vector<char> in_chain(E, 0);
  for (int e = 0; e < E; ++e) {
    const int pn = (int)t.anc[e + 1];
    const bool head = pn == 0 || nch[pn] != 1;
    if (!head) continue;
    std::vector<int> path{e};
    int x = e;
    while (nch[x + 1] == 1) {
      x = (int)t.child_start[x + 1] - 1;
      path.push_back(x);
    }
    if (nch[x + 1] == 0) {
      if ((int)path.size() > tile_lim) {
        out.why = "leaf chain longer than a tile (" + std::to_string(path.size()) + " edges)";
        return out;
      }
      for (int c : path) in_chain[c] = 1;
      chains.push_back(std::move(path));
    }
  }
  std::vector<int> tpos(E, -1);
  for (int e = 0; e < E; ++e)
    if (!in_chain[e]) {
      tpos[e] = (int)out.trunk_edge.size();
      out.trunk_edge.push_back(e);
    }
  const int T = (int)out.trunk_edge.size();
  out.n_trunk = T;
  out.n_chains = (int)chains.size();
  std::sort(chains.begin(), chains.end(), [](const auto& a, const auto& b) { return a[0] < b[0]; });
  out.total_chains = (int)chains.size();
  // ---- sharding: groups of chains hanging from the same node, split contiguously
  out.towned.assign(T, 1);
  out.trole.assign(T, kRoleOwn);
  out.txrow.assign(T, -1);
  // (world 1 with TSMPC_SHARD_FULL: the one rank exchanges every position's head sums
  // with itself -- exercises the exchange paths on a single GPU)
  if (sharded && (world > 1 || std::getenv("TSMPC_SHARD_FULL"))) {
    std::vector<int> gnode;             // group -> parent node
    std::vector<long long> grows;       // group -> rows
    std::vector<int> group_of(chains.size());
    for (size_t i = 0; i < chains.size(); ++i) {
      const int pn = (int)t.anc[chains[i][0] + 1];
      if (gnode.empty() || gnode.back() != pn) {
        // chains are sorted by head edge, and siblings are contiguous edges
        gnode.push_back(pn);
        grows.push_back(0);
      }
      group_of[i] = (int)gnode.size() - 1;
      grows.back() += (long long)chains[i].size();
    }
    long long Rg = 0;
    for (long long r : grows) Rg += r;
    std::vector<int> gowner(gnode.size());
    long long pre = 0;
    for (size_t gi = 0; gi < gnode.size(); ++gi) {
      const long long mid2 = 2 * pre + grows[gi];
      gowner[gi] = std::min(world - 1, (int)((mid2 * world) / (2 * std::max<long long>(Rg, 1))));
      pre += grows[gi];
    }
    std::vector<std::vector<int>> kept;
    for (size_t i = 0; i < chains.size(); ++i)
      if (gowner[group_of[i]] == rank) kept.push_back(chains[i]);
    for (int tp = 0; tp < T; ++tp) out.towned[tp] = 0;
    for (size_t gi = 0; gi < gnode.size(); ++gi)
      if (gowner[gi] == rank && gnode[gi] > 0 && tpos[gnode[gi] - 1] >= 0) out.towned[tpos[gnode[gi] - 1]] = 1;
    // the cut: ranks owning chains below each trunk position
    std::vector<int> towner(T, -2);  // -2: none yet, -1: several ranks
    for (size_t i = 0; i < chains.size(); ++i) {
      const int g = gowner[group_of[i]];
      for (int e = (int)t.anc[chains[i][0] + 1] - 1; e >= 0; e = (int)t.anc[e + 1] - 1) {
        int& o = towner[tpos[e]];
        o = (o == -2 || o == g) ? g : -1;
      }
    }
    std::vector<int> xrow(T, -1);
    for (int tp = 0; tp < T; ++tp) {
      const int pa = (int)t.anc[out.trunk_edge[tp] + 1] - 1;
      const bool cut = pa >= 0 && towner[tpos[pa]] < 0;
      if (towner[tp] < 0) out.trole[tp] = kRoleMixed;
      else if (towner[tp] == rank) out.trole[tp] = cut ? kRoleCutOwn : kRoleOwn;
      else out.trole[tp] = cut ? kRoleCutForeign : kRoleForeign;
      if (towner[tp] < 0 || cut) xrow[tp] = out.n_xch++;
    }
    out.txrow = xrow;
    out.cut = true;
    // small trunks (SMPC3 on 8 ranks: 32 cut rows of 344 doubles vs 37 x 164 head
    // sums): replicate the whole trunk and exchange every position's head sums
    if ((long long)out.n_xch * (NVP + 2 * NXP + NUP) >= (long long)T * (NVP + NXP) ||
        std::getenv("TSMPC_SHARD_FULL")) {
      out.cut = false;
      out.n_xch = T;
      for (int tp = 0; tp < T; ++tp) {
        out.trole[tp] = kRoleMixed;
        out.txrow[tp] = tp;
      }
    }
    chains.swap(kept);
  }
  out.n_chains = (int)chains.size();
  for (auto& ch : chains) {
    out.owned_rows += (int)ch.size();
    out.owned_edges.insert(out.owned_edges.end(), ch.begin(), ch.end());
  }
  std::sort(out.owned_edges.begin(), out.owned_edges.end());
  out.result_edges = out.owned_edges;
  for (int tp = 0; tp < T; ++tp)
    if (out.trole[tp] != kRoleForeign && out.trole[tp] != kRoleCutForeign) out.result_edges.push_back(out.trunk_edge[tp]);
  std::sort(out.result_edges.begin(), out.result_edges.end());

  // ---- split mode: a CTA per chain, the trunk on split_n further CTAs
  int split_n = 0;
  const int ncomp_all = nv + nx + nu;
  if (allow_split && !wide && !sharded && T > 0 && !chains.empty() && !std::getenv("TSMPC_NO_SPLIT")) {
    const int spare = max_ctas - (int)chains.size();
    // enough trunk CTAs that one sweep slice (T x components) stays under ~300 items
    // (measured on SMPC3: 27 CTAs at 384 items 22.5 us/iteration, 34 at 300 22.2)
    int want = std::max(kMinTrunkCtas, (int)(((long long)ncomp_all * T + 299) / 300));
    if (const char* e = std::getenv("TSMPC_TRUNK_CTAS")) want = std::max(kMinTrunkCtas, std::atoi(e));
    if (spare >= kMinTrunkCtas) split_n = std::min(spare, want);
  }
  // ---- CTA count and chain assignment (contiguous, balanced by rows)
  long long R = 0;
  for (auto& ch : chains) R += (long long)ch.size();
  // rows of the fullest CTA when the chains are spread over C CTAs by the midpoint rule
  auto fullest = [&](int C) {
    std::vector<long long> rows(C, 0);
    long long pre = 0, mx = 0;
    for (auto& ch : chains) {
      const long long mid2 = 2 * pre + (long long)ch.size();
      const int c = std::min(std::max((int)((mid2 * C) / (2 * std::max<long long>(R, 1))), 0), C - 1);
      mx = std::max(mx, rows[c] += (long long)ch.size());
      pre += (long long)ch.size();
    }
    return mx;
  };
  // wide split mode: the fewest chain CTAs that keep the fullest CTA at its
  // all-CTA load (one wide tile each); the rest run the trunk
  int nch_wide = 0;
  if (wide && allow_split && !sharded && T > 0 && !chains.empty() && !std::getenv("TSMPC_NO_SPLIT")) {
    const long long full = fullest(max_ctas);
    if (full <= kTileW) {
      for (int c0 = (int)std::max<long long>(1, (R + full - 1) / full); c0 <= max_ctas - kMinTrunkCtas; ++c0)
        if (fullest(c0) <= full) {
          nch_wide = c0;
          break;
        }
      if (const char* e = std::getenv("TSMPC_TRUNK_CTAS"))
        nch_wide = std::max(nch_wide, max_ctas - std::max(kMinTrunkCtas, std::atoi(e)));
      if (nch_wide > 0) split_n = max_ctas - nch_wide;
    }
  }
  const int nch_split = split_n ? (nch_wide ? nch_wide : (int)chains.size()) : 0;
  int C = T > 0 ? max_ctas : std::max(1, std::min(max_ctas, (int)chains.size()));
  if (T > 0) C = std::max(1, std::min(max_ctas, (int)chains.size() + T));
  if (split_n) C = nch_split + split_n;
  std::vector<std::vector<int>> cta_chains(C);
  if (split_n && !nch_wide) {
    for (int i = 0; i < nch_split; ++i) cta_chains[i].push_back(i);
  } else {
    const int Cc = nch_wide ? nch_wide : C;  // CTAs holding chains
    long long pre = 0;
    for (int i = 0; i < (int)chains.size(); ++i) {
      const long long mid2 = 2 * pre + (long long)chains[i].size();
      int c = (int)((mid2 * Cc) / (2 * std::max<long long>(R, 1)));
      c = std::min(std::max(c, 0), Cc - 1);
      cta_chains[c].push_back(i);
      pre += (long long)chains[i].size();
    }
  }
  // trunk rows -> the CTA minimising load + 4 x (new "needs": trunk edges on the
  // row's root path the CTA does not evaluate yet; 0 when its chains hang below
  // the edge); at most ceil(T / C) + 1 rows per CTA.
  // This keeps each CTA's needs close to its chains' root paths (also on shards,
  // where many trunk edges have no owned chains below them).
  std::vector<std::vector<int>> cta_own(C);
  // depth-0 ancestor (trunk subtree root) of every trunk position
  std::vector<int> troot(T, -1);
  for (int tp = 0; tp < T; ++tp) {
    int e = out.trunk_edge[tp];
    while ((int)t.anc[e + 1] - 1 >= 0) e = (int)t.anc[e + 1] - 1;
    troot[tp] = tpos[e];
  }
  if (split_n) {  // trunk rows in contiguous runs of (subtree, position) order
    std::vector<int> order(T);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return troot[a] < troot[b]; });
    for (int i = 0; i < T; ++i) cta_own[nch_split + (int)((long long)i * split_n / T)].push_back(order[i]);
  } else {
    std::vector<long long> load(C, 0);
    std::vector<std::set<int>> need(C);
    for (int c = 0; c < C; ++c)
      for (int i : cta_chains[c]) {
        load[c] += (long long)chains[i].size();
        for (int e = (int)t.anc[chains[i][0] + 1] - 1; e >= 0; e = (int)t.anc[e + 1] - 1) need[c].insert(tpos[e]);
      }
    const int cap_rows = (T + C - 1) / std::max(C, 1) + 1;
    std::vector<int> path;
    for (int tp = 0; tp < T; ++tp) {
      if (out.trole[tp] == kRoleForeign || out.trole[tp] == kRoleCutForeign) continue;  // another rank's
      path.clear();
      for (int e = out.trunk_edge[tp]; e >= 0; e = (int)t.anc[e + 1] - 1) path.push_back(tpos[e]);
      int best = -1, best_add = 0;
      for (int c = 0; c < C; ++c) {
        if ((int)cta_own[c].size() >= cap_rows) continue;
        int add = 0;
        for (int q : path) add += need[c].count(q) ? 0 : 1;
        // a new need costs ~4 rows of work (it is evaluated once per iteration)
        const long long cost = load[c] + 4LL * add;
        if (best < 0 || cost < load[best] + 4LL * best_add) {
          best = c;
          best_add = add;
        }
      }
      if (best < 0) best = tp % C;
      cta_own[best].push_back(tp);
      load[best] += 1;
      for (int q : path) need[best].insert(q);
    }
  }

  // ---- trunk schedule
  {
    std::vector<int> lev_ptr;  // trunk positions grouped by edge stage (ascending)
    int last_stage = -1;
    for (int tp = 0; tp < T; ++tp) {
      const int st = stage_of_edge[out.trunk_edge[tp]];
      if (st != last_stage) {
        lev_ptr.push_back(tp);
        last_stage = st;
      }
    }
    lev_ptr.push_back(T);
    const int nlev = (int)lev_ptr.size() - 1;
    std::vector<int> pos(8 * (size_t)T, 0), tch, hch;
    for (int tp = 0; tp < T; ++tp) {
      const int a = out.trunk_edge[tp], node = a + 1;
      const int pa = (int)t.anc[node] - 1;
      int* p = &pos[8 * (size_t)tp];
      p[0] = a;
      p[1] = stage_of_edge[a];
      p[2] = pa >= 0 ? tpos[pa] : -1;
      p[3] = (int)tch.size();
      p[5] = (int)hch.size();
      std::vector<int> hc;
      for (int64_t ch = t.child_start[node] - 1; ch < t.child_stop[node] - 1; ++ch) {
        if (tpos[ch] >= 0) tch.push_back(tpos[ch]);
        else hch.push_back((int)ch);
      }
      p[4] = (int)tch.size() - p[3];
      p[6] = (int)hch.size() - p[5];
      p[7] = out.trole[tp] | ((out.txrow[tp] + 1) << 3);
    }
    out.tsched = {T, nlev, (int)tch.size(), (int)hch.size()};
    if (T == 0) out.tsched[1] = 0;
    if (T > 0) out.tsched.insert(out.tsched.end(), lev_ptr.begin(), lev_ptr.end());
    else out.tsched.push_back(0);
    out.tsched.insert(out.tsched.end(), pos.begin(), pos.end());
    out.tsched.insert(out.tsched.end(), tch.begin(), tch.end());
    out.tsched.insert(out.tsched.end(), hch.begin(), hch.end());
  }

  // ---- per-CTA meta
  std::vector<int> depth(T, 0);
  for (int tp = 0; tp < T; ++tp) {
    int d = 0;
    for (int e = out.trunk_edge[tp]; e >= 0; e = (int)t.anc[e + 1] - 1) ++d;
    depth[tp] = d;
  }
  std::vector<int> cta_rows(C, 0), cta_needs(C, 0);
  int sub_max = 0;  // largest trunk-subtree set of a split-mode trunk CTA
  std::vector<std::vector<int>> metas(C);
  int total_tiles = 0;
  for (int c = 0; c < C; ++c) {
    // tiles: consecutive chains packed up to tile_lim rows
    std::vector<std::vector<int>> tiles;
    int fill = tile_lim + 1;
    for (int i : cta_chains[c]) {
      const int len = (int)chains[i].size();
      if (fill + len > tile_lim) {
        tiles.emplace_back();
        fill = 0;
      }
      tiles.back().push_back(i);
      fill += len;
    }
    // needs: trunk paths of the chain heads' parents and of own trunk rows
    std::set<std::pair<int, int>> need_set;  // (depth, tp)
    auto add_path = [&](int e) {
      for (; e >= 0; e = (int)t.anc[e + 1] - 1) need_set.insert({depth[tpos[e]], tpos[e]});
    };
    if (!split_n)  // split mode: chain CTAs read their trunk parents from TR
      for (int i : cta_chains[c]) {
        const int pa = (int)t.anc[chains[i][0] + 1] - 1;
        if (pa >= 0) add_path(pa);
      }
    for (int tp : cta_own[c]) add_path(out.trunk_edge[tp]);
    std::vector<int> need_tp;
    std::map<int, int> need_idx;
    std::vector<int> lev{0};
    int last_d = -1;
    for (auto& [d, tp] : need_set) {
      if (d != last_d && last_d >= 0) lev.push_back((int)need_tp.size());
      last_d = d;
      need_idx[tp] = (int)need_tp.size();
      need_tp.push_back(tp);
    }
    lev.push_back((int)need_tp.size());
    if (need_tp.empty()) lev = {0};
    const int nlev = (int)lev.size() - 1;
    int nrows = 0, nsegs = 0;
    for (auto& tl : tiles)
      for (int i : tl) nrows += (int)chains[i].size(), ++nsegs;
    std::vector<int>& m = metas[c];
    m = {(int)tiles.size(), nrows, nsegs, (int)need_tp.size(), nlev, (int)cta_own[c].size(), 0, 0};
    std::vector<int> rows, segs;
    int row = 0, seg = 0;
    for (auto& tl : tiles) {
      const int row0 = row, seg0 = seg;
      int lo = 0;
      for (int i : tl) {
        const auto& ch = chains[i];
        const int pa = (int)t.anc[ch[0] + 1] - 1;
        const int pref = pa < 0 ? -1 : (split_n ? tpos[pa] : need_idx[tpos[pa]]);
        segs.insert(segs.end(), {lo, lo + (int)ch.size(), pref, 0});
        for (int e : ch) {
          const double inv2p = 1.0 / (2.0 * t.prob[e + 1]);
          int w[2];
          std::memcpy(w, &inv2p, sizeof(w));
          rows.insert(rows.end(), {e, stage_of_edge[e], w[0], w[1]});
        }
        lo += (int)ch.size();
        ++seg;
      }
      row += lo;
      m.insert(m.end(), {row0, lo, seg0, (int)tl.size()});
    }
    m.insert(m.end(), rows.begin(), rows.end());
    m.insert(m.end(), segs.begin(), segs.end());
    for (int tp : need_tp) {
      const int a = out.trunk_edge[tp], pa = (int)t.anc[a + 1] - 1;
      m.insert(m.end(), {tp, pa >= 0 ? need_idx[tpos[pa]] : -1, a, stage_of_edge[a]});
    }
    m.insert(m.end(), lev.begin(), lev.end());
    for (int tp : cta_own[c]) m.push_back(need_idx[tp]);
    if (split_n && c >= nch_split) {
      // the trunk subtrees of the owned rows: {nsub, nslev, slev[nslev+1], sub tp[nsub], local index of tp[T]}
      std::set<int> roots;
      for (int tp : cta_own[c]) roots.insert(troot[tp]);
      std::vector<std::pair<int, int>> sub;  // (depth, tp)
      for (int tp = 0; tp < T; ++tp)
        if (roots.count(troot[tp])) sub.push_back({depth[tp], tp});
      std::sort(sub.begin(), sub.end());
      std::vector<int> slev{0}, stp, lio(T, -1);
      for (size_t i = 0; i < sub.size(); ++i) {
        if (i > 0 && sub[i].first != sub[i - 1].first) slev.push_back((int)i);
        lio[sub[i].second] = (int)i;
        stp.push_back(sub[i].second);
      }
      slev.push_back((int)sub.size());
      if (sub.empty()) slev = {0};
      m.push_back((int)sub.size());
      m.push_back((int)slev.size() - 1);
      m.insert(m.end(), slev.begin(), slev.end());
      m.insert(m.end(), stp.begin(), stp.end());
      m.insert(m.end(), lio.begin(), lio.end());
      sub_max = std::max(sub_max, (int)sub.size());
    }
    cta_rows[c] = nrows;
    cta_needs[c] = (int)need_tp.size();
    total_tiles += (int)tiles.size();
  }
  out.n_tiles = total_tiles;
  out.n_ctas = C;

  // ---- sparse operators
  {
    std::vector<double> Bd(ops.B, ops.B + (size_t)nx * nu), Lsd(ops.Ls, ops.Ls + (size_t)nu * nv),
        Lt((size_t)nu * nv);
    for (int j = 0; j < nu; ++j)
      for (int k = 0; k < nv; ++k) {
        const double l = Lsd[(size_t)j * nv + k];
        Lt[(size_t)j * nv + k] = l == 0.0 ? 0.0 : -(l / ops.lam[k]);
      }
    std::vector<int> p1, i1, p2, i2, p3, i3, p4, i4;
    std::vector<double> v1, v2, v3, v4;
    csr(nx, nu, Bd, true, p1, i1, v1);    // B by column j
    csr(nx, nu, Bd, false, p2, i2, v2);   // B by row i
    csr(nu, nv, Lsd, true, p3, i3, v3);   // Ls by column k
    csr(nu, nv, Lt, false, p4, i4, v4);   // Lt by row j
    SParams& S = out.S;
    auto put = [&](const std::vector<int>& v) { int o = (int)out.spi.size(); out.spi.insert(out.spi.end(), v.begin(), v.end()); return o; };
    auto putv = [&](const std::vector<double>& v) { int o = (int)out.spv.size(); out.spv.insert(out.spv.end(), v.begin(), v.end()); return o; };
    S.Bc_ptr = put(p1); S.Bc_idx = put(i1); S.Bc_val = putv(v1);
    S.Br_ptr = put(p2); S.Br_idx = put(i2); S.Br_val = putv(v2);
    S.Lc_ptr = put(p3); S.Lc_idx = put(i3); S.Lc_val = putv(v3);
    S.Lr_ptr = put(p4); S.Lr_idx = put(i4); S.Lr_val = putv(v4);
    S.n_spi = (int)out.spi.size();
    S.n_spv = (int)out.spv.size();
    // combined trunk-forward operators on a KY row (split mode):
    //   du = Lt (K + Ls'(Ypsi + B' Yx)) = M1 [K | Yx | Ypsi],  B du = (B M1) [K | Yx | Ypsi]
    {
      const int KY_LD = NVP + NXP + NUP;
      std::vector<double> M1((size_t)nu * KY_LD, 0.0), M2((size_t)nx * KY_LD, 0.0);
      std::vector<double> LsB((size_t)nv * nx, 0.0);  // Ls' B' (nv x nx)
      for (int k = 0; k < nv; ++k)
        for (int i = 0; i < nx; ++i) {
          double a = 0.0;
          for (int j = 0; j < nu; ++j) a += Lsd[(size_t)j * nv + k] * Bd[(size_t)i * nu + j];
          LsB[(size_t)k * nx + i] = a;
        }
      for (int j = 0; j < nu; ++j)
        for (int k = 0; k < nv; ++k) {
          const double l = Lt[(size_t)j * nv + k];
          if (l == 0.0) continue;
          M1[(size_t)j * KY_LD + k] += l;
          for (int i = 0; i < nx; ++i) M1[(size_t)j * KY_LD + NVP + i] += l * LsB[(size_t)k * nx + i];
          for (int j2 = 0; j2 < nu; ++j2) M1[(size_t)j * KY_LD + NVP + NXP + j2] += l * Lsd[(size_t)j2 * nv + k];
        }
      for (int i = 0; i < nx; ++i)
        for (int j = 0; j < nu; ++j) {
          const double b = Bd[(size_t)i * nu + j];
          if (b == 0.0) continue;
          for (int col = 0; col < KY_LD; ++col) M2[(size_t)i * KY_LD + col] += b * M1[(size_t)j * KY_LD + col];
        }
      std::vector<int> q1, c1, q2, c2;
      std::vector<double> w1, w2;
      csr(nu, KY_LD, M1, false, q1, c1, w1);
      csr(nx, KY_LD, M2, false, q2, c2, w2);
      auto tput = [&](const std::vector<int>& v) { int o = (int)out.tpi.size(); out.tpi.insert(out.tpi.end(), v.begin(), v.end()); return o; };
      auto tputv = [&](const std::vector<double>& v) { int o = (int)out.tpv.size(); out.tpv.insert(out.tpv.end(), v.begin(), v.end()); return o; };
      S.M1_ptr = tput(q1); S.M1_col = tput(c1); S.M1_val = tputv(w1);
      S.M2_ptr = tput(q2); S.M2_col = tput(c2); S.M2_val = tputv(w2);
      if (out.tpv.empty()) out.tpv.push_back(0.0);
    }
  }

  // ---- shared-memory layout (doubles)
  SParams& S = out.S;
  const int need_max = *std::max_element(cta_needs.begin(), cta_needs.end());
  int meta_max = 0;
  out.meta_ptr.assign(C + 1, 0);
  for (int c = 0; c < C; ++c) {
    meta_max = std::max(meta_max, (int)metas[c].size());
    out.meta_ptr[c + 1] = out.meta_ptr[c] + (int)metas[c].size();
  }
  auto even = [](long long v) { return (v + 1) / 2 * 2; };
  // rows of the work regions: kTileS, or the widest tile of a wide plan
  int tcap = kTileS;
  if (wide) {
    tcap = 1;
    for (int c = 0; c < C; ++c) {
      const int* m = metas[c].data();
      for (int ti = 0; ti < m[0]; ++ti) tcap = std::max(tcap, m[8 + 4 * ti + 1]);
    }
  }
  S.tile_cap = tcap;
  S.wide = wide ? 1 : 0;
  S.YW = 2 * NXP + NUP;
  S.need_ld = NVP + NXP + NUP;
  S.need_max = need_max;
  S.LA = (int)even(std::max(NXP, NVP));
  long long off = 0;
  S.O_BND = 0;
  off += even(5LL * NXP + 2LL * NUP);
  S.O_SCL = (int)off;
  off += even(4LL * N);
  S.O_RED = (int)off;
  off += (5 * tcap + 1) / 2 + 1;  // epilogue row descriptors
  off = even(off);
  S.O_PSI = (int)off;
  S.psi_smem = psi_in_smem ? 1 : 0;
  if (psi_in_smem) off += even((long long)N * NUP);
  S.O_SPV = (int)off;
  off += even(S.n_spv);
  S.O_NEED = (int)off;
  off += (long long)need_max * S.need_ld;
  S.O_WORK = (int)off;
  S.n_work = (int)even((long long)tcap * (S.LA + NUP));
  off += S.n_work;
  S.O_SLOT = (int)off;
  long long ints_d = ((long long)meta_max + S.n_spi + 1) / 2 + 1;
  const long long limit_d = (long long)(smem_limit / sizeof(double));
  long long slot_avail = limit_d - off - ints_d;
  S.rows_window = 0;
  S.O_WIN = 0;
  if (wide && slot_avail < 0 && !std::getenv("TSMPC_NO_WINDOW")) {
    // meta windows: the staged ints keep everything but the rows and segments, which
    // come in per tile (window of 4 tcap row ints + 4 tcap segment ints)
    int compact = 0;
    bool multi = false;
    for (int c = 0; c < C; ++c) {
      compact = std::max(compact, (int)metas[c].size() - 4 * metas[c][1] - 4 * metas[c][2]);
      multi |= metas[c][0] > 1;
    }
    const int wmeta = (compact + 1) / 2 * 2 + 8 * tcap;
    const long long ints_w = ((long long)wmeta + S.n_spi + 1) / 2 + 1;
    if (multi && limit_d - off - ints_w >= 0) {
      S.rows_window = 1;
      S.O_WIN = (compact + 1) / 2 * 2;
      meta_max = wmeta;
      ints_d = ints_w;
      slot_avail = limit_d - off - ints_d;
    }
  }
  // slot rows: both dual rows + ergodic rows; t rows join them only for resident
  // CTAs with several tiles (tmode 1); a single resident tile keeps t in region A
  const long long base_ld = 2LL * S.YW + NXP + NUP;
  const long long t_ld = base_ld + NVP;
  if (std::getenv("TSMPC_PLAN_DEBUG"))
    std::fprintf(stderr, "plan_sparse: rank %d/%d C=%d need_max=%d meta_max=%d n_spi=%d work=%d off=%lld ints_d=%lld "
                 "slot_avail=%lld base_ld=%lld psi=%d\n", rank, world, C, need_max, meta_max, S.n_spi, S.n_work,
                 off, ints_d, slot_avail, base_ld, (int)psi_in_smem);
  if (wide) {
    // no slot rows: t stays in region A when a CTA has one tile (and the launch runs
    // whole iterations), else it goes through TG
    int max_rows_w = 0;
    bool any_t0 = false, any_t2 = false;
    for (int c = 0; c < C; ++c) {
      metas[c][6] = 0;
      metas[c][7] = (metas[c][0] <= 1 && !sharded) ? 0 : 2;
      any_t0 |= metas[c][7] == 0;
      any_t2 |= metas[c][7] == 2;
      max_rows_w = std::max(max_rows_w, cta_rows[c]);
    }
    S.FL = any_t2 ? NXP + NUP : 0;  // fill rows through HBM (FG) for multi-tile / sharded CTAs
    if (std::getenv("TSMPC_PLAN_DEBUG"))
      std::fprintf(stderr, "plan_sparse wide: tcap=%d off=%lld ints_d=%lld limit=%lld psi=%d window=%d\n", tcap, off,
                   ints_d, limit_d, (int)psi_in_smem, S.rows_window);
    if (slot_avail < 0) {
      if (psi_in_smem)
        return plan_sparse(t, ops, NXP, NUP, NVP, max_ctas, smem_limit, sharded, rank, world, false, allow_split,
                           true);
      out.why = "shared memory too small for the wide tiles";
      return out;
    }
    const int ncomp = nv + nx + nu;
    const long long nc_max = (ncomp + C - 1) / C;
    const long long cap = any_t0 ? (long long)tcap * NUP : (long long)S.n_work;
    const long long zx = 2LL * T * nc_max + T;
    const long long sched = ((long long)out.tsched.size() + 1) / 2 + 2;
    S.sweep_in_a = any_t0 ? 0 : 1;
    S.sched_smem = zx + sched <= cap ? 1 : 0;
    if (zx > cap) {
      out.why = "trunk too large for the work region";
      return out;
    }
    S.slot_ld = (int)base_ld;
    S.slot_rows = 0;
    S.wide_prefill = 1;
    S.split = 0;
    S.TR_LD = NUP + 2 * NXP;
    {
      const long long sched_d = ((long long)out.tsched.size() + 1) / 2 + 1;
      S.sched_resident = (T > 0 && off + ints_d + sched_d <= limit_d) ? 1 : 0;
      S.O_SLOT = (int)off;
      S.O_SCHED = (int)off;
      if (S.sched_resident) off += sched_d;
    }
    S.O_INT = (int)off;
    off += ints_d;
    S.O_HSUM = (int)off;
    if (split_n) {
      // chain CTAs: per chain [sum beta_s (NVP)] and a scratch row of max(NXP + 2 NUP,
      // TR_LD) (head sums during the backward, the parent's TR row in the finish)
      int nsm = 1;
      for (int c = 0; c < nch_split; ++c) nsm = std::max(nsm, metas[c][2]);
      const long long hsum = (long long)nsm * (NVP + std::max(NXP + 2LL * NUP, (long long)S.TR_LD));
      const bool fits = off + even(hsum) <= limit_d;
      bool single = true;
      for (int c = 0; c < nch_split; ++c) single &= metas[c][0] == 1;
      if (!fits || !single)  // no room for the head sums / multi-tile chain CTAs: plain wide
        return plan_sparse(t, ops, NXP, NUP, NVP, max_ctas, smem_limit, sharded, rank, world, psi_in_smem, false,
                           true);
      off += even(hsum);
      S.hsum_nseg = nsm;
      S.split = 1;
      S.split_c0 = nch_split;
      S.split_n = split_n;
      S.split_flags = 1;
      S.split_heads = 1;
      S.split_local = 0;
      S.tops = 0;
      S.sweep_in_a = 1;  // the trunk CTAs hold no tiles: the whole work region is theirs
      const long long zx = 2LL * T * ((ncomp + split_n - 1) / split_n) + T;
      S.sched_smem = zx + sched <= (long long)S.n_work ? 1 : 0;
      if (zx > (long long)S.n_work) {
        out.why = "trunk too large for the work region";
        return out;
      }
      // the trunk CTAs' combined forward operators (du = M1 KY, B du = M2 KY: one
      // pass instead of three) after the sweep buffers in region A, staged at launch;
      // the needs' KY / uhat / e rows are staged in region B
      S.n_tpi = (int)out.tpi.size();
      S.n_tpv = (int)out.tpv.size();
      const long long sld = (long long)(NVP + NXP + NUP) + NUP + NXP;
      const long long otops = even(zx + (S.sched_smem && !S.sched_resident ? sched : 0));
      if (otops + S.n_tpv + (S.n_tpi + 1) / 2 + 1 <= (long long)tcap * S.LA && (long long)need_max * sld <= (long long)tcap * NUP &&
          !std::getenv("TSMPC_NO_TOPS")) {
        S.O_SLOT = S.O_WORK;
        S.O_TOPS = (int)otops;
        S.tops = 1;
      }
    }
    if (std::getenv("TSMPC_PLAN_DEBUG"))
      std::fprintf(stderr, "plan_sparse wide: split %d (chain CTAs %d, trunk CTAs %d), smem %lld doubles, tops %d\n",
                   S.split, nch_split, split_n, off, S.tops);
    S.meta_max = meta_max;
    out.smem = (size_t)off * sizeof(double);
    out.meta.clear();
    for (int c = 0; c < C; ++c) out.meta.insert(out.meta.end(), metas[c].begin(), metas[c].end());
    S.n_tsched = (int)out.tsched.size();
    out.resident_ctas = 0;
    out.max_rows = max_rows_w;
    out.max_needs = need_max;
    out.ok = true;
    return out;
  }
  if (slot_avail / base_ld < kTileS) {
    if (psi_in_smem) return plan_sparse(t, ops, NXP, NUP, NVP, max_ctas, smem_limit, sharded, rank, world, false);
    out.why = "shared memory too small for one tile slot";
    return out;
  }
  int max_rows = 0;
  for (int c = 0; c < C; ++c) max_rows = std::max(max_rows, cta_rows[c]);
  std::vector<int> ntiles_c(C);
  for (int c = 0; c < C; ++c) ntiles_c[c] = metas[c][0];
  // resident: all rows of the CTA fit; multi-tile residents need the t column
  auto plan_ld = [&](long long ld, long long& rows_out, int& res_out, bool& need_t) {
    const long long cap = slot_avail / ld;
    rows_out = 0;
    res_out = 0;
    need_t = false;
    for (int c = 0; c < C; ++c)
      if (cta_rows[c] <= cap) {
        rows_out = std::max<long long>(rows_out, cta_rows[c]);
        ++res_out;
        if (ntiles_c[c] > 1) need_t = true;
      }
  };
  long long rows_b, rows_t;
  int res_b, res_t;
  bool nt_b, nt_t;
  plan_ld(base_ld, rows_b, res_b, nt_b);
  plan_ld(t_ld, rows_t, res_t, nt_t);
  long long slot_ld, want_rows;
  if (!nt_b) {  // no multi-tile resident CTA with the narrow pitch
    slot_ld = base_ld;
    want_rows = rows_b;
  } else {      // multi-tile residents need t in the slot: use the wide pitch
    slot_ld = t_ld;
    want_rows = rows_t;
  }
  const bool any_stream = sharded || (slot_ld == base_ld ? res_b : res_t) < C;
  if (any_stream) want_rows = std::max<long long>(want_rows, kTileS);  // one streamed tile slot
  if (want_rows * slot_ld > slot_avail) want_rows = slot_avail / slot_ld;
  if (any_stream && want_rows < kTileS && want_rows * slot_ld < kTileS * base_ld) {
    out.why = "shared memory too small for one tile slot";
    return out;
  }
  S.slot_ld = (int)slot_ld;
  int resident = 0;
  for (int c = 0; c < C; ++c) {
    const bool res = !sharded && cta_rows[c] <= want_rows;
    metas[c][6] = res ? 1 : 0;
    metas[c][7] = !res ? 2 : (ntiles_c[c] <= 1 ? 0 : 1);
    if (res && ntiles_c[c] > 1 && slot_ld != t_ld) {  // cannot happen by construction
      out.why = "internal: multi-tile resident CTA without a t column";
      return out;
    }
    resident += res;
  }
  // trunk phases: the sweep's component slices (+ its schedule when it fits) use
  // work region B, or A + B when no CTA keeps t rows in region A; the own trunk
  // rows are staged in region B one slot row at a time at least
  {
    bool any_t0 = false;
    for (int c = 0; c < C; ++c) any_t0 |= metas[c][7] == 0;
    const int ncomp = nv + nx + nu;
    const int nsl = split_n ? split_n : C;  // CTAs sharing the sweep
    const long long nc_max = (ncomp + nsl - 1) / nsl;
    const long long regB = (long long)kTileS * NUP;
    const long long cap = any_t0 ? regB : (long long)S.n_work;
    const long long zx = 2LL * T * nc_max + T;  // Zs, Xs, 1/(2p) per trunk edge
    const long long sched = ((long long)out.tsched.size() + 1) / 2 + 2;
    S.sweep_in_a = any_t0 ? 0 : 1;
    S.sched_smem = zx + sched <= cap ? 1 : 0;
    if (zx > cap || slot_ld > regB) {
      out.why = "trunk too large for the work region";
      return out;
    }
  }
  S.slot_rows = (int)want_rows;
  off += want_rows * slot_ld;
  // the trunk schedule stays in shared memory for the launch when it fits
  {
    const long long sched_d = ((long long)out.tsched.size() + 1) / 2 + 1;
    const long long limit_d2 = (long long)(smem_limit / sizeof(double));
    S.sched_resident = (T > 0 && off + ints_d + sched_d <= limit_d2) ? 1 : 0;
    S.O_SCHED = (int)off;
    if (S.sched_resident) off += sched_d;
  }
  S.O_INT = (int)off;
  off += ints_d;
  // split mode: per-chain head sums (early head publication, tsmpc_sparse.cu bwd_tile)
  S.O_HSUM = (int)off;
  S.split_heads = 0;
  // [sum beta_s (NVP) | scratch: head sums 2 NUP + NXP during the backward, the
  // parent's TR row NUP + 2 NXP during fwd_finish]
  const long long hsum = NVP + std::max(2LL * NUP + NXP, (long long)NUP + 2LL * NXP);
  if (split_n && off + even(hsum) <= (long long)(smem_limit / sizeof(double)) &&
      !std::getenv("TSMPC_NO_EARLY_HEADS")) {
    S.split_heads = 1;
    off += even(hsum);
  }
  S.split = split_n ? 1 : 0;
  S.split_c0 = nch_split;
  S.split_n = split_n;
  S.TR_LD = NUP + 2 * NXP;
  {
    // local subtree sweeps: [Z | X] x all components + 1/(2p) per subtree position in
    // the (unused) slot region of the trunk CTAs; needs staged on chip (trunk_needs)
    const long long KY_LD = (long long)NVP + NXP + NUP;
    const long long sld = KY_LD + NUP + NXP;
    const bool fits = (long long)sub_max * (2LL * ncomp_all + 1) <= (long long)S.slot_rows * S.slot_ld &&
                      (long long)need_max * sld <= (long long)kTileS * NUP;
    S.split_local = (split_n && fits && !std::getenv("TSMPC_SPLIT_GLOBAL_SWEEP")) ? 1 : 0;
    // combined trunk-forward operators staged in the trunk CTAs' slot region
    S.n_tpi = (int)out.tpi.size();
    S.n_tpv = (int)out.tpv.size();
    S.O_TOPS = S.split_local ? (int)even((long long)sub_max * (2LL * ncomp_all + 1)) : 0;
    S.tops = (split_n && (long long)S.O_TOPS + S.n_tpv + (S.n_tpi + 1) / 2 + 1 <= (long long)S.slot_rows * S.slot_ld &&
              (long long)need_max * sld <= (long long)kTileS * NUP && !std::getenv("TSMPC_NO_TOPS")) ? 1 : 0;
    if (std::getenv("TSMPC_PLAN_DEBUG"))
      std::fprintf(stderr, "plan_sparse: split %d (trunk CTAs %d from %d) local %d sub_max %d need_max %d\n",
                   S.split, split_n, nch_split, S.split_local, sub_max, need_max);
  }
  if (split_n)  // the chain CTAs keep their one tile resident (else no split)
    for (int c = 0; c < nch_split; ++c)
      if (metas[c][6] == 0 || metas[c][0] != 1)
        return plan_sparse(t, ops, NXP, NUP, NVP, max_ctas, smem_limit, sharded, rank, world, psi_in_smem, false);
  S.meta_max = meta_max;
  out.smem = (size_t)off * sizeof(double);
  out.meta.clear();
  for (int c = 0; c < C; ++c) out.meta.insert(out.meta.end(), metas[c].begin(), metas[c].end());
  S.n_tsched = (int)out.tsched.size();
  out.resident_ctas = resident;
  out.max_rows = max_rows;
  out.max_needs = need_max;
  out.ok = true;
  return out;
}

}  // namespace tsmpc
