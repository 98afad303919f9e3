"""Subtree sharding, host side, on CPU with two gloo ranks (no GPU): the NCCL id
rendezvous, the chain partition each rank's planner builds, and the row
assembly of shard results (paper_1604_01074_b200/shard.py)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1604_01074_b200 import compute_basis, factor_step, synth
from paper_1604_01074_b200.plan import describe_shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, tree_name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1604_01074_b200.shard import _broadcast_id, gather_rows
        nid = _broadcast_id(rank)
        ids = [None] * world
        dist.all_gather_object(ids, nid)
        m = synth.bcn63_network()
        b = compute_basis(m)
        f = factor_step(b, m)
        t = synth.paper_tree(*synth.PAPER_TREES[tree_name])
        d = describe_shard(m, t, f, rank, world)
        parts = [None] * world
        dist.all_gather_object(parts, d["edges"].tolist())
        # fake shard outputs: row values encode the edge id, assembled on rank 0
        E, n = t.n_edges, t.n_nodes
        trunk = np.array(sorted(set(range(E)) - set(sum(parts, []))), dtype=np.int64)
        mine = np.unique(np.concatenate([d["edges"], trunk])).astype(np.int64)
        out = {k: np.zeros((E, 3)) for k in ("u", "u_avg", "dual_sig", "dual_zeta", "dual_psi")}
        out.update({k: np.zeros((n, 3)) for k in ("x", "x_avg")})
        for k in ("u", "u_avg", "dual_sig", "dual_zeta", "dual_psi"):
            out[k][mine] = mine[:, None] + 1.0
        for k in ("x", "x_avg"):
            out[k][mine + 1] = mine[:, None] + 1.0
        out["residual_inf"] = 1.0
        full = gather_rows(out, mine, E, n)
        ok_full = None
        if rank == 0:
            ok_full = bool(np.array_equal(full["u"][:, 0], np.arange(E) + 1.0)
                           and np.array_equal(full["x"][1:, 0], np.arange(E) + 1.0))
        q.put((rank, len(set(ids)) == 1 and len(ids[0]) == 128, parts, d, ok_full))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("tree_name", ["SMPC1", "SMPC3"])
def test_two_rank_partition_and_gather(tree_name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, tree_name, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    assert all(r[1] for r in res)                         # one NCCL id, 128 bytes, on every rank
    parts = res[0][2]
    owned = [set(pt) for pt in parts]
    t = synth.paper_tree(*synth.PAPER_TREES[tree_name])
    d0, d1 = res[0][3], res[1][3]
    # every row computed by one rank, except the mixed (replicated) trunk positions
    assert owned[0] | owned[1] == set(range(t.n_edges))
    assert len(owned[0] & owned[1]) == d0["mixed_positions"] == d1["mixed_positions"] >= 1
    assert d0["owned_rows"] + d1["owned_rows"] + d0["trunk_edges"] == t.n_edges
    assert d0["owned_chains"] + d1["owned_chains"] == d0["total_chains"]
    assert d0["owned_trunk_nodes"] + d1["owned_trunk_nodes"] <= d0["trunk_edges"]
    # balanced up to one group of sibling chains (SMPC1: 3 groups of 2 chains)
    assert abs(d0["owned_rows"] - d1["owned_rows"]) <= 0.1 * (d0["owned_rows"] + d1["owned_rows"]) + 44
    assert res[0][4] is True                               # rank 0 assembled every row


def test_shard_partition_world8_heads_grouped():
    m = synth.bcn63_network()
    f = factor_step(compute_basis(m), m)
    t = synth.paper_tree(*synth.PAPER_TREES["SMPC8"])
    owner, mixed = {}, set()
    for r in range(8):
        d = describe_shard(m, t, f, r, 8)
        for e in d["edges"]:
            if int(e) in owner:
                mixed.add(int(e))
            owner[int(e)] = r
        assert d["mixed_positions"] == len(mixed) or r < 7
    assert len(owner) == t.n_edges
    for e in mixed:                                       # replicated rows are trunk edges
        pn = int(t.anc[e + 1])
        assert int(t.child_stop[e + 1] - t.child_start[e + 1]) > 1 or pn == 0
    # all chain heads hanging from one node are owned by one rank
    heads_by_node = {}
    for e in owner:
        pn = int(t.anc[e + 1])
        chain = int(t.child_stop[e + 1] - t.child_start[e + 1]) <= 1
        if chain and int(t.child_stop[pn] - t.child_start[pn]) != 1:   # e is a chain head
            heads_by_node.setdefault(pn, set()).add(owner[e])
    assert heads_by_node and all(len(v) == 1 for v in heads_by_node.values())


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_cut_exchange_w4k(world):
    """only sums that cross the cut are exchanged.  W4k [32,16,8]: the
    root edge is the only position with several ranks' chains below when world
    divides 32 (cut: the 32 stage-2 edges); otherwise a split stage-2 subtree adds
    its edge to the mixed set and its stage-3 edges to the cut."""
    m = synth.bcn63_network()
    f = factor_step(compute_basis(m), m)
    t = synth.paper_tree(*synth.PAPER_TREES["W4k"])
    ds = [describe_shard(m, t, f, r, world) for r in range(world)]
    d0 = ds[0]
    assert all(d["exchange_rows"] == d0["exchange_rows"] for d in ds)
    assert d0["exchange_rows"] == d0["mixed_positions"] + d0["cut_positions"]
    if 32 % world == 0:
        assert (d0["mixed_positions"], d0["cut_positions"]) == (1, 32)
    else:
        assert 1 < d0["mixed_positions"] <= world and d0["cut_positions"] > 32
    # vs every trunk position's head sums (T x (n_v + n_x) doubles)
    assert d0["exchange_doubles"] * (7 if 32 % world == 0 else 3) < d0["trunk_edges"] * (100 + 64)
    # the trunk rows are shared out: own positions are disjoint, mixed are replicated
    own = sum(d["own_trunk_positions"] for d in ds)
    assert own + d0["mixed_positions"] == d0["trunk_edges"]
    rows = [set(map(int, d["edges"])) for d in ds]
    assert set().union(*rows) == set(range(t.n_edges))
    assert sum(len(r) for r in rows) == t.n_edges + (world - 1) * d0["mixed_positions"]


class _FakePeerPlan:
    """Stands in for a shard DevicePlan: records the peer-exchange calls."""

    def __init__(self, rank, fail_open):
        self.rank, self.fail_open, self.calls = rank, fail_open, []

    def peer_handles(self):
        self.calls.append("handles")
        return bytes([self.rank]) * 160

    def peer_open(self, blobs):
        self.calls.append(("open", [b[0] for b in blobs]))
        if self.fail_open:
            raise RuntimeError("cannot map")

    def peer_close(self):
        self.calls.append("close")


def _peer_worker(rank, world, port, fail_rank, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1604_01074_b200.shard import ShardedSolver
        s = ShardedSolver.__new__(ShardedSolver)
        s.rank, s.world = rank, world
        s.plan = _FakePeerPlan(rank, rank == fail_rank)
        on = s._open_peers(None)
        q.put((rank, on, s.plan.calls))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank", [-1, 1])
def test_peer_exchange_agreement(fail_rank):
    """The in-kernel exchange is all-or-nothing across ranks: the blobs are
    all-gathered in rank order and every rank opens them; if any rank cannot map
    its peers, the ranks that did close theirs and all keep the NCCL path."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, fail_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for rank, on, calls in res:
        assert calls[0] == "handles" and calls[1] == ("open", [0, 1])
        assert on == (fail_rank < 0)
        assert ("close" in calls) == (fail_rank >= 0 and rank != fail_rank)
