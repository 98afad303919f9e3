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
    assert not (owned[0] & owned[1])                       # disjoint chain ownership
    t = synth.paper_tree(*synth.PAPER_TREES[tree_name])
    d0, d1 = res[0][3], res[1][3]
    assert len(owned[0]) + len(owned[1]) + d0["trunk_edges"] == t.n_edges
    assert d0["owned_chains"] + d1["owned_chains"] == d0["total_chains"]
    assert d0["owned_trunk_nodes"] + d1["owned_trunk_nodes"] <= d0["trunk_edges"]
    # balanced up to one group of sibling chains (SMPC1: 3 groups of 2 chains)
    assert abs(d0["owned_rows"] - d1["owned_rows"]) <= 0.1 * (d0["owned_rows"] + d1["owned_rows"]) + 44
    assert res[0][4] is True                               # rank 0 assembled every row


def test_shard_partition_world8_heads_grouped():
    m = synth.bcn63_network()
    f = factor_step(compute_basis(m), m)
    t = synth.paper_tree(*synth.PAPER_TREES["SMPC8"])
    owner = {}
    for r in range(8):
        d = describe_shard(m, t, f, r, 8)
        for e in d["edges"]:
            assert e not in owner
            owner[int(e)] = r
    # all chain heads hanging from one node are owned by one rank
    heads_by_node = {}
    for e in owner:
        pn = int(t.anc[e + 1])
        if int(t.child_stop[pn] - t.child_start[pn]) != 1:   # e is a chain head
            heads_by_node.setdefault(pn, set()).add(owner[e])
    assert heads_by_node and all(len(v) == 1 for v in heads_by_node.values())
