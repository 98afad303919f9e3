"""Subtree sharding of one scenario-tree solve across the GPUs of a node.

One process per GPU (``torchrun`` / ``torch.distributed``, any backend for the
host-side rendezvous).  The reference has no multi-process layer — its only
parallelism is the per-stage thread pool (``pkg/src/treesmpc/_parallel.py``,
``factor.py:107-128``); this module is the node-level equivalent:

* the leaf chains are split by the trunk node they hang from (all chains of a
  node go to one rank), contiguously, balanced by rows;
* a trunk position with only one rank's chains below is computed by that rank
  alone; the positions with several ranks' chains below ("mixed": the top of
  the tree, the root edge alone for W4k on 2/4/8 GPUs) are replicated;
* each APG iteration runs phase 1 (backward over the owned chains, the
  bottom-up sums of the owned subtrees) -> one ``ncclAllReduce`` of the sums
  that cross the cut (per cut position -- a single-rank subtree hanging from a
  mixed position -- its bottom-up sums, per mixed position its chain-head sums:
  33 rows of 344 doubles for W4k instead of every trunk node's head sums) ->
  phase 2 (the sweep above the cut, forward, prox / dual update) inside
  ``libtsmpc``.

The cross-rank sum is exact (one non-zero contributor per entry) and the sums
above the cut see the cut positions' values in node order, so a shard solve
reproduces the single-GPU iterates up to the summation order of the chain-head
sums (ulp level).  The duality gap (engine.py:458-480) is evaluated after the
loop: every rank assembles the full ergodic averages and final dual by an
all-reduce sum (each row counted by one rank; exact) and evaluates the same gap
as a single-GPU plan.  With a communicator the 2 x iters launches and
all-reduces are replayed from a CUDA graph.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .plan import DevicePlan

__all__ = ["nccl_unique_id", "ShardedSolver", "LocalShardGroup", "MultiDeviceSolver", "gather_rows",
           "merge_rows"]


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (128 bytes) from the process's libnccl."""
    buf = (ctypes.c_uint8 * 128)()
    nat.check(nat.load_library().tsmpc_nccl_unique_id(buf), "tsmpc_nccl_unique_id")
    return bytes(buf)


def _broadcast_id(rank: int, group=None) -> bytes:
    import torch.distributed as dist
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def open_peer_exchange(plan, world: int, group=None) -> bool:
    """Map every rank's exchange buffers into this rank's shard plan (CUDA IPC
    handles, all-gathered in rank order) so that each solve runs both phases and
    the cut exchange over NVLink inside one launch (include/tsmpc.h,
    tsmpc_plan_peer_open).  Collective over the ranks of ``group``; all ranks end
    up in the same mode: if any rank cannot map its peers, every rank keeps the
    two launches + ncclAllReduce per iteration.  ``world == 1`` needs no process
    group (the plan is its own peer)."""
    if world == 1:
        try:
            plan.peer_open([plan.peer_handles()])
            return True
        except Exception:
            return False
    import torch.distributed as dist
    try:
        blob = plan.peer_handles()
    except Exception:  # not a wide shard plan: the NCCL path
        blob = None
    blobs = [None] * world
    dist.all_gather_object(blobs, blob, group=group)
    ok = all(b is not None for b in blobs)
    if ok:
        try:
            plan.peer_open(blobs)
        except Exception:
            ok = False
    flags = [None] * world
    dist.all_gather_object(flags, ok, group=group)
    if not all(flags):
        if ok:
            plan.peer_close()
        return False
    return True


class ShardedSolver:
    """This rank's share of a tree solve; construct on every rank collectively.
    With ``peer`` (default unless TSMPC_NO_PEER is set) the ranks map each other's
    exchange buffers and every solve is one launch per rank with the cut exchange
    inside the kernel; otherwise two launches and an ncclAllReduce per iteration."""

    def __init__(self, model, tree, factor, scaling=None, device: int = 0, group=None,
                 peer: bool | None = None):
        import os

        import torch.distributed as dist
        if peer is None:
            peer = not os.environ.get("TSMPC_NO_PEER")
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.group = group
        nid = _broadcast_id(self.rank, group)
        self.plan = DevicePlan(model, tree, factor, scaling, device=device,
                               shard=(self.rank, self.world, nid))
        self.edges = self.plan.edges(0)
        self.trunk = self.plan.edges(1)
        self.peer_exchange = self._open_peers(group) if peer else False

    def _open_peers(self, group) -> bool:
        return open_peer_exchange(self.plan, self.world, group)

    def set_cache(self, cache, model=None):
        self.plan.set_cache(cache, model)

    def solve(self, p, iters: int, lam: float, theta=None, coef=None, warm=None,
              keep_device: bool = False, skip_gap: bool = False) -> dict:
        return self.plan.solve(p, iters, lam, warm=warm, theta=theta, coef=coef,
                               skip_gap=skip_gap, keep_device=keep_device)


class LocalShardGroup:
    """All ``world`` shards of one tree on ONE device, solved in lockstep in one
    process (``tsmpc_solve_group``): per iteration phase 1 of every shard, an
    in-place device sum of their cut exchange rows (the exchange the NCCL
    all-reduce performs across GPUs), phase 2 of every shard.  It runs exactly
    the per-rank kernels of a ``world``-GPU job, so the multi-rank split is
    checked on one GPU; the kernels of different shards never wait on each other.
    """

    def __init__(self, model, tree, factor, world: int, scaling=None, device: int = 0):
        self.world = int(world)
        self.n_edges, self.n_nodes = int(tree.n_nodes) - 1, int(tree.n_nodes)
        self.plans = [DevicePlan(model, tree, factor, scaling, device=device,
                                 shard=(r, self.world, None)) for r in range(self.world)]
        self.edges = [pl.edges(0) for pl in self.plans]

    def set_cache(self, cache, model=None):
        for pl in self.plans:
            pl.set_cache(cache, model)

    def solve(self, p, iters: int, lam: float, theta=None, coef=None,
              record_residuals: bool = False, skip_gap: bool = True) -> list[dict]:
        """Per-rank result dicts (rows of ``edges[r]`` valid in result r; with
        ``skip_gap=False`` every result carries the duality gap of the whole tree)."""
        bufs = [pl._result_buffers(iters, False, record_residuals) for pl in self.plans]
        results = (nat.Result * self.world)(*(b[1] for b in bufs))
        handles = (ctypes.c_void_p * self.world)(*(pl._h for pl in self.plans))
        flags = (nat.RECORD_RESIDUALS if record_residuals else 0) | (nat.SKIP_GAP if skip_gap else 0)
        th = np.ascontiguousarray(theta, dtype=float) if theta is not None else None
        cf = np.ascontiguousarray(coef, dtype=float) if coef is not None else None
        pv = np.ascontiguousarray(p, dtype=float)
        lib = self.plans[0]._lib
        nat.check(lib.tsmpc_solve_group(handles, self.world, nat.dptr(pv), int(iters), float(lam),
                                        nat.dptr(th), nat.dptr(cf), flags, results),
                  "tsmpc_solve_group")
        return [DevicePlan._result_dict(b[0], results[r], b[2]) for r, b in enumerate(bufs)]

    def assemble(self, outs: list[dict]) -> dict:
        """Full per-edge / per-node arrays from the per-rank results."""
        parts = [_owned(o, e) for o, e in zip(outs, self.edges)]
        return merge_rows(parts, outs[0], self.n_edges, self.n_nodes)


class MultiDeviceSolver:
    """Every shard of one tree, each on its own GPU of THIS process
    (``tsmpc_plans_create_multi`` / ``tsmpc_solve_multi``: one host thread drives
    all GPUs, the per-iteration all-reduces go out as one NCCL group).  This is
    what ``engine.solve`` runs for ``SolverConfig(devices=(...))``."""

    def __init__(self, model, tree, factor, scaling=None, devices=(0,)):
        self.devices = tuple(int(d) for d in devices)
        self.world = len(self.devices)
        self.n_edges, self.n_nodes = int(tree.n_nodes) - 1, int(tree.n_nodes)
        self.plans = DevicePlan.create_multi(model, tree, factor, scaling, self.devices)
        self.edges = [pl.edges(0) for pl in self.plans]
        self.model, self.tree, self.factor, self.scaling = model, tree, factor, scaling

    def set_cache(self, cache, model=None):
        for pl in self.plans:
            pl.set_cache(cache, model)

    def set_forecast(self, forecast, q, basis, model=None):
        for pl in self.plans:
            pl.set_forecast(forecast, q, basis, model)

    def solve(self, p, iters: int, lam: float, theta=None, coef=None, record_residuals: bool = False,
              skip_gap: bool = False) -> list[dict]:
        bufs = [pl._result_buffers(iters, False, record_residuals) for pl in self.plans]
        results = (nat.Result * self.world)(*(b[1] for b in bufs))
        handles = (ctypes.c_void_p * self.world)(*(pl._h for pl in self.plans))
        flags = (nat.RECORD_RESIDUALS if record_residuals else 0) | (nat.SKIP_GAP if skip_gap else 0)
        th = np.ascontiguousarray(theta, dtype=float) if theta is not None else None
        cf = np.ascontiguousarray(coef, dtype=float) if coef is not None else None
        pv = np.ascontiguousarray(p, dtype=float)
        nat.check(self.plans[0]._lib.tsmpc_solve_multi(handles, self.world, nat.dptr(pv), int(iters),
                                                       float(lam), nat.dptr(th), nat.dptr(cf), flags,
                                                       results), "tsmpc_solve_multi")
        return [DevicePlan._result_dict(b[0], results[r], b[2]) for r, b in enumerate(bufs)]

    def assemble(self, outs: list[dict]) -> dict:
        parts = [_owned(o, e) for o, e in zip(outs, self.edges)]
        full = merge_rows(parts, outs[0], self.n_edges, self.n_nodes)
        full.update(gap=outs[0]["gap"], iterations=outs[0]["iterations"],
                    device_ms=max(o["device_ms"] for o in outs), resid_trace=outs[0]["resid_trace"])
        return full


_EDGE_KEYS = ("u", "u_avg", "dual_sig", "dual_zeta", "dual_psi")
_NODE_KEYS = ("x", "x_avg")


def _owned(out: dict, edges: np.ndarray) -> dict:
    part = {k: out[k][edges] for k in _EDGE_KEYS}
    part.update({k: out[k][edges + 1] for k in _NODE_KEYS})
    part["edges"] = edges
    return part


def merge_rows(parts: list[dict], out: dict, n_edges: int, n_nodes: int) -> dict:
    """Full arrays from per-rank owned rows (each edge is computed by exactly
    one rank or replicated); ``out`` supplies the root row and the residual."""
    full = {k: np.zeros((n_edges, out[k].shape[1])) for k in _EDGE_KEYS}
    full.update({k: np.zeros((n_nodes, out[k].shape[1])) for k in _NODE_KEYS})
    full["x"][0] = out["x"][0]
    full["x_avg"][0] = out["x_avg"][0]
    for pt in parts:
        e = pt["edges"]
        for k in _EDGE_KEYS:
            full[k][e] = pt[k]
        for k in _NODE_KEYS:
            full[k][e + 1] = pt[k]
    full["u0"] = full["u_avg"][0]
    full["residual_inf"] = out["residual_inf"]
    return full


def gather_rows(out: dict, edges: np.ndarray, n_edges: int, n_nodes: int, group=None,
                dst: int = 0) -> dict | None:
    """Assemble full per-edge / per-node arrays on rank ``dst`` from every rank's
    owned rows (each edge is computed by exactly one rank or replicated)."""
    import torch.distributed as dist
    part = _owned(out, edges)
    parts = [None] * dist.get_world_size(group) if dist.get_rank(group) == dst else None
    dist.gather_object(part, parts, dst=dst, group=group)
    if parts is None:
        return None
    return merge_rows(parts, out, n_edges, n_nodes)
