"""Subtree sharding of one scenario-tree solve across the GPUs of a node.

One process per GPU (``torchrun`` / ``torch.distributed``, any backend for the
host-side rendezvous).  The reference has no multi-process layer — its only
parallelism is the per-stage thread pool (``pkg/src/treesmpc/_parallel.py``,
``factor.py:107-128``); this module is the node-level equivalent:

* the trunk (every edge above the leaf chains) is replicated on every rank,
* the leaf chains are split by the trunk node they hang from, so every
  chain-head sum of a trunk node has exactly one owning rank,
* each APG iteration runs phase 1 (backward over the owned chains + per-node
  head sums) -> one ``ncclAllReduce`` of T x (n_v + n_x) doubles -> phase 2
  (replicated trunk sweep, forward, prox / dual update) inside ``libtsmpc``.

The cross-rank sum is exact (one non-zero contributor per entry), so a shard
solve reproduces the single-GPU iterates up to the summation order of the
chain-head sums (ulp level).  The duality gap is not evaluated by shard plans.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .plan import DevicePlan

__all__ = ["nccl_unique_id", "ShardedSolver", "gather_rows"]


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


class ShardedSolver:
    """This rank's share of a tree solve; construct on every rank collectively."""

    def __init__(self, model, tree, factor, scaling=None, device: int = 0, group=None):
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.group = group
        nid = _broadcast_id(self.rank, group)
        self.plan = DevicePlan(model, tree, factor, scaling, device=device,
                               shard=(self.rank, self.world, nid))
        self.edges = self.plan.edges(0)
        self.trunk = self.plan.edges(1)

    def set_cache(self, cache, model=None):
        self.plan.set_cache(cache, model)

    def solve(self, p, iters: int, lam: float, theta=None, coef=None, warm=None,
              keep_device: bool = False) -> dict:
        return self.plan.solve(p, iters, lam, warm=warm, theta=theta, coef=coef,
                               skip_gap=True, keep_device=keep_device)


def gather_rows(out: dict, edges: np.ndarray, n_edges: int, n_nodes: int, group=None,
                dst: int = 0) -> dict | None:
    """Assemble full per-edge / per-node arrays on rank ``dst`` from every rank's
    owned rows (each edge is computed by exactly one rank or replicated)."""
    import torch.distributed as dist
    part = {k: out[k][edges] for k in ("u", "u_avg", "dual_sig", "dual_zeta", "dual_psi")}
    part.update({k: out[k][edges + 1] for k in ("x", "x_avg")})
    part["edges"] = edges
    parts = [None] * dist.get_world_size(group) if dist.get_rank(group) == dst else None
    dist.gather_object(part, parts, dst=dst, group=group)
    if parts is None:
        return None
    full = {k: np.zeros((n_edges, out[k].shape[1])) for k in ("u", "u_avg", "dual_sig", "dual_zeta",
                                                           "dual_psi")}
    full.update({k: np.zeros((n_nodes, out[k].shape[1])) for k in ("x", "x_avg")})
    full["x"][0] = out["x"][0]
    full["x_avg"][0] = out["x_avg"][0]
    for pt in parts:
        e = pt["edges"]
        for k in ("u", "u_avg", "dual_sig", "dual_zeta", "dual_psi"):
            full[k][e] = pt[k]
        for k in ("x", "x_avg"):
            full[k][e + 1] = pt[k]
    full["u0"] = full["u_avg"][0]
    full["residual_inf"] = out["residual_inf"]
    return full
