"""Drop-in ``factor`` module: factor step (host, one-time) and the device solve step.

``factor_step`` / ``FactorCache`` are the one-time host precomputation
(reference ``pkg/src/treesmpc/factor.py:38-76``).  ``SolveContext.solve`` and
``solve_step`` (reference ``factor.py:79-217``) evaluate the exact inner
minimiser with one backward and one forward sweep of the persistent device
kernel (``csrc/tsmpc_apg.cu``, STEP mode).
"""

from __future__ import annotations

import numpy as np

from .errors import DimensionError
from .plan import DevicePlan
from .points import DualPoint, PrimalPoint
from .precompute import FactorCache, factor_step

__all__ = ["FactorCache", "factor_step", "solve_step", "SolveContext"]


class _StepModel:
    """Placeholder model for a solve-step-only plan (bounds/costs unused by STEP)."""

    gap_inputs = False

    def __init__(self, factor):
        n_x, n_u = factor.n_x, factor.n_u
        self.B = np.zeros((n_x, n_u))
        self.Gd = np.zeros((n_x, 1))
        self.Wu = np.eye(n_u)
        self.E = np.eye(1, n_u)
        self.Ed = np.zeros((1, 1))
        self.u_min, self.u_max = -np.ones(n_u), np.ones(n_u)
        self.x_min, self.x_max, self.x_s = -np.ones(n_x), np.ones(n_x), np.zeros(n_x)
        self.W_alpha, self.Wx, self.gamma_d = 1.0, 1.0, 1.0
        self.n_x, self.n_u = n_x, n_u

    def price(self, k):
        return np.zeros(self.n_u)


def _check_dual_shapes(tree, factor, w):
    """Every block of the dual bundle has one row per edge (DimensionError otherwise)."""
    widths = {"sig": factor.n_x, "zeta": factor.n_x, "psi": factor.n_u}
    for block, width in widths.items():
        got = np.shape(getattr(w, block))
        if got != (tree.n_edges, width):
            raise DimensionError(f"dual block {block}: shape {got}, expected ({tree.n_edges}, {width})")


class SolveContext:
    """Device workspace bound to one (factor, tree) pair (reference ``factor.py:79-138``).

    ``solve`` returns a PrimalPoint whose arrays are owned by the context and
    overwritten by the next call (the reference returns workspace views).
    ``threads`` is accepted for compatibility and ignored.
    """

    def __init__(self, factor, tree, threads: int = 1, device: int = 0):
        self.factor, self.tree = factor, tree
        self.threads = max(1, int(threads))
        self._plan = _step_plan(factor, tree, device)
        self.x = np.zeros((tree.n_nodes, factor.n_x))
        self.u = np.zeros((tree.n_edges, factor.n_u))
        # the device decomposition both sweeps run over (segments of only-child
        # chains grouped into levels, packed into CTA tiles; tsmpc_capi.cu decompose)
        info = self._plan.info()
        sweep = {k: info[k] for k in ("levels", "segments", "tiles", "ctas", "collapsed", "trunk_edges")}
        sweep["kernel"] = "tsmpc::apg_persistent_kernel (STEP mode)"
        self.backward_plan = dict(sweep, order="stages N-1 .. 0")
        self.forward_plan = dict(sweep, order="stages 0 .. N-1")

    def close(self):
        self._plan = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def solve(self, cache, w: DualPoint, p) -> PrimalPoint:
        _check_dual_shapes(self.tree, self.factor, w)
        self._plan.set_cache(cache)
        z = self._plan.solve_step(w, np.asarray(p, dtype=float))
        self.x[...] = z.x
        self.u[...] = z.u
        return PrimalPoint(self.x, self.u)


_STEP_PLANS: dict = {}


def _step_plan(factor, tree, device: int) -> DevicePlan:
    """One solve-step plan per (factor, tree, device), reused across calls."""
    key = (id(factor), id(tree), device)
    hit = _STEP_PLANS.get(key)
    if hit is not None and hit.factor is factor and hit.tree is tree:
        return hit
    if len(_STEP_PLANS) >= 4:
        _STEP_PLANS.pop(next(iter(_STEP_PLANS)))
    plan = DevicePlan(_StepModel(factor), tree, factor, None, device, warn_dense=False)
    _STEP_PLANS[key] = plan
    return plan


def solve_step(factor, cache, tree, w: DualPoint, p, q=None, threads: int = 1) -> PrimalPoint:
    """Exact minimiser of <z, H'w> + f(z) over the tree, fresh arrays (``factor.py:198-217``)."""
    _check_dual_shapes(tree, factor, w)
    p = np.asarray(p, dtype=float)
    checks = ((cache.beta.shape[0] == tree.n_edges, "the stage cache belongs to another tree"),
              (p.shape == (factor.n_x,), f"initial state of shape {p.shape}, expected ({factor.n_x},)"),
              (q is None or np.array_equal(np.asarray(q, dtype=float), cache.q),
               "q is not the control the stage cache was built with"))
    for ok, msg in checks:
        if not ok:
            raise DimensionError(msg)
    with SolveContext(factor, tree, threads=threads) as ctx:
        z = ctx.solve(cache, w, p)
        return PrimalPoint(z.x.copy(), z.u.copy())
