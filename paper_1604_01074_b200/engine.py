"""Drop-in ``engine`` module: the APG solve on the B200.

Same public surface as the reference's ``treesmpc.engine``
(``pkg/src/treesmpc/engine.py``): ``SolverConfig``, ``SolveReport``,
``DualScaling``, ``apply_H``, ``adjoint_H``, ``prox_g``, ``theta_update``,
``extrapolate``, ``compute_lambda``, ``compute_preconditioner``, ``solve`` and
``smooth_cost``.  ``solve`` does only one-time host work (basis, factor,
cache, preconditioner when not supplied) and then runs the whole fixed-iteration
loop plus the duality gap on the device through ``libtsmpc`` — there is no host
fallback.  ``apply_H`` / ``adjoint_H`` / ``extrapolate`` / ``smooth_cost`` are
small host utilities kept for API compatibility; on the solve path the device
fuses them into its kernels.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .errors import DimensionError, ValidationError
from .plan import plan_for
from .points import DualPoint, PrimalPoint, SplitPoint
from .precompute import (DualScaling, build_stage_cache, compute_basis,
                         compute_preconditioner, dual_hessian_row_sums, factor_step,
                         theta_schedule, theta_update)

__all__ = [
    "SolverConfig", "SolveReport", "DualScaling",
    "apply_H", "adjoint_H", "prox_g", "theta_update", "extrapolate",
    "compute_lambda", "compute_preconditioner", "solve", "smooth_cost",
    "dual_hessian_row_sums",
]


@dataclass
class SolverConfig:
    """Solve knobs (reference ``engine.py:40-57``).  ``threads`` is accepted for
    API compatibility; the device ignores it.  ``device``, ``tol`` and
    ``check_every`` are extensions: :func:`solve` reads them with ``getattr``, so
    the reference's own ``SolverConfig`` objects (which lack them) work too."""

    max_iters: int = 500
    lam: float | None = None
    precondition: bool = True
    threads: int = 1
    record_residuals: bool = False
    warm_start: bool = False
    device: int = 0
    # extension (the reference loop is fixed-iteration): stop as soon as the
    # residual_inf checked every `check_every` iterations on the device is <= tol
    tol: float | None = None
    check_every: int = 25
    # extension: split the tree by subtree over these GPUs of this process (one
    # NCCL all-reduce of chain-head sums per iteration; shard.MultiDeviceSolver)
    devices: tuple | None = None

    def __post_init__(self):
        if self.max_iters < 1:
            raise ValidationError("max_iters must be >= 1")
        if self.lam is not None and self.lam <= 0:
            raise ValidationError("lambda override must be positive")
        if self.threads < 1:
            raise ValidationError("thread count must be >= 1")
        if self.tol is not None and self.record_residuals:
            # the reference's traces are per iteration of the fixed-length loop
            raise ValidationError("tol (early stop) and record_residuals exclude each other")
        if self.check_every < 1:
            raise ValidationError("check_every must be >= 1")


@dataclass
class SolveReport:
    u0: np.ndarray
    x: np.ndarray
    u: np.ndarray
    x_avg: np.ndarray
    u_avg: np.ndarray
    residual_inf: float
    gap: float
    iterations: int
    wall_time_s: float
    lam: float
    preconditioned: bool
    residual_trace: np.ndarray | None = None
    gap_trace: np.ndarray | None = None
    dual: DualPoint | None = field(default=None, repr=False)
    device_ms: float | None = None

    def to_dict(self) -> dict:
        d = {"u0": self.u0.tolist(), "x": self.x.tolist(), "u": self.u.tolist(),
             "x_avg": self.x_avg.tolist(), "u_avg": self.u_avg.tolist(),
             "residual_inf": self.residual_inf, "gap": self.gap,
             "iterations": self.iterations, "wall_time_s": self.wall_time_s,
             "lambda": self.lam, "preconditioned": self.preconditioned}
        if self.residual_trace is not None:
            d["residual_trace"] = self.residual_trace.tolist()
        if self.gap_trace is not None:
            d["gap_trace"] = self.gap_trace.tolist()
        return d


# -- host utilities (API mirrors; fused into the device kernels on the solve path)

def apply_H(z: PrimalPoint) -> SplitPoint:
    """Copy map Hz = (x[1:], x[1:], u)  (reference ``engine.py:106-108``)."""
    return SplitPoint(z.x[1:].copy(), z.x[1:].copy(), z.u.copy())


def adjoint_H(y: DualPoint) -> PrimalPoint:
    """H'y = ([0; sig + zeta], psi)  (reference ``engine.py:111-115``)."""
    n_x = y.sig.shape[1]
    return PrimalPoint(np.vstack([np.zeros((1, n_x)), y.sig + y.zeta]), y.psi.copy())


def extrapolate(y: DualPoint, y_prev: DualPoint, theta: float, theta_prev: float) -> DualPoint:
    c = theta * (1.0 / theta_prev - 1.0)
    return DualPoint(y.sig + c * (y.sig - y_prev.sig), y.zeta + c * (y.zeta - y_prev.zeta),
                     y.psi + c * (y.psi - y_prev.psi))


def smooth_cost(model, tree, cache, u) -> float:
    """Probability-weighted economic + smoothing cost (reference ``engine.py:347-357``)."""
    pa = tree.parent_edge()
    u_prev = np.where((pa >= 0)[:, None], u[pa], cache.q[None, :])
    du = u - u_prev
    st = tree.edge_stage()
    prices = np.stack([model.price(cache.k + j) for j in range(tree.N)])
    econ = model.W_alpha * np.einsum("ej,ej->e", prices[st], u)
    quad = np.einsum("ej,jk,ek->e", du, model.Wu, du)
    return float(np.dot(tree.edge_prob, econ + quad))


# -- device-backed operators ------------------------------------------------------

def prox_g(t: SplitPoint, lam: float, model, scaling_edges=None, *, tree=None,
           factor=None, scaling=None) -> SplitPoint:
    """prox of g with parameter ``lam`` (reference ``engine.py:157-183``) on the device.

    With ``scaling_edges`` (the expanded per-edge arrays of the reference API) the
    rows are scaled accordingly; the device evaluates them row-wise.
    """
    if lam <= 0:
        raise ValidationError("prox parameter must be positive")
    rows = t.sig.shape[0]
    if t.sig.shape != t.zeta.shape or t.sig.shape[1] != model.n_x or t.psi.shape != (rows, model.n_u):
        raise DimensionError("prox operand blocks have inconsistent shapes")
    plan = _prox_plan(model, rows, scaling_edges)
    s, z, p = plan.prox(t, lam, scaled=scaling_edges is not None)
    return SplitPoint(s, z, p)


def _prox_plan(model, rows, scaling_edges):
    """A plan whose 'tree' is a chain of ``rows`` edges, one stage per row, so the
    per-stage scaling table of the device equals the per-row scaling given."""
    from .precompute import EliminationBasis, FactorCache  # noqa: F401
    from .tree import _finish
    n = rows + 1
    starts = np.arange(n + 1, dtype=np.int64)
    anc = np.arange(-1, n - 1, dtype=np.int64)
    tree = _finish(rows, starts, anc, np.ones(n), np.zeros((n, 1)))
    n_x, n_u = model.n_x, model.n_u
    fac = _IdentityFactor(n_x, n_u)
    scaling = None
    if scaling_edges is not None:
        s, z, p = scaling_edges
        scaling = DualScaling(np.ascontiguousarray(np.broadcast_to(s, (rows, 1))[:, 0]),
                              np.ascontiguousarray(np.broadcast_to(z, (rows, 1))[:, 0]),
                              np.ascontiguousarray(np.broadcast_to(p, (rows, n_u))))
    key = ("prox", id(model), rows, None if scaling is None else
           (scaling.sig_stage.tobytes(), scaling.zeta_stage.tobytes(), scaling.psi_stage.tobytes()))
    hit = _PROX_PLANS.get(key)
    if hit is None:
        from .plan import DevicePlan
        hit = DevicePlan(model, tree, fac, scaling, warn_dense=False)
        _PROX_PLANS.clear()
        _PROX_PLANS[key] = hit
    return hit


_PROX_PLANS: dict = {}


class _IdentityFactor:
    def __init__(self, n_x, n_u):
        self.A = np.eye(n_x)
        self.L = np.eye(n_u)[:, :1]
        self.Bbar = np.zeros((n_x, 1))
        self.Phi = np.zeros((1, n_x))
        self.Psi = np.zeros((1, n_u))
        self.n_x, self.n_u, self.n_v = n_x, n_u, 1


def _zero_cache(basis, model, tree):
    demands = np.zeros((tree.n_edges, model.n_d))
    return build_stage_cache(basis, model, tree, demands, k=0, q=np.zeros(model.n_u))


def compute_lambda(basis, factor, model, tree, scaling=None, tol: float = 1e-8,
                   max_iter: int = 600, device: int = 0) -> float:
    """Step size 0.995 / lambda_max of the scaled dual-gradient operator, by
    deterministic power iteration with every operator application on the device
    (reference ``engine.py:286-337``)."""
    if basis.sigma <= 0:
        raise ValidationError("strong convexity modulus must be positive")
    plan = plan_for(model, tree, factor, scaling, device)
    key = ("lam", id(basis), id(scaling), float(tol), int(max_iter))
    memo = getattr(plan, "_lam_memo", None)
    if memo is not None and memo[0] == key and memo[1] is basis and memo[2] is scaling:
        return memo[3]
    cache0 = _zero_cache(basis, model, tree)
    plan.dual_operator_begin(cache0.beta)
    lam_max = 0.0
    for _ in range(max_iter):
        new, _dd, _yy = plan.dual_operator_step()
        if abs(new - lam_max) <= tol * max(1.0, abs(new)):
            lam_max = new
            break
        lam_max = new
    if not np.isfinite(lam_max) or lam_max <= 0:
        raise ValidationError(f"dual Lipschitz estimate invalid: {lam_max!r}")
    plan._lam_memo = (key, basis, scaling, 0.995 / lam_max)
    return 0.995 / lam_max


# one-time setup derived inside solve() when the caller does not pass it: kept per
# (model, tree) object so that repeat drop-in calls reuse one device plan and one
# step size instead of re-deriving and re-uploading them every call
_SETUP: dict = {}


def _setup_for(model, tree, precondition: bool):
    key = (id(model), id(tree), bool(precondition))
    hit = _SETUP.get(key)
    if hit is not None and hit[0] is model and hit[1] is tree:
        return hit[2:]
    basis = compute_basis(model)
    factor = factor_step(basis, model)
    scaling = compute_preconditioner(basis, model, tree.N, tree=tree) if precondition else None
    if len(_SETUP) >= 4:
        _SETUP.pop(next(iter(_SETUP)))
    _SETUP[key] = (model, tree, basis, factor, scaling)
    return basis, factor, scaling


def solve(model, tree, forecast, p, q, config: SolverConfig | None = None, *,
          basis=None, factor=None, cache=None, scaling=None, lam=None,
          warm_dual: DualPoint | None = None) -> SolveReport:
    """Fixed-iteration accelerated dual proximal gradient solve on the B200.

    Signature and result of the reference ``engine.solve`` (``engine.py:485-601``).
    """
    config = config or SolverConfig()
    p = np.asarray(p, dtype=float)
    q = np.asarray(q, dtype=float)
    if p.shape != (model.n_x,):
        raise DimensionError(f"p: shape {p.shape}, expected ({model.n_x},)")
    if q.shape != (model.n_u,):
        raise DimensionError(f"q: shape {q.shape}, expected ({model.n_u},)")
    device = int(getattr(config, "device", 0))
    tol = getattr(config, "tol", None)
    check_every = int(getattr(config, "check_every", 25))
    if basis is None and factor is None:
        basis, factor, derived = _setup_for(model, tree, config.precondition)
        if config.precondition and scaling is None:
            scaling = derived
    else:
        basis = basis or compute_basis(model)
        factor = factor or factor_step(basis, model)
        if config.precondition and scaling is None:
            scaling = compute_preconditioner(basis, model, tree.N, tree=tree)
    if not config.precondition:
        scaling = None
    lam = lam if lam is not None else config.lam
    if lam is None:
        lam = compute_lambda(basis, factor, model, tree, scaling=scaling, device=device)

    devices = getattr(config, "devices", None)
    if devices:
        return _solve_multi(model, tree, forecast, p, q, config, basis, factor, cache, scaling,
                            float(lam), tuple(devices), warm_dual)
    plan = plan_for(model, tree, factor, scaling, device)
    if cache is None:
        # stage cache built on the device from the forecast
        if forecast.dhat.shape[0] != tree.N:
            raise DimensionError(
                f"forecast horizon {forecast.dhat.shape[0]} does not match tree horizon {tree.N}")
        plan.set_forecast(forecast, q, basis, model)
    else:
        plan.set_cache(cache, model)
    theta, coef = theta_schedule(config.max_iters)
    warm = warm_dual if (config.warm_start and warm_dual is not None) else None
    t0 = time.perf_counter()
    # record_residuals: the residual and the duality gap of every iteration
    # (engine.py:577-582), evaluated in the same device solve (one launch per iteration)
    trace_on_device = bool(config.record_residuals) and plan.info()["sparse"] == 1
    out = plan.solve(p, config.max_iters, float(lam), warm=warm, theta=theta, coef=coef,
                     record_residuals=config.record_residuals, tol=tol,
                     check_every=check_every, gap_trace=trace_on_device)
    gap_trace = out["gap_trace"]
    if config.record_residuals and not trace_on_device:
        gap_trace = _gap_trace_dense(plan, p, config, lam, warm, theta, coef)
    wall = time.perf_counter() - t0
    return SolveReport(
        u0=out["u0"], x=out["x"], u=out["u"], x_avg=out["x_avg"], u_avg=out["u_avg"],
        residual_inf=out["residual_inf"], gap=out["gap"], iterations=out["iterations"],
        wall_time_s=wall, lam=float(lam), preconditioned=scaling is not None,
        residual_trace=out["resid_trace"], gap_trace=gap_trace,
        dual=DualPoint(out["dual_sig"], out["dual_zeta"], out["dual_psi"]),
        device_ms=out["device_ms"])


_MULTI: dict = {}


def _solve_multi(model, tree, forecast, p, q, config, basis, factor, cache, scaling, lam, devices,
                 warm_dual):
    """engine.solve over several GPUs of this process (SolverConfig.devices)."""
    from .shard import MultiDeviceSolver
    if config.warm_start and warm_dual is not None:
        raise ValidationError("warm_dual is not supported with SolverConfig.devices")
    if config.tol is not None:
        raise ValidationError("tol (early stop) is not supported with SolverConfig.devices")
    key = (id(model), id(tree), id(factor), id(scaling), devices)
    hit = _MULTI.get(key)
    if hit is None or hit.model is not model or hit.tree is not tree or hit.factor is not factor \
            or hit.scaling is not scaling:
        _MULTI.clear()
        hit = MultiDeviceSolver(model, tree, factor, scaling, devices)
        _MULTI[key] = hit
    if cache is None:
        if forecast.dhat.shape[0] != tree.N:
            raise DimensionError(
                f"forecast horizon {forecast.dhat.shape[0]} does not match tree horizon {tree.N}")
        hit.set_forecast(forecast, q, basis, model)
    else:
        hit.set_cache(cache, model)
    theta, coef = theta_schedule(config.max_iters)
    t0 = time.perf_counter()
    outs = hit.solve(p, config.max_iters, lam, theta=theta, coef=coef,
                     record_residuals=config.record_residuals)
    full = hit.assemble(outs)
    wall = time.perf_counter() - t0
    return SolveReport(
        u0=full["u0"], x=full["x"], u=full["u"], x_avg=full["x_avg"], u_avg=full["u_avg"],
        residual_inf=full["residual_inf"], gap=full["gap"], iterations=full["iterations"],
        wall_time_s=wall, lam=lam, preconditioned=scaling is not None,
        residual_trace=full["resid_trace"], gap_trace=None,
        dual=DualPoint(full["dual_sig"], full["dual_zeta"], full["dual_psi"]),
        device_ms=full["device_ms"])


def _gap_trace_dense(plan, p, config, lam, warm, theta, coef):
    """Per-iteration duality gap on a dense-kernel plan (non-diagonal A), whose
    persistent kernel has no launch windows: iteration nu's gap is the gap after a
    fresh nu+1-iteration device solve (identical iterates; O(iters^2) work, only
    for this rare plan type)."""
    gaps = np.empty(config.max_iters)
    for nu in range(config.max_iters):
        r = plan.solve(p, nu + 1, float(lam), warm=warm, theta=theta[:nu + 1],
                       coef=coef[:nu + 1], keep_device=True)
        gaps[nu] = r["gap"]
    return gaps
