"""One-time host precomputation (per model, per tree, per forecast).

Everything here runs once on the host in float64 numpy/LAPACK and is then
uploaded to HBM by :class:`.plan.DevicePlan`; none of it is on the per-iteration
path.  The maths follows the reference so that the device solve sees the same
operators:

* junction elimination ``u = L v + uhat(d)`` with ``L`` an orthonormal basis of
  ker(E) from a pivoted QR of E' (``elimination.py:68-103``);
* the per-forecast vectors uhat, e, beta (``elimination.py:114-158``);
* factor matrices ``Bbar = B L`` and ``Lam = -Rbar^{-1}`` (``factor.py:67-76``);
* the single-branch diagonal dual preconditioner (``engine.py:206-277``).

The device kernels consume two fused operator blocks derived here (see
``DESIGN.md`` "operator fusion"): ``W_up = [Bbar; L]`` (backward sweep,
(n_x+n_u) x n_v) and ``W_down = [Psi | Phi] = -Rbar^{-1} [L' | Bbar']``
(forward sweep, n_v x (n_u+n_x)).
"""

from __future__ import annotations

import functools
import warnings
from dataclasses import dataclass

import numpy as np
import scipy.linalg

from .errors import DimensionError, ValidationError

__all__ = ["EliminationBasis", "StageCache", "FactorCache", "DualScaling",
           "compute_basis", "particular_solution", "build_stage_cache",
           "lift_controls", "factor_step", "compute_preconditioner",
           "dual_hessian_row_sums", "theta_update", "theta_schedule",
           "StructuredBasis", "structured_basis"]


@dataclass(frozen=True)
class EliminationBasis:
    L: np.ndarray          # (n_u, n_v) orthonormal, spans ker(E)
    part_map: np.ndarray   # (n_u, n_d) minimum-norm particular solution map
    Rhat: np.ndarray       # Wu L
    Rbar: np.ndarray       # L' Wu L (symmetrised)
    Rbar_chol: np.ndarray  # lower Cholesky factor of Rbar
    sigma: float           # 2 * lambda_min(Rbar)

    n_u = property(lambda self: self.L.shape[0])
    n_v = property(lambda self: self.L.shape[1])


@dataclass
class StageCache:
    k: int
    q: np.ndarray
    demands: np.ndarray   # (n_edges, n_d)
    uhat: np.ndarray      # (n_edges, n_u)
    evec: np.ndarray      # (n_edges, n_x)
    beta: np.ndarray      # (n_edges, n_v)
    alpha_bar: np.ndarray  # (N, n_v)
    pbar: np.ndarray      # (n_edges,)


@dataclass(frozen=True)
class FactorCache:
    Bbar: np.ndarray       # (n_x, n_v)
    Phi: np.ndarray        # (n_v, n_x) = -Rbar^{-1} Bbar'
    Psi: np.ndarray        # (n_v, n_u) = -Rbar^{-1} L'
    Rbar_chol: np.ndarray
    A: np.ndarray
    L: np.ndarray

    n_x = property(lambda self: self.A.shape[0])
    n_u = property(lambda self: self.L.shape[0])
    n_v = property(lambda self: self.L.shape[1])

    def apply_lambda(self, X: np.ndarray) -> np.ndarray:
        """Rows of X times ``Lam = -Rbar^{-1}`` (two triangular solves)."""
        return -scipy.linalg.cho_solve((self.Rbar_chol, True), X.T, check_finite=False).T


@dataclass(frozen=True)
class DualScaling:
    """Per-stage diagonal dual scaling (``engine.py:120-143``).

    Index j-1 scales the stage-j state copies (one scalar each for sig and
    zeta) and the controls entering stage j (per component).
    """

    sig_stage: np.ndarray   # (N,)
    zeta_stage: np.ndarray  # (N,)
    psi_stage: np.ndarray   # (N, n_u)

    @classmethod
    def identity(cls, N: int, n_u: int) -> "DualScaling":
        return cls(np.ones(N), np.ones(N), np.ones((N, n_u)))

    def expand(self, tree):
        s = tree.edge_stage()
        return (self.sig_stage[s][:, None], self.zeta_stage[s][:, None],
                self.psi_stage[s])


def compute_basis(model) -> EliminationBasis:
    E = np.asarray(model.E, dtype=float)
    n_e, n_u = E.shape
    if n_u - n_e < 1:
        raise ValidationError("junction equations leave no control freedom (n_u - n_e < 1)")
    Q, R, _ = scipy.linalg.qr(E.T, pivoting=True)
    tol = max(n_u, n_e) * np.finfo(float).eps * abs(R[0, 0])
    if int(np.sum(np.abs(np.diag(R)) > tol)) < n_e:
        raise ValidationError("E not full row rank")
    L = Q[:, n_e:].copy()
    part_map = -E.T @ scipy.linalg.cho_solve(scipy.linalg.cho_factor(E @ E.T), model.Ed)
    Rhat = model.Wu @ L
    Rbar = L.T @ Rhat
    Rbar = 0.5 * (Rbar + Rbar.T)
    try:
        chol = scipy.linalg.cholesky(Rbar, lower=True)
    except scipy.linalg.LinAlgError:
        raise ValidationError("reduced weight matrix L'WuL not positive definite") from None
    sigma = 2.0 * float(scipy.linalg.eigvalsh(Rbar)[0])
    if sigma <= 0:
        raise ValidationError(f"reduced curvature not positive (sigma={sigma:.3e})")
    for arr in (L, part_map, Rhat, Rbar, chol):
        arr.setflags(write=False)
    return EliminationBasis(L=L, part_map=part_map, Rhat=Rhat, Rbar=Rbar,
                            Rbar_chol=chol, sigma=sigma)


def particular_solution(basis, model, d) -> np.ndarray:
    d = np.asarray(d, dtype=float)
    if d.shape != (model.n_d,):
        raise DimensionError(f"d: shape {d.shape}, expected ({model.n_d},)")
    return basis.part_map @ d


def build_stage_cache(basis, model, tree, demands, k: int, q) -> StageCache:
    """uhat, e = B uhat + Gd d and the reduced linear terms beta for one forecast."""
    demands = np.asarray(demands, dtype=float)
    if demands.shape != (tree.n_edges, model.n_d):
        raise DimensionError(
            f"demands: shape {demands.shape}, expected ({tree.n_edges}, {model.n_d})")
    q = np.asarray(q, dtype=float)
    if q.shape != (model.n_u,):
        raise DimensionError(f"q: shape {q.shape}, expected ({model.n_u},)")
    uhat = demands @ basis.part_map.T
    evec = uhat @ model.B.T + demands @ model.Gd.T
    abar = np.stack([model.W_alpha * (basis.L.T @ model.price(k + j)) for j in range(tree.N)])

    p = tree.edge_prob
    pa = tree.parent_edge()
    inner = pa >= 0
    kids_p = np.zeros(tree.n_edges)
    np.add.at(kids_p, pa[inner], p[inner])
    pbar = p + kids_p
    uhat_up = np.where(inner[:, None], uhat[pa], q[None, :])
    kids_u = np.zeros_like(uhat)
    np.add.at(kids_u, pa[inner], p[inner, None] * uhat[inner])
    combo = pbar[:, None] * uhat - p[:, None] * uhat_up - kids_u
    beta = p[:, None] * abar[tree.edge_stage()] + 2.0 * (combo @ basis.Rhat)
    return StageCache(k=int(k), q=q.copy(), demands=demands, uhat=uhat, evec=evec,
                      beta=beta, alpha_bar=abar, pbar=pbar)


def lift_controls(basis, cache, v) -> np.ndarray:
    v = np.asarray(v, dtype=float)
    if v.ndim != 2 or v.shape != (cache.uhat.shape[0], basis.n_v):
        raise DimensionError(
            f"v: shape {v.shape}, expected ({cache.uhat.shape[0]}, {basis.n_v})")
    return v @ basis.L.T + cache.uhat


def factor_step(basis, model) -> FactorCache:
    Bbar = model.B @ basis.L
    chol = basis.Rbar_chol
    Phi = -scipy.linalg.cho_solve((chol, True), Bbar.T.copy())
    Psi = -scipy.linalg.cho_solve((chol, True), basis.L.T.copy())
    for arr in (Bbar, Phi, Psi):
        arr.setflags(write=False)
    return FactorCache(Bbar=Bbar, Phi=Phi, Psi=Psi, Rbar_chol=chol, A=model.A, L=basis.L)


# -- block-structured elimination basis (device fast path) ------------------------

@dataclass(frozen=True)
class StructuredBasis:
    """A second orthonormal basis ``Ls`` of ker(E) in which ``Ls' Wu Ls`` is diagonal.

    Flows couple when they share a junction row of E or an off-diagonal entry of
    Wu.  Each connected component of that graph gets its own orthonormal kernel
    basis, rotated by the eigenvectors of its reduced weight block.  Hence Ls is
    block-sparse (for a water network: identity columns for junction-free flows,
    3 x 2 blocks for a junction with three flows) and ``Rbar_s = Ls' Wu Ls =
    diag(lam)``.  ``Ls = L M`` with ``M = L' Ls`` orthogonal, so reduced
    coordinates map as ``v = M v_s`` and ``beta_s = M' beta``.  The exact
    minimiser of the solve step (``factor.py:142-170``) does not depend on the
    basis of ker(E); the device uses this one so that the factor step becomes
    sparse (``Rbar_s^{-1}`` diagonal, two sparse products per sweep).
    """

    Ls: np.ndarray    # (n_u, n_v)
    lam: np.ndarray   # (n_v,) diagonal of Ls' Wu Ls
    M: np.ndarray     # (n_v, n_v) = L' Ls (orthogonal)
    blocks: int       # connected components
    nnz: int          # structural non-zeros of Ls


def structured_basis(model, basis) -> StructuredBasis:
    E = np.asarray(model.E, dtype=float)
    Wu = np.asarray(model.Wu, dtype=float)
    n_e, n_u = E.shape
    parent = list(range(n_u))

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    def union(a, b):
        ra, rb = find(a), find(b)
        if ra != rb:
            parent[max(ra, rb)] = min(ra, rb)

    for row in E:
        nz = np.flatnonzero(row)
        for j in nz[1:]:
            union(int(nz[0]), int(j))
    ii, jj = np.nonzero(Wu)
    for a, b in zip(ii, jj):
        if a != b:
            union(int(a), int(b))
    comps: dict[int, list[int]] = {}
    for j in range(n_u):
        comps.setdefault(find(j), []).append(j)
    cols, lams = [], []
    for root in sorted(comps):
        F = comps[root]
        rows = [r for r in range(n_e) if np.any(E[r, F] != 0.0)]
        if rows:
            Ec = E[np.ix_(rows, F)]
            _, s, vt = np.linalg.svd(Ec)
            rank = int(np.sum(s > max(Ec.shape) * np.finfo(float).eps * s[0]))
            K = vt[rank:].T
        else:
            K = np.eye(len(F))
        if K.shape[1] == 0:
            continue
        Rc = K.T @ Wu[np.ix_(F, F)] @ K
        w, Q = np.linalg.eigh(0.5 * (Rc + Rc.T))
        Kc = K @ Q
        for c in range(Kc.shape[1]):
            col = np.zeros(n_u)
            col[F] = Kc[:, c]
            cols.append(col)
            lams.append(w[c])
    Ls = np.array(cols).T if cols else np.zeros((n_u, 0))
    if Ls.shape[1] != basis.n_v:
        raise ValidationError(f"structured kernel basis has {Ls.shape[1]} columns, expected {basis.n_v}")
    lam = np.array(lams)
    if not (lam > 0).all():
        raise ValidationError("reduced weight matrix not positive definite")
    M = basis.L.T @ Ls
    nnz = int(sum(len(c) * len(c) for c in comps.values()))
    return StructuredBasis(Ls=Ls, lam=lam, M=M, blocks=len(comps),
                           nnz=int(np.count_nonzero(Ls)) if nnz else 0)


# -- dual preconditioner ---------------------------------------------------------

def _branch_lift(model, basis, N):
    """Stacked reduced controls -> stacked (x_1..x_N, u_0..u_{N-1}) of one branch."""
    n_x, n_v = model.n_x, basis.n_v
    Bbar = model.B @ basis.L
    Mx = np.zeros((N * n_x, N * n_v))
    Apow = [np.eye(n_x)]
    for _ in range(N):
        Apow.append(model.A @ Apow[-1])
    for i in range(1, N + 1):
        for j in range(i):
            Mx[(i - 1) * n_x:i * n_x, j * n_v:(j + 1) * n_v] = Apow[i - 1 - j] @ Bbar
    return Mx, np.kron(np.eye(N), basis.L)


def dual_hessian_row_sums(W, K, block: int = 512) -> np.ndarray:
    """Row sums of |W K^{-1} W'| (``engine.py:227-236``)."""
    fac = scipy.linalg.cho_factor(0.5 * (K + K.T))
    G = scipy.linalg.cho_solve(fac, W.T).T
    out = np.empty(W.shape[0])
    for s in range(0, W.shape[0], block):
        e = min(s + block, W.shape[0])
        out[s:e] = np.abs(G[s:e] @ W.T).sum(axis=1)
    return out


def compute_preconditioner(basis, model, N: int, tree=None) -> DualScaling:
    n_x = model.n_x
    Mx, Mu = _branch_lift(model, basis, N)
    T = 2.0 * np.eye(N) - np.eye(N, k=1) - np.eye(N, k=-1)
    T[-1, -1] = 1.0
    d = dual_hessian_row_sums(np.vstack([Mx, Mx, Mu]), 2.0 * np.kron(T, basis.Rbar))
    m = N * n_x
    d_sig = d[:m].reshape(N, n_x)
    d_zeta = d[m:2 * m].reshape(N, n_x)
    d_psi = d[2 * m:].reshape(N, model.n_u)
    if tree is not None:
        pmin = np.array([float(tree.prob[tree.stage_slice(j)].min())
                         for j in range(1, N + 1)])
        d_sig = d_sig / pmin[:, None]
        d_zeta = d_zeta / pmin[:, None]
        d_psi = d_psi / pmin[:, None]
    s_m, z_m = d_sig.mean(axis=1), d_zeta.mean(axis=1)
    bad = any((~np.isfinite(a)).any() or (a <= 0).any() for a in (s_m, z_m, d_psi))
    if bad:
        warnings.warn("dual Hessian diagonal not positive; preconditioner "
                      "falls back to identity scaling")
        return DualScaling.identity(N, model.n_u)
    return DualScaling(1.0 / np.sqrt(s_m), 1.0 / np.sqrt(z_m), 1.0 / np.sqrt(d_psi))


# -- momentum schedule -------------------------------------------------------------

def theta_update(theta: float) -> float:
    """``0.5 (sqrt(th^4 + 4 th^2) - th^2)`` (``engine.py:188-192``)."""
    if not 0.0 < theta <= 1.0:
        raise ValidationError(f"theta must lie in (0, 1], got {theta!r}")
    return 0.5 * (np.sqrt(theta ** 4 + 4.0 * theta ** 2) - theta ** 2)


@functools.lru_cache(maxsize=16)
def theta_schedule(iters: int):
    """Per-iteration (theta_nu, extrapolation coefficient) tables, host fp64.

    The momentum sequence is data-independent, so the device reads it from a
    table instead of recomputing it.  ``coef[nu] = theta_nu
    (1/theta_{nu-1} - 1)`` with theta_{-1} = theta_0 = 1, as in the reference
    loop (``engine.py:527,538,585``).
    """
    theta = np.empty(iters)
    coef = np.empty(iters)
    th, th_prev = 1.0, 1.0
    for nu in range(iters):
        theta[nu] = th
        coef[nu] = th * (1.0 / th_prev - 1.0)
        th_prev, th = th, theta_update(th)
    theta.setflags(write=False)  # cached: shared by every solve with this iteration count
    coef.setflags(write=False)
    return theta, coef
