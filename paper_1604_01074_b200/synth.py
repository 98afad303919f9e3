"""Synthetic Barcelona-dimension inputs.

The Barcelona drinking-water-network matrices are not shipped with the
reference (``SPEC.md:14``), so benchmarks and parity tests use a seeded
synthetic network with the paper's dimensions (n_x=63, n_u=114, n_d=88,
n_e=17; ``PAPER.md:729-731``) and paper-shaped N=24 trees
``mu = [1, 1, b1, b1*b2, n_s, ..., n_s]`` that reproduce Table I's edge counts
(``PAPER.md:817-844``): CE 24, SMPC1 136, SMPC3 2431, SMPC8 10486 edges.
The 3-tank network and ``tree_doc`` recipe of the reference's fixture script
(``pkg/scripts/make_fixtures.py:12-65``) are restated for N=24 regenerations.
"""

from __future__ import annotations

import numpy as np

from .model import NetworkModel, validate_model
from .tree import DemandForecast, _finish

__all__ = ["bcn63_network", "three_tank_network", "paper_tree", "PAPER_TREES",
           "base_demand", "forecast_profile", "uniform_tree", "initial_state", "input_arrays"]

# name -> (b1, b2, n_s); edges = 1 + b1 + b1*b2 + 21*n_s at N = 24
PAPER_TREES = {
    "CE": (1, 1, 1),
    "SMPC1": (3, 2, 6),
    "SMPC3": (6, 5, 114),
    "SMPC8": (12, 10, 493),
    "W4k": (32, 16, 4096),
    "W16k": (32, 32, 16384),
}


def bcn63_network(seed: int = 1604, paper_weights: bool = False) -> NetworkModel:
    rng = np.random.default_rng(seed)
    n_x, n_u, n_d, n_e = 63, 114, 88, 17
    B = np.zeros((n_x, n_u))
    E = np.zeros((n_e, n_u))
    u_max = np.zeros(n_u)
    sourced = np.zeros(n_u, dtype=bool)
    f = 0
    for j in range(17):                       # source -> junction j
        E[j, f] = 1.0
        u_max[f] = rng.uniform(150, 250)
        sourced[f] = True
        f += 1
    targets = list(range(30, 63)) + [int(rng.integers(0, 63))]
    for k, t in enumerate(targets):           # junction (k mod 17) -> tank
        E[k % 17, f] = -1.0
        B[t, f] = 1.0
        u_max[f] = rng.uniform(40, 80)
        f += 1
    for t in range(30):                       # source -> tank t
        B[t, f] = 1.0
        u_max[f] = rng.uniform(40, 80)
        sourced[f] = True
        f += 1
    for _ in range(33):                       # tank a -> tank b
        a, b = rng.choice(63, size=2, replace=False)
        B[a, f] = -1.0
        B[b, f] = 1.0
        u_max[f] = rng.uniform(10, 30)
        f += 1
    assert f == n_u
    Ed = np.zeros((n_e, n_d))
    Gd = np.zeros((n_x, n_d))
    for j in range(17):
        Ed[j, j] = -1.0
    for d in range(17, n_d):
        Gd[(d - 17) % 63, d] = -1.0
    x_max = rng.uniform(200, 600, n_x)
    x_s = rng.uniform(0.2, 0.3, n_x) * x_max
    alpha1 = np.where(sourced, rng.uniform(0.5, 2.0, n_u), 0.2)
    k = np.arange(24)
    shape = 1.0 + 0.75 * np.sin(2 * np.pi * (k - 8) / 24.0)
    weight = np.where(sourced, rng.uniform(1.0, 1.2, n_u), 0.0)
    alpha2 = np.round(shape, 6)[:, None] * weight[None, :]
    Wu = np.diag(rng.uniform(0.2, 0.5, n_u))
    if paper_weights:
        W_alpha, Wu, Wx, gamma_d = 2e4, 1e5 * np.eye(n_u), 1e7, 5e7
    else:
        W_alpha, Wx, gamma_d = 1.0, 5.0, 20.0
    model = NetworkModel(A=np.eye(n_x), B=B, Gd=Gd, E=E, Ed=Ed, u_min=np.zeros(n_u),
                         u_max=u_max, x_min=np.zeros(n_x), x_max=x_max, x_s=x_s,
                         alpha1=alpha1, alpha2_schedule=alpha2, W_alpha=W_alpha, Wu=Wu,
                         Wx=Wx, gamma_d=gamma_d)
    bad = validate_model(model)
    if bad:
        raise AssertionError(bad)
    return model


def three_tank_network() -> NetworkModel:
    """The reference's shipped 3-tank network (``make_fixtures.py:12-41``)."""
    shape = [round(1.0 + 0.75 * np.sin(2 * np.pi * (k - 8) / 24.0), 6) for k in range(24)]
    return NetworkModel(
        A=np.eye(3),
        B=np.array([[1.0, 0, 0, 0], [0, 0, 1.0, 0], [0, 0, 0, 1.0]]),
        Gd=np.array([[0.0, -1.0], [0, 0], [0, 0]]),
        E=np.array([[0.0, 1.0, -1.0, -1.0]]),
        Ed=np.array([[-1.0, 0.0]]),
        u_min=np.zeros(4), u_max=np.array([40.0, 80.0, 60.0, 60.0]),
        x_min=np.zeros(3), x_max=np.array([500.0, 400.0, 400.0]),
        x_s=np.array([100.0, 80.0, 80.0]), alpha1=np.array([2.0, 1.5, 0.2, 0.2]),
        alpha2_schedule=np.array([[s * w for w in (1.0, 1.2, 0.0, 0.0)] for s in shape]),
        W_alpha=1.0, Wu=np.diag([0.5, 0.3, 0.2, 0.2]), Wx=5.0, gamma_d=20.0)


def base_demand(n_d: int = 88, seed: int = 99) -> np.ndarray:
    return np.random.default_rng(seed).uniform(3.0, 12.0, n_d)


def forecast_profile(base: np.ndarray, k: int, N: int) -> np.ndarray:
    """d_hat[k+j] = b (1 + 0.3 sin(2 pi (k + j - 7) / 24))."""
    t = np.arange(k, k + N)
    return base[None, :] * (1.0 + 0.3 * np.sin(2 * np.pi * (t - 7) / 24.0))[:, None]


def paper_tree(b1: int, b2: int, n_s: int, N: int = 24, base=None, seed: int = 0):
    """Paper-shaped tree mu = [1, 1, b1, b1 b2, n_s, ..., n_s] (ragged last split)."""
    if base is None:
        base = base_demand()
    rng = np.random.default_rng(seed)
    mu = [1, 1, b1, b1 * b2] + [n_s] * (N - 3)
    mu = mu[:N + 1]
    anc = [-1]
    starts = [0, 1]
    for j in range(1, N + 1):
        prev0, prev1 = starts[j - 1], starts[j]
        n_prev = prev1 - prev0
        if mu[j] == n_prev:
            kids = [1] * n_prev
        elif mu[j] % n_prev == 0:
            kids = [mu[j] // n_prev] * n_prev
        else:
            q, r = divmod(mu[j], n_prev)
            kids = [q + (1 if i < r else 0) for i in range(n_prev)]
        for i, c in enumerate(kids):
            anc.extend([prev0 + i] * c)
        starts.append(len(anc))
    anc = np.asarray(anc, dtype=np.int64)
    n = anc.shape[0]
    starts = np.asarray(starts, dtype=np.int64)
    # leaf probability 1/n_s, parents sum their children
    prob = np.zeros(n)
    prob[starts[N]:] = 1.0 / (starts[N + 1] - starts[N])
    for node in range(n - 1, 0, -1):
        prob[anc[node]] += prob[node]
    prob[0] = 1.0
    nkids = np.bincount(anc[1:], minlength=n)
    eps = np.zeros((n, base.shape[0]))
    for node in range(1, n):
        s = 0.1 if nkids[anc[node]] > 1 else 0.05
        eps[node] = rng.normal(0.0, s * base)
    return _finish(N, starts, anc, prob, eps)


def uniform_tree(branching, N: int, n_d: int, seed: int, eps_scales=None):
    """Reference ``make_fixtures.tree_doc`` shape (uniform probabilities), in memory."""
    rng = np.random.default_rng(seed)
    scales = np.asarray(eps_scales if eps_scales is not None else [6.0, 4.0][:n_d], dtype=float)
    factors = list(branching) + [1] * (N - len(branching))
    anc, prob, eps = [-1], [1.0], [np.zeros(n_d)]
    starts = [0, 1]
    prev = [(0, 1.0)]
    for j in range(1, N + 1):
        b = factors[j - 1]
        cur = []
        for (node, pp) in prev:
            for _ in range(b):
                s = scales if b > 1 else 0.5 * scales
                eps.append(np.round(rng.normal(0.0, s), 6))
                anc.append(node)
                prob.append(pp / b)
                cur.append((len(anc) - 1, pp / b))
        starts.append(len(anc))
        prev = cur
    return _finish(N, np.asarray(starts), np.asarray(anc), np.asarray(prob), np.vstack(eps))


def initial_state(model) -> tuple[np.ndarray, np.ndarray]:
    """A feasible (p, q): mid-range volumes and the zero-flow predecessor."""
    p = 0.5 * (np.asarray(model.x_s) + np.asarray(model.x_max))
    q = np.clip(np.zeros(model.n_u), model.u_min, model.u_max)
    return p, q


def forecast_for(tree, k: int = 0, base=None) -> DemandForecast:
    if base is None:
        base = base_demand(tree.n_d)
    return DemandForecast(forecast_profile(base, k, tree.N), k=k)


def input_arrays(model, tree, forecast, p, q) -> list:
    """Every input array a solve reads, in a fixed order (fixture digests of
    tests/golden/make_golden_large.py: regenerated inputs are checked against the
    sha256 of the arrays the reference was fed)."""
    keys = ("A", "B", "Gd", "E", "Ed", "u_min", "u_max", "x_min", "x_max", "x_s", "alpha1",
            "alpha2_schedule", "Wu")
    out = [np.asarray(getattr(model, k), dtype=np.float64) for k in keys]
    out.append(np.array([model.W_alpha, model.Wx, model.gamma_d], dtype=np.float64))
    out += [np.asarray(tree.stage_starts, dtype=np.int64), np.asarray(tree.anc, dtype=np.int64),
            np.asarray(tree.prob, dtype=np.float64), np.asarray(tree.eps, dtype=np.float64),
            np.asarray(forecast.dhat, dtype=np.float64), np.array([forecast.k], dtype=np.int64),
            np.asarray(p, dtype=np.float64), np.asarray(q, dtype=np.float64)]
    return out
