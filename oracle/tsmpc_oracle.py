"""CPU oracle for the APG hot path — TEST INFRASTRUCTURE ONLY.

A plain numpy/scipy restatement of the reference ``treesmpc`` algorithm for
the path this repository accelerates (the reference is pure Python; see
SURVEY.md §8).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline leg may import this module, and only as the checker / CPU
baseline — the product (``paper_1604_01074_b200``) never calls it.

Parity pinning: every function here is checked against golden vectors produced
by the real reference (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src`` in the build container and stores
``tests/golden/*.npz``); see ``tests/test_oracle_golden.py``.

Each function cites the reference lines it restates (paths relative to
``/root/reference/pkg/src/treesmpc``).
"""

from __future__ import annotations

import numpy as np
import scipy.linalg

CHUNKS = 8  # factor.py:35 — fixed node chunks per stage (order of the reduceat sums)


def _chunks(n, k=CHUNKS):
    k = max(1, min(k, n))
    size = -(-n // k)
    return [(i, min(i + size, n)) for i in range(0, n, size)]


def _run(pool, fn, tasks):
    """Run one stage's chunk tasks: in order, or on the worker pool with a barrier at
    the end (the reference's ``WorkerPool.run``, ``_parallel.py``; chunks of a stage
    write disjoint rows, so the result does not depend on the thread count)."""
    if pool is None:
        for t in tasks:
            fn(*t)
    else:
        for f in [pool.submit(fn, *t) for t in tasks]:
            f.result()


def solve_step(fac, beta, uhat, evec, tree, w_sig, w_zeta, w_psi, p, pool=None):
    """Backward + forward stage sweep (factor.py:142-185).

    ``fac`` provides A, Bbar, L, Rbar_chol.  Returns (x (n_nodes, n_x), u (E, n_u)).
    ``pool`` (a ``concurrent.futures`` executor) runs each stage's chunks in
    parallel, as ``SolveContext(threads > 1)`` does (factor.py:176-185).
    """
    A, Bbar, L, chol = fac["A"], fac["Bbar"], fac["L"], fac["Rbar_chol"]
    A_T, Bbar_T, L_T = A.T.copy(), Bbar.T.copy(), L.T.copy()   # factor.py:100-102
    n_nodes, E = tree["n_nodes"], tree["n_nodes"] - 1
    ss, anc, cs, ce = tree["stage_starts"], tree["anc"], tree["child_start"], tree["child_stop"]
    N = len(ss) - 2
    n_x, n_v, n_u = A.shape[0], L.shape[1], L.shape[0]
    inv2p = 1.0 / (2.0 * tree["prob"][1:])
    pa_edge = anc[1:] - 1
    r_node = np.zeros((n_nodes, n_v))
    q_node = np.zeros((n_nodes, n_x))
    delta = np.empty((E, n_v))
    v = np.empty((E, n_v))
    x = np.empty((n_nodes, n_x))
    u = np.empty((E, n_u))

    def backward_chunk(pa_, pb_):                           # factor.py:142-156
        ea, eb = int(cs[pa_]) - 1, int(ce[pb_ - 1]) - 1
        rows, nodes = slice(ea, eb), slice(ea + 1, eb + 1)
        xiq = w_sig[rows] + w_zeta[rows]                   # factor.py:147-148
        xiq += q_node[nodes]
        g = beta[rows] + r_node[nodes]                     # factor.py:149-151
        g += xiq @ Bbar
        g += w_psi[rows] @ L
        lam_g = -scipy.linalg.cho_solve((chol, True), g.T, check_finite=False).T
        delta[rows] = lam_g * inv2p[rows, None]            # factor.py:153
        offs = (cs[pa_:pb_] - (ea + 1)).astype(np.intp)
        r_node[pa_:pb_] = np.add.reduceat(g, offs, axis=0)        # factor.py:155
        q_node[pa_:pb_] = np.add.reduceat(xiq, offs, axis=0) @ A  # factor.py:156

    def forward_chunk(j, ea, eb):                           # factor.py:158-170
        rows = slice(ea, eb)
        nodes = slice(ea + 1, eb + 1)
        if j == 0:
            v[rows] = delta[rows]
        else:
            v[rows] = delta[rows] + v[pa_edge[rows]]
        u[rows] = v[rows] @ L_T + uhat[rows]
        xs = x[anc[nodes]] @ A_T
        xs += v[rows] @ Bbar_T
        xs += evec[rows]
        x[nodes] = xs

    for j in range(N - 1, -1, -1):                         # factor.py:110-119, 179-180
        ps, pe = int(ss[j]), int(ss[j + 1])
        _run(pool, backward_chunk, [(ps + a, ps + b) for a, b in _chunks(pe - ps)])
    x[0] = p                                               # factor.py:181
    for j in range(N):                                     # factor.py:121-126, 182-184
        es, ee = int(ss[j + 1]) - 1, int(ss[j + 2]) - 1
        _run(pool, forward_chunk, [(j, es + a, es + b) for a, b in _chunks(ee - es)])
    return x, u


def prox_g(t_sig, t_zeta, t_psi, lam, mdl, scal=None):
    """engine.py:146-183; ``scal`` = (sig (E,1), zeta (E,1), psi (E,n_u)) or None."""
    if scal is None:
        s_s = z_s = np.ones((t_sig.shape[0], 1))
        p_s = np.ones((1, t_psi.shape[1]))
    else:
        s_s, z_s, p_s = scal

    def shrink(t, proj, weight):
        gap = proj - t
        dist = np.linalg.norm(gap, axis=1)
        wt = np.broadcast_to(np.asarray(weight, dtype=float), dist.shape)
        f = np.ones_like(dist)
        out = dist > wt
        f[out] = wt[out] / dist[out]
        return t + f[:, None] * gap

    sig = shrink(t_sig, np.maximum(t_sig, s_s * mdl["x_s"][None, :]), lam * mdl["Wx"] / s_s[:, 0])
    zeta = shrink(t_zeta, np.clip(t_zeta, z_s * mdl["x_min"][None, :], z_s * mdl["x_max"][None, :]),
                  lam * mdl["gamma_d"] / z_s[:, 0])
    psi = np.clip(t_psi, p_s * mdl["u_min"][None, :], p_s * mdl["u_max"][None, :])
    return sig, zeta, psi


def theta_next(theta):
    """engine.py:188-192."""
    return 0.5 * (np.sqrt(theta ** 4 + 4.0 * theta ** 2) - theta ** 2)


def expand_scaling(scaling, edge_stage):
    """engine.py:138-143."""
    if scaling is None:
        return None
    s, z, p = scaling
    return s[edge_stage][:, None], z[edge_stage][:, None], p[edge_stage]


def apg(fac, cache, tree, mdl, p, lam, iters, scaling=None, warm=None, record=False, threads=1):
    """Fixed-iteration APG loop (engine.py:519-600), without the final gap.

    Returns a dict with u0, x, u, x_avg, u_avg, residual_inf, dual (scaled), and
    residual_trace when ``record``.  ``threads`` > 1 runs the solve step's stage
    chunks on a thread pool (``SolverConfig.threads``, engine.py:47, 536).
    """
    if threads > 1:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=threads) as pool:
            return _apg(fac, cache, tree, mdl, p, lam, iters, scaling, warm, record, pool)
    return _apg(fac, cache, tree, mdl, p, lam, iters, scaling, warm, record, None)


def _apg(fac, cache, tree, mdl, p, lam, iters, scaling, warm, record, pool):
    E = tree["n_nodes"] - 1
    n_x, n_u = fac["A"].shape[0], fac["L"].shape[0]
    edges = expand_scaling(scaling, tree["edge_stage"])
    if warm is None:
        y = [np.zeros((E, n_x)), np.zeros((E, n_x)), np.zeros((E, n_u))]
    else:
        y = [b.copy() for b in warm]
    y_prev = [b.copy() for b in y]
    theta, theta_prev = 1.0, 1.0
    x_avg = np.zeros((tree["n_nodes"], n_x))
    u_avg = np.zeros((E, n_u))
    trace = np.empty(iters) if record else None
    resid = np.inf
    x = u = None
    for nu in range(iters):
        c = theta * (1.0 / theta_prev - 1.0)                      # engine.py:198
        w = [a + c * (a - b) for a, b in zip(y, y_prev)]
        w_orig = w if edges is None else [w[k] * edges[k] for k in range(3)]
        x, u = solve_step(fac, cache["beta"], cache["uhat"], cache["evec"], tree, *w_orig, p, pool=pool)
        Hz = [x[1:].copy(), x[1:].copy(), u.copy()]              # engine.py:106-108
        Hz_s = Hz if edges is None else [Hz[k] * edges[k] for k in range(3)]
        t_arg = [w[k] / lam + Hz_s[k] for k in range(3)]          # engine.py:552-554
        t = prox_g(*t_arg, 1.0 / lam, mdl, edges)                 # engine.py:555
        y_next = [w[k] + lam * (Hz_s[k] - t[k]) for k in range(3)]
        x_avg *= (1.0 - theta)                                    # engine.py:562-565
        x_avg += theta * x
        u_avg *= (1.0 - theta)
        u_avg += theta * u
        if edges is not None:                                     # engine.py:567-575
            resid = max(np.max(np.abs(Hz[0] - t[0] / edges[0])),
                        np.max(np.abs(Hz[1] - t[1] / edges[1])),
                        np.max(np.abs(Hz[2] - t[2] / edges[2])))
        else:
            resid = max(np.max(np.abs(Hz[k] - t[k])) for k in range(3))
        if record:
            trace[nu] = resid
        y_prev, y = y, y_next
        theta_prev, theta = theta, theta_next(theta)
    return {"u0": u_avg[0].copy(), "x": x.copy(), "u": u.copy(), "x_avg": x_avg,
            "u_avg": u_avg, "residual_inf": float(resid), "dual": y, "residual_trace": trace}


# -- duality gap (engine.py:347-480) -------------------------------------------------

def smooth_cost(mdl, tree, cache, u):
    pa = tree["anc"][1:] - 1
    u_prev = np.where((pa >= 0)[:, None], u[pa], cache["q"][None, :])
    du = u - u_prev
    econ = mdl["W_alpha"] * np.einsum("ej,ej->e", cache["prices"][tree["edge_stage"]], u)
    smooth = np.einsum("ej,jk,ek->e", du, mdl["Wu"], du)
    return float(np.dot(tree["prob"][1:], econ + smooth))


def soft_cost(mdl, xn):
    below = np.maximum(mdl["x_s"][None, :] - xn, 0.0)
    outside = xn - np.clip(xn, mdl["x_min"], mdl["x_max"])
    return float(mdl["Wx"] * np.linalg.norm(below, axis=1).sum()
                 + mdl["gamma_d"] * np.linalg.norm(outside, axis=1).sum())


def project_junction_box(mdl, demands, u):
    lo, hi = mdl["u_min"][None, :], mdl["u_max"][None, :]
    E, Ed = mdl["E"], mdl["Ed"]
    if E.shape[0] == 1:                                           # engine.py:383-405
        a = E[0]
        b = -(demands @ Ed.T)[:, 0]
        mlo = np.full(u.shape[0], -1.0)
        mhi = np.full(u.shape[0], 1.0)
        bal = lambda m: np.clip(u - m[:, None] * a[None, :], lo, hi) @ a  # noqa: E731
        for _ in range(60):
            need = bal(mlo) < b
            if not need.any() and not (bal(mhi) > b).any():
                break
            mlo[need] *= 2.0
            high = bal(mhi) > b
            mhi[high] *= 2.0
        for _ in range(80):
            mid = 0.5 * (mlo + mhi)
            th = bal(mid) > b
            mlo = np.where(th, mid, mlo)
            mhi = np.where(th, mhi, mid)
        return np.clip(u - (0.5 * (mlo + mhi))[:, None] * a[None, :], lo, hi)
    pinv = E.T @ np.linalg.inv(E @ E.T)                            # engine.py:407-419
    tgt = -(demands @ Ed.T)
    xi = u.copy()
    inc = np.zeros_like(u)
    for _ in range(200):
        ya = xi - (xi @ E.T - tgt) @ pinv.T
        xn = np.clip(ya + inc, lo, hi)
        inc = ya + inc - xn
        if np.max(np.abs(xn - xi)) < 1e-13:
            xi = xn
            break
        xi = xn
    return xi - (xi @ E.T - tgt) @ pinv.T


def duality_gap(fac, cache, tree, mdl, p, x_avg, u_avg, y_unscaled):
    d = cache["demands"]
    u_f = project_junction_box(mdl, d, u_avg)
    x_f = np.empty((tree["n_nodes"], mdl["A"].shape[0]))
    x_f[0] = p
    ss, anc = tree["stage_starts"], tree["anc"]
    for j in range(len(ss) - 2):                                   # engine.py:422-432
        nodes = slice(int(ss[j + 1]), int(ss[j + 2]))
        rows = slice(nodes.start - 1, nodes.stop - 1)
        x_f[nodes] = x_f[anc[nodes]] @ mdl["A"].T + u_f[rows] @ mdl["B"].T + d[rows] @ mdl["Gd"].T
    primal = smooth_cost(mdl, tree, cache, u_f) + soft_cost(mdl, x_f[1:])
    sig = np.minimum(y_unscaled[0], 0.0)                           # engine.py:435-445
    nrm = np.linalg.norm(sig, axis=1)
    over = nrm > mdl["Wx"]
    sig[over] *= (mdl["Wx"] / nrm[over])[:, None]
    zeta = y_unscaled[1].copy()
    nrm = np.linalg.norm(zeta, axis=1)
    over = nrm > mdl["gamma_d"]
    zeta[over] *= (mdl["gamma_d"] / nrm[over])[:, None]
    psi = y_unscaled[2].copy()
    xh, uh = solve_step(fac, cache["beta"], cache["uhat"], cache["evec"], tree, sig, zeta, psi, p)
    pairing = float((xh[1:] * sig).sum() + (xh[1:] * zeta).sum() + (uh * psi).sum())
    conj = float((sig * mdl["x_s"][None, :]).sum())                # engine.py:448-455
    conj += float(np.where(zeta > 0, zeta * mdl["x_max"][None, :], zeta * mdl["x_min"][None, :]).sum())
    conj += float(np.where(psi > 0, psi * mdl["u_max"][None, :], psi * mdl["u_min"][None, :]).sum())
    return primal - (pairing + smooth_cost(mdl, tree, cache, uh) - conj)


def solve(fac, cache, tree, mdl, p, lam, iters, scaling=None, warm=None, record=False):
    """engine.solve with precomputed setup: APG loop + final duality gap."""
    out = apg(fac, cache, tree, mdl, p, lam, iters, scaling, warm, record)
    edges = expand_scaling(scaling, tree["edge_stage"])
    y = out["dual"]
    y_un = y if edges is None else [y[k] * edges[k] for k in range(3)]
    out["gap"] = duality_gap(fac, cache, tree, mdl, p, out["x_avg"], out["u_avg"], y_un)
    return out


def power_lambda(fac, beta0, tree, scaling=None, tol=1e-8, max_iter=600):
    """compute_lambda's power iteration (engine.py:299-337) given the zero cache's beta."""
    E = tree["n_nodes"] - 1
    n_x, n_u = fac["A"].shape[0], fac["L"].shape[0]
    zeros_u, zeros_x = np.zeros((E, n_u)), np.zeros((E, n_x))
    edges = expand_scaling(scaling, tree["edge_stage"])
    p0 = np.zeros(n_x)
    x0, u0 = solve_step(fac, beta0, zeros_u, zeros_x, tree, zeros_x, zeros_x, zeros_u, p0)
    z0 = [x0[1:], x0[1:], u0]
    y = [np.ones((E, n_x)), np.ones((E, n_x)), np.ones((E, n_u))]
    dot = lambda a, b: float((a[0] * b[0]).sum() + (a[1] * b[1]).sum() + (a[2] * b[2]).sum())  # noqa
    lam_max = 0.0
    for _ in range(max_iter):
        nrm = np.sqrt(dot(y, y))
        y = [b / nrm for b in y]
        w = y if edges is None else [y[k] * edges[k] for k in range(3)]
        x, u = solve_step(fac, beta0, zeros_u, zeros_x, tree, *w, p0)
        d = [z0[0] - x[1:], z0[1] - x[1:], z0[2] - u]
        if edges is not None:
            d = [d[k] * edges[k] for k in range(3)]
        new = dot(y, d)
        if abs(new - lam_max) <= tol * max(1.0, abs(new)):
            lam_max = new
            break
        lam_max = new
        y = d
    return 0.995 / lam_max


# -- adapters from package / reference objects ---------------------------------------

def tree_dict(tree):
    st = np.empty(tree.n_edges, dtype=np.int64)
    ss = tree.stage_starts
    for j in range(tree.N):
        st[ss[j + 1] - 1:ss[j + 2] - 1] = j
    return {"n_nodes": int(tree.n_nodes), "stage_starts": np.asarray(ss),
            "anc": np.asarray(tree.anc), "child_start": np.asarray(tree.child_start),
            "child_stop": np.asarray(tree.child_stop), "prob": np.asarray(tree.prob),
            "edge_stage": st}


def model_dict(model):
    keys = ("A", "B", "Gd", "E", "Ed", "u_min", "u_max", "x_min", "x_max", "x_s", "Wu")
    d = {k: np.asarray(getattr(model, k), dtype=float) for k in keys}
    d.update(Wx=float(model.Wx), gamma_d=float(model.gamma_d), W_alpha=float(model.W_alpha))
    return d


def factor_dict(factor):
    return {"A": np.asarray(factor.A), "Bbar": np.asarray(factor.Bbar),
            "L": np.asarray(factor.L), "Rbar_chol": np.asarray(factor.Rbar_chol)}


def cache_dict(cache, model, tree):
    prices = np.stack([model.price(cache.k + j) for j in range(tree.N)])
    return {"beta": np.asarray(cache.beta), "uhat": np.asarray(cache.uhat),
            "evec": np.asarray(cache.evec), "q": np.asarray(cache.q),
            "demands": np.asarray(cache.demands), "prices": prices}


def scaling_tuple(scaling):
    if scaling is None:
        return None
    return (np.asarray(scaling.sig_stage), np.asarray(scaling.zeta_stage),
            np.asarray(scaling.psi_stage))
