"""Generate golden vectors by running the REAL reference in this container.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports ``treesmpc`` from ``/root/reference/pkg/src`` (read-only; never copied)
and stores, per case, every input (model / tree / forecast arrays, so the
fixture is self-contained on the GPU box where /root/reference does not exist),
the reference's setup outputs (basis, factor, stage cache, scaling, lambda) and
its results: ``solve`` at a fixed iteration count, ``solve_step`` on a seeded
dual, ``prox_g`` on seeded rows and ``compute_lambda``.

Tolerance calibration: each solve case is re-run with the
reference's own solve-step outputs perturbed by relative 2e-16 noise; the
resulting deviation of every report field is stored as ``ulp_<field>`` and the
parity tests allow 10x that (plus a floor).
"""

from __future__ import annotations

import json
import pathlib
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = pathlib.Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "scripts"))
sys.path.insert(0, str(REF / "tests"))
ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import treesmpc  # noqa: E402
from treesmpc import engine as R_engine  # noqa: E402
from treesmpc import factor as R_factor  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent

MODEL_KEYS = ("A", "B", "Gd", "E", "Ed", "u_min", "u_max", "x_min", "x_max", "x_s",
              "alpha1", "alpha2_schedule", "Wu")


def ref_model(m):
    """Our synthetic NetworkModel (or a dict) -> the reference's NetworkModel."""
    kw = {k: np.asarray(getattr(m, k), dtype=float) for k in MODEL_KEYS}
    kw.update(W_alpha=float(m.W_alpha), Wx=float(m.Wx), gamma_d=float(m.gamma_d))
    return treesmpc.NetworkModel(**kw)


def ref_tree(t):
    return R_tree_build(np.asarray(t.stage_starts), np.asarray(t.anc), np.asarray(t.prob),
                        np.asarray(t.eps), int(t.N))


def R_tree_build(ss, anc, prob, eps, N):
    from treesmpc.tree import _validate_and_build
    return _validate_and_build(N, ss, anc, prob, eps)


def pack_inputs(d, model, tree, forecast, p, q):
    for k in MODEL_KEYS:
        d[f"m_{k}"] = np.asarray(getattr(model, k), dtype=float)
    d["m_scalars"] = np.array([model.W_alpha, model.Wx, model.gamma_d])
    d["t_stage_starts"] = np.asarray(tree.stage_starts)
    d["t_anc"] = np.asarray(tree.anc)
    d["t_prob"] = np.asarray(tree.prob)
    d["t_eps"] = np.asarray(tree.eps)
    d["t_N"] = np.array(tree.N)
    d["f_dhat"] = np.asarray(forecast.dhat)
    d["f_k"] = np.array(forecast.k)
    d["p"] = np.asarray(p, dtype=float)
    d["q"] = np.asarray(q, dtype=float)


class _Perturb:
    """Multiply solve-step outputs by (1 + 2e-16 * N(0,1)) noise (calibration)."""

    def __init__(self, seed=0):
        self.rng = np.random.default_rng(seed)
        self.orig = R_factor.SolveContext.solve

    def __enter__(self):
        rng, orig = self.rng, self.orig

        def solve(ctx, cache, w, p):
            z = orig(ctx, cache, w, p)
            z.x[...] *= 1.0 + 2e-16 * rng.standard_normal(z.x.shape)
            z.u[...] *= 1.0 + 2e-16 * rng.standard_normal(z.u.shape)
            return z
        R_factor.SolveContext.solve = solve
        return self

    def __exit__(self, *a):
        R_factor.SolveContext.solve = self.orig


def rel_dev(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


def make_case(name, model, tree, forecast, p, q, iters=500, precondition=True, seed=0,
              calibrate=True):
    rm = model if isinstance(model, treesmpc.NetworkModel) else ref_model(model)
    rt = tree if isinstance(tree, treesmpc.ScenarioTree) else ref_tree(tree)
    d = {}
    pack_inputs(d, rm, rt, forecast, p, q)
    basis = treesmpc.compute_basis(rm)
    factor = treesmpc.factor_step(basis, rm)
    demands = treesmpc.node_demands(rt, treesmpc.DemandForecast(forecast.dhat, k=forecast.k))
    cache = treesmpc.build_stage_cache(basis, rm, rt, demands, k=forecast.k, q=q)
    scaling = R_engine.compute_preconditioner(basis, rm, rt.N, tree=rt) if precondition else None
    lam = R_engine.compute_lambda(basis, factor, rm, rt, scaling=scaling)
    lam_plain = R_engine.compute_lambda(basis, factor, rm, rt, scaling=None)
    cache0 = R_engine._zero_cache(basis, rm, rt)
    d.update(L=basis.L, part_map=basis.part_map, Rbar=basis.Rbar, Rbar_chol=basis.Rbar_chol,
             sigma=np.array(basis.sigma), Bbar=factor.Bbar, Phi=factor.Phi, Psi=factor.Psi,
             beta=cache.beta, uhat=cache.uhat, evec=cache.evec, demands=cache.demands,
             pbar=cache.pbar, alpha_bar=cache.alpha_bar, beta0=cache0.beta,
             lam=np.array(lam), lam_plain=np.array(lam_plain),
             precondition=np.array(precondition), iters=np.array(iters))
    if scaling is not None:
        d.update(sig_stage=scaling.sig_stage, zeta_stage=scaling.zeta_stage,
                 psi_stage=scaling.psi_stage)
    cfg = R_engine.SolverConfig(max_iters=iters, precondition=precondition)
    rep = R_engine.solve(rm, rt, forecast, p, q, cfg, basis=basis, factor=factor, cache=cache,
                         scaling=scaling, lam=lam)
    for k in ("u0", "x", "u", "x_avg", "u_avg"):
        d[f"r_{k}"] = getattr(rep, k)
    d["r_residual_inf"] = np.array(rep.residual_inf)
    d["r_gap"] = np.array(rep.gap)
    d["r_dual_sig"], d["r_dual_zeta"], d["r_dual_psi"] = rep.dual.sig, rep.dual.zeta, rep.dual.psi
    if calibrate:
        with _Perturb(seed):
            rp = R_engine.solve(rm, rt, forecast, p, q, cfg, basis=basis, factor=factor,
                                cache=cache, scaling=scaling, lam=lam)
        for k in ("u0", "x", "u", "x_avg", "u_avg"):
            d[f"ulp_{k}"] = np.array(rel_dev(getattr(rp, k), getattr(rep, k)))
        d["ulp_dual"] = np.array(max(rel_dev(rp.dual.sig, rep.dual.sig),
                                     rel_dev(rp.dual.zeta, rep.dual.zeta),
                                     rel_dev(rp.dual.psi, rep.dual.psi)))
        d["ulp_residual_inf"] = np.array(abs(rp.residual_inf - rep.residual_inf)
                                         / max(1.0, abs(rep.residual_inf)))
        d["ulp_gap"] = np.array(abs(rp.gap - rep.gap) / max(1.0, abs(rep.gap)))
    # solve step on a seeded dual
    rng = np.random.default_rng(1000 + seed)
    E, n_x, n_u = rt.n_edges, rm.n_x, rm.n_u
    ws = [rng.standard_normal((E, n_x)), rng.standard_normal((E, n_x)), rng.standard_normal((E, n_u))]
    z = R_factor.solve_step(factor, cache, rt, treesmpc.DualPoint(*ws), p)
    d.update(w_sig=ws[0], w_zeta=ws[1], w_psi=ws[2], s_x=z.x, s_u=z.u)
    # prox on seeded rows, plain and scaled
    t = [rng.normal(0, 5, (E, n_x)) + rm.x_s[None, :], rng.normal(0, 5, (E, n_x)),
         rng.normal(0, 5, (E, n_u))]
    pr = R_engine.prox_g(treesmpc.SplitPoint(*t), 0.7, rm)
    d.update(t_sig=t[0], t_zeta=t[1], t_psi=t[2], pr_sig=pr.sig, pr_zeta=pr.zeta, pr_psi=pr.psi)
    if scaling is not None:
        ps = R_engine.prox_g(treesmpc.SplitPoint(*t), 0.7, rm, scaling_edges=scaling.expand(rt))
        d.update(prs_sig=ps.sig, prs_zeta=ps.zeta, prs_psi=ps.psi)
    np.savez_compressed(OUT / f"{name}.npz", **d)
    print(f"{name}: edges={rt.n_edges} lam={lam:.6g} resid={rep.residual_inf:.4g} "
          f"gap={rep.gap:.6g} ulp_u_avg={d.get('ulp_u_avg', np.nan)}")


def main():
    from make_fixtures import tree_doc  # reference fixture recipe (pkg/scripts)
    from conftest import make_instance  # reference test factory (pkg/tests)
    from paper_1604_01074_b200 import synth

    data = REF / "data"
    tt = treesmpc.load_network(data / "networks" / "three_tank.json")
    x0 = np.array(json.loads((data / "x0_three_tank.json").read_text()))
    up = np.array(json.loads((data / "uprev_three_tank.json").read_text()))
    nominal = np.array(json.loads((data / "demands" / "week_nominal.json").read_text())["demands"])
    cases = []
    for tname in ("tree_1", "tree_6", "tree_30"):
        tr = treesmpc.load_tree(data / "trees" / f"{tname}.json")
        fc = treesmpc.DemandForecast(nominal[:tr.N], k=0)
        cases.append((f"tank3_{tname}_N8", tt, tr, fc, x0, up, {}))
    tr24 = treesmpc.load_tree(json.dumps(tree_doc([6, 5], N=24, seed=13)))
    cases.append(("tank3_tree30_N24", tt, tr24, treesmpc.DemandForecast(nominal[5:29], k=5), x0, up, {}))
    for seed, kw in ((0, {}), (1, {}), (2, {"hetero": 3.0}), (3, {}), (4, {"n_e": 2}),
                     (5, {"n_e": 2, "N": 4, "branching": [2, 2]})):
        m, tr, fc, p, q = make_instance(seed, **kw)
        cases.append((f"small_s{seed}", m, tr, fc, p, q, {"iters": 300, "seed": seed}))
    m, tr, fc, p, q = make_instance(7, n_x=3, n_u=5, n_e=2)
    rng = np.random.default_rng(77)
    A = 0.95 * np.eye(3) + 0.02 * rng.standard_normal((3, 3))
    kw = {k: getattr(m, k) for k in MODEL_KEYS}
    kw.update(A=A, W_alpha=m.W_alpha, Wx=m.Wx, gamma_d=m.gamma_d)
    cases.append(("small_denseA", treesmpc.NetworkModel(**kw), tr, fc, p, q, {"iters": 300}))
    cases.append(("small_s6_plain", *make_instance(6), {"iters": 200, "precondition": False}))
    bcn = synth.bcn63_network()
    p_b, q_b = synth.initial_state(bcn)
    for tname in ("CE", "SMPC1"):
        tr = synth.paper_tree(*synth.PAPER_TREES[tname])
        fc = synth.forecast_for(tr, k=0)
        cases.append((f"bcn63_{tname}_N24", bcn, tr, fc, p_b, q_b, {}))
    only = set(sys.argv[1:])
    for (name, m, tr, fc, p, q, kw) in cases:
        if only and name not in only:
            continue
        make_case(name, m, tr, fc, p, q, **kw)


if __name__ == "__main__":
    main()
