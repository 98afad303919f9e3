"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the pinned CPU oracle.

Tolerances: solve step and prox are single-pass fp64 contractions (rel 1e-11);
APG outputs after the fixed iteration count use 10x the reference's own
ulp-perturbation deviation for that case and field (stored in the
fixture by make_golden.py), floored at 1e-11.
"""

import numpy as np
import pytest

from conftest import ALL_CASES, SMALL_CASES, has_gpu, load_case, rel_err

pytestmark = pytest.mark.gpu

if not has_gpu():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1604_01074_b200 import DualPoint, SplitPoint, engine, factor  # noqa: E402
from paper_1604_01074_b200.plan import DevicePlan  # noqa: E402
from oracle import tsmpc_oracle as O  # noqa: E402


def _plan(c, scaled=True):
    plan = DevicePlan(c.model, c.tree, c.factor, c.scaling if scaled else None)
    plan.set_cache(c.cache, c.model)
    return plan


@pytest.mark.parametrize("name", ALL_CASES)
def test_solve_step_matches_reference(name):
    c = load_case(name)
    z = c.z
    out = factor.solve_step(c.factor, c.cache, c.tree,
                            DualPoint(z["w_sig"], z["w_zeta"], z["w_psi"]), c.p)
    assert rel_err(out.x, z["s_x"]) <= 1e-11
    assert rel_err(out.u, z["s_u"]) <= 1e-11


@pytest.mark.parametrize("path", ["sparse", "sparse-nosplit", "dense"])
@pytest.mark.parametrize("name", ALL_CASES)
def test_apg_solve_matches_reference(name, path, monkeypatch):
    """Every persistent-kernel path: the structured-basis sparse kernel (default
    when A is diagonal; split mode where the plan allows it), the same kernel with
    split mode off (two grid barriers per iteration), and the dense fused-operator
    DMMA kernel (TSMPC_FORCE_DENSE)."""
    c = load_case(name)
    z = c.z
    monkeypatch.setenv("TSMPC_FORCE_DENSE", "1" if path == "dense" else "0")
    if path == "sparse-nosplit":
        monkeypatch.setenv("TSMPC_NO_SPLIT", "1")
    plan = _plan(c)
    info = plan.info()
    diag = np.count_nonzero(c.model.A - np.diag(np.diag(c.model.A))) == 0
    assert info["sparse"] == (1 if (path != "dense" and diag) else 0), info["path"]
    if path == "sparse-nosplit":
        assert info["trunk_ctas"] == 0
    th, cf = engine.theta_schedule(c.iters)
    out = plan.solve(c.p, c.iters, c.lam, theta=th, coef=cf)
    for f in ("u0", "x", "u", "x_avg", "u_avg"):
        assert rel_err(out[f], z[f"r_{f}"]) <= c.tol(f), (f, rel_err(out[f], z[f"r_{f}"]), c.tol(f))
    for k in ("sig", "zeta", "psi"):
        assert rel_err(out[f"dual_{k}"], z[f"r_dual_{k}"]) <= c.tol("dual"), k
    r_ref = float(z["r_residual_inf"])
    assert abs(out["residual_inf"] - r_ref) <= c.tol("residual_inf") * max(1.0, abs(r_ref))
    g_ref = float(z["r_gap"])
    assert abs(out["gap"] - g_ref) <= max(1e-8, c.tol("gap")) * max(1.0, abs(g_ref))


@pytest.mark.parametrize("name", ALL_CASES)
def test_prox_matches_reference(name):
    c = load_case(name)
    z = c.z
    t = SplitPoint(z["t_sig"], z["t_zeta"], z["t_psi"])
    out = engine.prox_g(t, 0.7, c.model)
    np.testing.assert_array_equal(out.psi, z["pr_psi"])
    assert rel_err(out.sig, z["pr_sig"]) <= 1e-13
    assert rel_err(out.zeta, z["pr_zeta"]) <= 1e-13
    if c.scaling is not None:
        out = engine.prox_g(t, 0.7, c.model, scaling_edges=c.scaling.expand(c.tree))
        assert rel_err(out.sig, z["prs_sig"]) <= 1e-13
        assert rel_err(out.zeta, z["prs_zeta"]) <= 1e-13
        np.testing.assert_array_equal(out.psi, z["prs_psi"])


@pytest.mark.parametrize("name", ["tank3_tree_6_N8", "small_s0", "small_s4", "small_denseA",
                                  "bcn63_CE_N24", "bcn63_SMPC1_N24"])
def test_lambda_power_iteration_matches_reference(name):
    c = load_case(name)
    lam = engine.compute_lambda(c.basis, c.factor, c.model, c.tree, scaling=c.scaling)
    assert lam == pytest.approx(c.lam, rel=1e-7)
    lam0 = engine.compute_lambda(c.basis, c.factor, c.model, c.tree, scaling=None)
    assert lam0 == pytest.approx(float(c.z["lam_plain"]), rel=1e-7)


@pytest.mark.parametrize("name", SMALL_CASES)
def test_dropin_solve_end_to_end(name):
    """Public ``solve`` with nothing precomputed: host setup + device lambda + loop."""
    c = load_case(name)
    z = c.z
    cfg = engine.SolverConfig(max_iters=c.iters, precondition=bool(z["precondition"]))
    rep = engine.solve(c.model, c.tree, c.forecast, c.p, c.q, cfg)
    assert rep.lam == pytest.approx(c.lam, rel=1e-7)
    # lambda differs at ~1e-9: allow the corresponding perturbation of the iterates
    for f in ("u0", "u_avg", "x_avg"):
        assert rel_err(getattr(rep, f), z[f"r_{f}"]) <= max(1e-6, c.tol(f)), f


def test_residual_trace_and_determinism():
    c = load_case("tank3_tree_30_N8")
    plan = _plan(c)
    th, cf = engine.theta_schedule(c.iters)
    a = plan.solve(c.p, c.iters, c.lam, theta=th, coef=cf, record_residuals=True)
    b = plan.solve(c.p, c.iters, c.lam, theta=th, coef=cf, record_residuals=True)
    for k in ("x_avg", "u_avg", "x", "u", "dual_sig", "dual_psi"):
        assert np.array_equal(a[k], b[k]), k          # bitwise run-to-run
    assert a["gap"] == b["gap"] and a["residual_inf"] == b["residual_inf"]
    tr = a["resid_trace"]
    assert tr.shape == (c.iters,) and tr[-1] == a["residual_inf"]
    fac, cache, tree, mdl = (O.factor_dict(c.factor), O.cache_dict(c.cache, c.model, c.tree),
                             O.tree_dict(c.tree), O.model_dict(c.model))
    ref = O.apg(fac, cache, tree, mdl, c.p, c.lam, c.iters, O.scaling_tuple(c.scaling), record=True)
    np.testing.assert_allclose(tr, ref["residual_trace"], rtol=1e-9, atol=1e-12)


def test_warm_start_matches_oracle():
    c = load_case("tank3_tree_6_N8")
    z = c.z
    warm = DualPoint(z["r_dual_sig"], z["r_dual_zeta"], z["r_dual_psi"])
    plan = _plan(c)
    th, cf = engine.theta_schedule(100)
    out = plan.solve(c.p, 100, c.lam, warm=warm, theta=th, coef=cf)
    fac, cache, tree, mdl = (O.factor_dict(c.factor), O.cache_dict(c.cache, c.model, c.tree),
                             O.tree_dict(c.tree), O.model_dict(c.model))
    ref = O.solve(fac, cache, tree, mdl, c.p, c.lam, 100, O.scaling_tuple(c.scaling),
                  warm=[warm.sig, warm.zeta, warm.psi])
    for f in ("u0", "u_avg", "x_avg"):
        assert rel_err(out[f], ref[f]) <= 1e-10, f
    assert abs(out["gap"] - ref["gap"]) <= 1e-8 * max(1.0, abs(ref["gap"]))


@pytest.mark.parametrize("name", ["bcn63_SMPC1_N24", "tank3_tree_30_N8"])
def test_residual_stopping_matches_fixed_iteration_solve(name):
    """SolverConfig(tol=...): the device checks residual_inf every 25 iterations and
    stops at the first check <= tol; the result equals a fixed solve of that length."""
    c = load_case(name)
    plan = _plan(c)
    n = 200
    th, cf = engine.theta_schedule(n)
    tr = plan.solve(c.p, n, c.lam, theta=th, coef=cf, record_residuals=True, skip_gap=True)["resid_trace"]
    tol = float(tr[124])
    want = next(j + 1 for j in range(n) if (j + 1) % 25 == 0 and j + 1 < n and tr[j] <= tol)
    a = plan.solve(c.p, n, c.lam, theta=th, coef=cf, tol=tol, check_every=25)
    assert a["iterations"] == want
    assert a["residual_inf"] == tr[want - 1]
    b = plan.solve(c.p, want, c.lam, theta=th[:want], coef=cf[:want])
    for k in ("x_avg", "u_avg", "x", "u", "dual_sig", "dual_psi", "u0"):
        assert np.array_equal(a[k], b[k]), k
    assert a["gap"] == b["gap"]
    never = plan.solve(c.p, n, c.lam, theta=th, coef=cf, tol=1e-300)
    assert never["iterations"] == n


@pytest.mark.parametrize("tree_name", ["SMPC1", "SMPC3", "SMPC8"])
def test_lockstep_dykstra_gap_equals_two_pass(tree_name, monkeypatch):
    """The Dykstra forms of the gap's projection -- a thread per (edge, junction
    row) in cooperative lockstep (default when that grid is co-resident), the same
    in two passes (the default for SMPC8's 178k components; a component stops once
    its state repeats), a warp per edge in lockstep, a warp per edge in two
    passes -- run the same per-element sweeps and stop at the same global sweep:
    bitwise-equal gap."""
    import bench
    W = bench.build_workload(tree_name)
    th, cf = engine.theta_schedule(120)
    gaps = []
    # (the variables accumulate: two-pass components, then warp lockstep, then warp two passes)
    for env in (None, "TSMPC_DYKSTRA_COMP2", "TSMPC_DYKSTRA_WARP", "TSMPC_DYKSTRA_TWO_PASS"):
        if env:
            monkeypatch.setenv(env, "1")
        plan = DevicePlan(W["model"], W["tree"], W["factor"], W["scaling"])
        plan.set_cache(W["caches"][0], W["model"])
        gaps.append(plan.solve(W["p"], 120, 0.05, theta=th, coef=cf, keep_device=True)["gap"])
    assert np.isfinite(gaps[0]) and gaps[0] == gaps[1] == gaps[2] == gaps[3], gaps


@pytest.mark.parametrize("tree_name", ["SMPC1", "SMPC3"])
def test_split_mode_matches_grid_barrier_mode(tree_name, monkeypatch):
    """Split mode (trunk on spare CTAs, directed signals, heads published from
    the fill, affine trunk terms, prefilled backward, combined trunk operators)
    against the two-grid-barrier plan of the same tree: same iterates up to
    summation order."""
    import bench
    W = bench.build_workload(tree_name)
    th, cf = engine.theta_schedule(200)
    outs = []
    for env in (None, "TSMPC_NO_SPLIT"):
        if env:
            monkeypatch.setenv(env, "1")
        plan = DevicePlan(W["model"], W["tree"], W["factor"], W["scaling"])
        assert plan.info()["trunk_ctas"] == (0 if env else plan.info()["trunk_ctas"])
        plan.set_cache(W["caches"][0], W["model"])
        outs.append(plan.solve(W["p"], 200, 0.05, theta=th, coef=cf, record_residuals=True))
    a, b = outs
    assert a["kernel_launches"] >= 1
    for f in ("u0", "x", "u", "x_avg", "u_avg", "dual_sig", "dual_zeta", "dual_psi"):
        assert rel_err(a[f], b[f]) <= 1e-9, (f, rel_err(a[f], b[f]))
    np.testing.assert_allclose(a["resid_trace"], b["resid_trace"], rtol=1e-8, atol=1e-9)
    assert abs(a["gap"] - b["gap"]) <= 1e-8 * max(1.0, abs(b["gap"]))


@pytest.mark.parametrize("tree_name,shard,record", [("W4k", False, False), ("W4k", False, True),
                                                    ("SMPC8", True, False)])
def test_fill_rows_through_hbm_equal_dual_row_fill(tree_name, shard, record, monkeypatch):
    """Multi-tile and sharded wide CTAs take the next backward's fill rows from FG,
    written by the previous iteration's epilogue (also across launches: per-iteration
    windows of record_residuals, the two launches of a sharded iteration); the same
    operations as the fill from both dual rows, so the bits must match TSMPC_NO_FG."""
    import bench
    from paper_1604_01074_b200.shard import nccl_unique_id
    W = bench.build_workload(tree_name)
    iters = 24
    th, cf = engine.theta_schedule(iters)
    outs = []
    for env in ("0", "1"):
        if env == "1":
            monkeypatch.setenv("TSMPC_NO_FG", "1")
        else:
            monkeypatch.delenv("TSMPC_NO_FG", raising=False)
        plan = DevicePlan(W["model"], W["tree"], W["factor"], W["scaling"],
                          shard=(0, 1, nccl_unique_id()) if shard else None)
        assert plan.info()["fill_rows_hbm"] == (0 if env == "1" else 1)
        plan.set_cache(W["caches"][0], W["model"])
        outs.append(plan.solve(W["p"], iters, 0.05, theta=th, coef=cf, record_residuals=record))
    a, b = outs
    for f in ("u0", "x", "u", "x_avg", "u_avg", "dual_sig", "dual_zeta", "dual_psi"):
        assert np.array_equal(a[f], b[f]), f
    assert a["gap"] == b["gap"]
    if record:
        assert np.array_equal(a["resid_trace"], b["resid_trace"])
