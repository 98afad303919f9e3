"""Closed loop (Algorithm 2, reference closed_loop.py:107-239) and the device
stage cache (elimination.py:114-158) against the real reference.

Golden trajectories come from tests/golden/make_closed_loop_golden.py (the
reference's run_closed_loop with its own step size, stored as ``lam``).  The
tolerance is 10x the reference's own ulp-perturbation deviation of each output
over the whole loop (controls feed back into the next solve), floored at 1e-9.
"""

import numpy as np
import pytest

from conftest import GOLDEN, has_gpu, load_case, rel_err
from paper_1604_01074_b200 import (DemandForecast, NetworkModel, SolverConfig, build_stage_cache,
                                   node_demands)
from paper_1604_01074_b200.closed_loop import SimulationConfig, compute_kpis, run_closed_loop
from paper_1604_01074_b200.tree import _finish

CL_CASES = ["tank3_tree6_warm", "tank3_tree6_cold", "bcn63_CE_warm"]
MODEL_KEYS = ("A", "B", "Gd", "E", "Ed", "u_min", "u_max", "x_min", "x_max", "x_s", "alpha1",
              "alpha2_schedule", "Wu")


def _load(name):
    raw = np.load(GOLDEN / f"cl_{name}.npz")
    z = {k: raw[k] for k in raw.files}
    sc = z["m_scalars"]
    model = NetworkModel(**{k: z[f"m_{k}"] for k in MODEL_KEYS}, W_alpha=float(sc[0]),
                         Wx=float(sc[1]), gamma_d=float(sc[2]))
    tree = _finish(int(z["t_N"]), z["t_stage_starts"], z["t_anc"], z["t_prob"], z["t_eps"])
    return z, model, tree


def _tol(z, f):
    return max(10.0 * float(z[f"ulp_{f}"]), 1e-9)


@pytest.mark.parametrize("name", CL_CASES)
def test_kpis_match_reference_formula(name):
    """compute_kpis on the reference's own trajectory reproduces its KPIs."""
    z, model, _ = _load(name)
    k = compute_kpis(z["r_states"][1:], z["r_controls"], model, u_prev=z["q"], k0=0)
    np.testing.assert_allclose([k.economic, k.smoothness, k.safety_shortfall, k.network_utility],
                               z["r_kpis"], rtol=1e-12, atol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CL_CASES)
def test_closed_loop_matches_reference(name):
    if not has_gpu():
        pytest.skip("no CUDA device")
    z, model, tree = _load(name)
    cfg = SimulationConfig(network=model, tree=tree, demands=z["cl_realized"],
                           forecast=z["cl_nominal"], h_s=z["cl_realized"].shape[0], x0=z["p"],
                           u_prev=z["q"], k0=0,
                           solver=SolverConfig(max_iters=int(z["cl_iters"]), lam=float(z["lam"]),
                                               warm_start=bool(z["cl_warm"]),
                                               precondition=bool(z["cl_precondition"])))
    res = run_closed_loop(cfg)
    assert rel_err(res.controls, z["r_controls"]) <= _tol(z, "controls")
    assert rel_err(res.states, z["r_states"]) <= _tol(z, "states")
    assert rel_err(res.residuals, z["r_residuals"]) <= max(_tol(z, "residuals"), 1e-8)
    assert rel_err(res.gaps, z["r_gaps"]) <= max(_tol(z, "gaps"), 1e-8)
    k = res.kpis
    np.testing.assert_allclose([k.economic, k.smoothness, k.safety_shortfall, k.network_utility],
                               z["r_kpis"], rtol=1e-8, atol=1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["bcn63_SMPC1_N24", "tank3_tree30_N24", "small_s4"])
def test_device_stage_cache_matches_host(name):
    """tsmpc_set_forecast (device) == build_stage_cache (host, reference formula)."""
    if not has_gpu():
        pytest.skip("no CUDA device")
    from paper_1604_01074_b200.plan import DevicePlan
    c = load_case(name)
    plan = DevicePlan(c.model, c.tree, c.factor, c.scaling)
    plan.set_forecast(c.forecast, c.q, c.basis, c.model)
    beta, uhat, evec = plan.get_cache()
    assert rel_err(uhat, c.cache.uhat) <= 1e-13
    assert rel_err(evec, c.cache.evec) <= 1e-13
    assert rel_err(beta, c.cache.beta) <= 1e-12
    host = build_stage_cache(c.basis, c.model, c.tree, node_demands(c.tree, c.forecast),
                             k=c.forecast.k, q=c.q)
    assert rel_err(beta, host.beta) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["bcn63_SMPC1_N24", "small_s4"])
def test_sparse_stage_cache_equals_dense(name, monkeypatch):
    """The stage-cache rows with the operators in CSR (cache_rows_sparse_kernel,
    default) give the dense kernel's bits (TSMPC_DENSE_CACHE): only fma(0, d, s)
    terms are skipped."""
    if not has_gpu():
        pytest.skip("no CUDA device")
    from paper_1604_01074_b200.plan import DevicePlan
    c = load_case(name)
    got = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("TSMPC_DENSE_CACHE", env)
        plan = DevicePlan(c.model, c.tree, c.factor, c.scaling)
        plan.set_forecast(c.forecast, c.q, c.basis, c.model)
        got.append(plan.get_cache())
    for a, b in zip(*got):
        assert np.array_equal(a, b)
