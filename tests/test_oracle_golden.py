"""Pin the CPU oracle (oracle/tsmpc_oracle.py) to the real reference's golden vectors.

The oracle is the checker for every GPU parity test, so it must itself agree
with the reference on every fixture first (CPU-only).
"""

import numpy as np
import pytest

from conftest import ALL_CASES, load_case, rel_err
from oracle import tsmpc_oracle as O


def _inputs(c):
    return (O.factor_dict(c.factor), O.cache_dict(c.cache, c.model, c.tree), O.tree_dict(c.tree),
            O.model_dict(c.model), O.scaling_tuple(c.scaling))


@pytest.mark.parametrize("name", ALL_CASES)
def test_oracle_solve_step_matches_reference(name):
    c = load_case(name)
    fac, cache, tree, mdl, _ = _inputs(c)
    z = c.z
    x, u = O.solve_step(fac, cache["beta"], cache["uhat"], cache["evec"], tree,
                        z["w_sig"], z["w_zeta"], z["w_psi"], c.p)
    assert rel_err(x, z["s_x"]) <= 1e-13
    assert rel_err(u, z["s_u"]) <= 1e-13


@pytest.mark.parametrize("name", ALL_CASES)
def test_oracle_prox_matches_reference(name):
    c = load_case(name)
    _, _, tree, mdl, scal = _inputs(c)
    z = c.z
    s, ze, p = O.prox_g(z["t_sig"], z["t_zeta"], z["t_psi"], 0.7, mdl)
    np.testing.assert_array_equal(p, z["pr_psi"])
    assert rel_err(s, z["pr_sig"]) <= 1e-14 and rel_err(ze, z["pr_zeta"]) <= 1e-14
    if scal is not None:
        s, ze, p = O.prox_g(z["t_sig"], z["t_zeta"], z["t_psi"], 0.7, mdl,
                            O.expand_scaling(scal, tree["edge_stage"]))
        assert rel_err(s, z["prs_sig"]) <= 1e-14 and rel_err(p, z["prs_psi"]) <= 1e-14


@pytest.mark.parametrize("name", ALL_CASES)
def test_oracle_apg_matches_reference(name):
    c = load_case(name)
    fac, cache, tree, mdl, scal = _inputs(c)
    out = O.solve(fac, cache, tree, mdl, c.p, c.lam, c.iters, scal)
    z = c.z
    for f in ("u0", "x", "u", "x_avg", "u_avg"):
        assert rel_err(out[f], z[f"r_{f}"]) <= c.tol(f, 1e-12), f
    for k, b in zip(("sig", "zeta", "psi"), out["dual"]):
        assert rel_err(b, z[f"r_dual_{k}"]) <= c.tol("dual", 1e-12)
    assert abs(out["residual_inf"] - float(z["r_residual_inf"])) <= \
        c.tol("residual_inf", 1e-12) * max(1.0, abs(float(z["r_residual_inf"])))
    assert abs(out["gap"] - float(z["r_gap"])) <= 1e-9 * max(1.0, abs(float(z["r_gap"]))) \
        + c.tol("gap", 0.0) * max(1.0, abs(float(z["r_gap"])))


@pytest.mark.parametrize("name", ["tank3_tree_30_N8", "bcn63_SMPC1_N24"])
def test_oracle_threaded_chunks_are_bitwise_equal(name):
    """The thread-pool form of the solve step (the reference's SolverConfig.threads,
    used by bench.py's reference arm) gives the sequential result bit for bit, as the
    reference guarantees for its own threads (t/test_factor_solve.py:165-185)."""
    c = load_case(name)
    fac, cache, tree, mdl, scal = _inputs(c)
    a = O.apg(fac, cache, tree, mdl, c.p, c.lam, 30, scal, threads=1)
    b = O.apg(fac, cache, tree, mdl, c.p, c.lam, 30, scal, threads=4)
    for f in ("x", "u", "x_avg", "u_avg"):
        assert np.array_equal(a[f], b[f]), f
    for ya, yb in zip(a["dual"], b["dual"]):
        assert np.array_equal(ya, yb)


@pytest.mark.parametrize("name", ["tank3_tree_6_N8", "small_s0", "small_s4", "small_denseA",
                                  "bcn63_CE_N24"])
def test_oracle_power_iteration_matches_reference(name):
    c = load_case(name)
    fac, _, tree, _, scal = _inputs(c)
    lam = O.power_lambda(fac, c.z["beta0"], tree, scal)
    assert lam == pytest.approx(c.lam, rel=1e-9)
    lam0 = O.power_lambda(fac, c.z["beta0"], tree, None)
    assert lam0 == pytest.approx(float(c.z["lam_plain"]), rel=1e-9)


def test_oracle_theta_sequence():
    th = 1.0
    assert O.theta_next(1.0) == pytest.approx((np.sqrt(5.0) - 1.0) / 2.0, abs=1e-15)
    for nu in range(1, 101):
        th = O.theta_next(th)
        assert 0.0 < th <= 2.0 / (nu + 2.0) + 1e-12
