"""One-time host precompute of the package vs the reference's own outputs.

basis / factor / stage cache / preconditioner / momentum table are computed by
``paper_1604_01074_b200.precompute`` and compared with the golden vectors the
real reference produced for the same inputs (tests/golden/make_golden.py).
"""

import numpy as np
import pytest

from conftest import ALL_CASES, load_case, rel_err
from oracle import tsmpc_oracle as O
from paper_1604_01074_b200 import (build_stage_cache, compute_basis, compute_preconditioner,
                                   factor_step, node_demands, theta_schedule, theta_update)
from paper_1604_01074_b200.errors import ValidationError


@pytest.mark.parametrize("name", ALL_CASES)
def test_basis_and_factor_match_reference(name):
    c = load_case(name)
    b = compute_basis(c.model)
    z = c.z
    # same LAPACK path (pivoted QR) -> same orthonormal basis, not just the same span
    assert rel_err(b.L, z["L"]) <= 1e-12
    assert rel_err(b.Rbar, z["Rbar"]) <= 1e-12
    assert rel_err(b.Rbar_chol, z["Rbar_chol"]) <= 1e-12
    assert b.sigma == pytest.approx(float(z["sigma"]), rel=1e-12)
    f = factor_step(b, c.model)
    for k in ("Bbar", "Phi", "Psi"):
        assert rel_err(getattr(f, k), z[k]) <= 1e-12, k


@pytest.mark.parametrize("name", ALL_CASES)
def test_stage_cache_matches_reference(name):
    c = load_case(name)
    b = compute_basis(c.model)
    cache = build_stage_cache(b, c.model, c.tree, node_demands(c.tree, c.forecast),
                              k=c.forecast.k, q=c.q)
    for k in ("uhat", "evec", "beta", "demands", "pbar", "alpha_bar"):
        assert rel_err(getattr(cache, k), c.z[k]) <= 1e-12, k


@pytest.mark.parametrize("name", [n for n in ALL_CASES if n != "small_s6_plain"])
def test_preconditioner_matches_reference(name):
    c = load_case(name)
    s = compute_preconditioner(compute_basis(c.model), c.model, c.tree.N, tree=c.tree)
    for k in ("sig_stage", "zeta_stage", "psi_stage"):
        assert rel_err(getattr(s, k), c.z[k]) <= 1e-10, k


def test_theta_schedule_matches_reference_recursion():
    th, cf = theta_schedule(300)
    t, tp = 1.0, 1.0
    for nu in range(300):
        assert th[nu] == t and cf[nu] == t * (1.0 / tp - 1.0)
        tp, t = t, O.theta_next(t)
    assert theta_update(1.0) == pytest.approx((np.sqrt(5.0) - 1.0) / 2.0, abs=1e-15)
    with pytest.raises(ValidationError):
        theta_update(1.5)
