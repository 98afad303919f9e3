"""Structured kernel basis of the sparse device path (CPU only).

The device's sparse persistent kernel evaluates the reference's solve step
(factor.py:142-170) in a second orthonormal basis Ls of ker(E) in which the
reduced weight Ls' Wu Ls is diagonal (precompute.structured_basis).  These tests
pin (a) the algebraic properties the kernel relies on, (b) that the reference's
APG iterates are unchanged by the basis change (oracle run in Ls against the
reference's golden vectors, within the calibrated tolerance), and (c) the host
planner of the kernel (chain tiles, residency, shared-memory budget).
"""

import numpy as np
import pytest

from conftest import ALL_CASES, load_case, rel_err
from oracle import tsmpc_oracle as O
from paper_1604_01074_b200 import compute_basis, factor_step, synth
from paper_1604_01074_b200.plan import describe_sparse
from paper_1604_01074_b200.precompute import structured_basis


def _check(model, L):
    class B:
        pass
    b = B()
    b.L, b.n_v = L, L.shape[1]
    sb = structured_basis(model, b)
    n_v = L.shape[1]
    Ls, E, Wu = sb.Ls, np.asarray(model.E), np.asarray(model.Wu)
    assert Ls.shape == L.shape
    np.testing.assert_allclose(Ls.T @ Ls, np.eye(n_v), atol=1e-13)
    np.testing.assert_allclose(E @ Ls, 0.0, atol=1e-13)
    R = Ls.T @ Wu @ Ls
    np.testing.assert_allclose(R, np.diag(sb.lam), atol=1e-12 * max(1.0, np.abs(R).max()))
    np.testing.assert_allclose(sb.M.T @ sb.M, np.eye(n_v), atol=1e-13)
    np.testing.assert_allclose(L @ sb.M, Ls, atol=1e-13)
    assert (sb.lam > 0).all()
    return sb


def test_bcn63_basis_is_block_sparse():
    m = synth.bcn63_network()
    sb = _check(m, compute_basis(m).L)
    # 63 junction-free flows (one column each) + 17 junctions with 3 flows / 2 columns
    assert sb.blocks == 63 + 17
    assert sb.nnz == 63 + 17 * 3 * 2
    assert np.count_nonzero(sb.Ls) == sb.nnz


def test_three_tank_basis():
    m = synth.three_tank_network()
    sb = _check(m, compute_basis(m).L)
    assert sb.blocks == 2 and sb.nnz == 1 + 3 * 2


@pytest.mark.parametrize("name", ["small_s0", "small_s4", "small_denseA"])
def test_dense_wu_gives_one_rotation_block(name):
    c = load_case(name)
    sb = _check(c.model, c.basis.L)
    assert sb.blocks == 1   # dense Wu couples every flow


@pytest.mark.parametrize("name", ALL_CASES)
def test_basis_change_keeps_reference_iterates(name):
    """Reference algorithm run in the structured basis reproduces the reference's own
    golden APG outputs within the calibrated tolerance (10x its ulp sensitivity)."""
    c = load_case(name)
    sb = _check(c.model, c.basis.L)
    fac = O.factor_dict(c.factor)
    fac.update(L=sb.Ls, Bbar=np.asarray(c.model.B) @ sb.Ls, Rbar_chol=np.diag(np.sqrt(sb.lam)))
    cache = O.cache_dict(c.cache, c.model, c.tree)
    cache["beta"] = cache["beta"] @ sb.M
    out = O.solve(fac, cache, O.tree_dict(c.tree), O.model_dict(c.model), c.p, c.lam, c.iters,
                  O.scaling_tuple(c.scaling))
    for f in ("u0", "x", "u", "x_avg", "u_avg"):
        assert rel_err(out[f], c.z[f"r_{f}"]) <= c.tol(f, 1e-12), f


def test_sparse_planner_paper_trees():
    m = synth.bcn63_network()
    b = compute_basis(m)
    f = factor_step(b, m)
    got = {}
    for name in ("CE", "SMPC1", "SMPC3", "SMPC8"):
        t = synth.paper_tree(*synth.PAPER_TREES[name])
        d = describe_sparse(m, t, f)
        assert d["smem_bytes"] <= 232448
        assert d["chains"] + d["trunk_edges"] <= t.n_edges
        got[name] = d
    assert got["CE"]["ctas"] == 1 and got["CE"]["trunk_edges"] == 0
    # SMPC3 (configs[1]): one scenario chain per CTA, everything SMEM-resident;
    # split mode: the trunk (37 edges) on spare CTAs
    assert got["SMPC3"]["chains"] == 114 and got["SMPC3"]["trunk_edges"] == 37
    assert got["SMPC3"]["trunk_ctas"] == 34
    assert got["SMPC3"]["resident_ctas"] == got["SMPC3"]["ctas"] == 114 + 34
    assert got["SMPC1"]["trunk_ctas"] == 8 and got["SMPC1"]["ctas"] == 6 + 8
    assert got["SMPC3"]["max_rows"] == 21
    # SMPC8: 3-4 chains per CTA -> wide mode (a CTA's chains as one tile, rows in HBM),
    # split: the fewest chain CTAs keeping 4 chains (84 rows) per CTA, the trunk on the rest
    assert got["SMPC8"]["chains"] == 493 and got["SMPC8"]["resident_ctas"] == 0
    assert got["SMPC8"]["wide"] == 1 and got["SMPC8"]["max_rows"] == 84
    assert got["SMPC8"]["trunk_ctas"] == 148 - 124 and got["SMPC8"]["tiles"] == 124
    assert got["CE"]["trunk_ctas"] == 0 and got["SMPC3"]["wide"] == 0


def test_sparse_planner_long_chains():
    """Chains longer than a slot tile (24 rows) run in wide mode (up to 96 rows per
    chain: any horizon N <= 96 for the paper's tree shapes); longer ones are refused
    (the dense kernel takes those plans)."""
    m = synth.three_tank_network()
    b = compute_basis(m)
    f = factor_step(b, m)
    t = synth.uniform_tree([2], N=30, n_d=2, seed=3)   # two chains of 30 edges > slot tile
    d = describe_sparse(m, t, f)
    assert d["wide"] == 1 and d["max_rows"] == 30
    t = synth.uniform_tree([2], N=100, n_d=2, seed=3)  # chains of 100 edges > wide tile
    from paper_1604_01074_b200.errors import ValidationError
    with pytest.raises(ValidationError):
        describe_sparse(m, t, f)


def test_sparse_planner_wide_trees():
    """W4k keeps its whole per-CTA meta in shared memory (7 tiles per CTA); W16k
    (345,121 edges, 28 tiles and 2,331 rows per CTA) only fits with the per-tile meta
    windows, and both run wide with fill rows through HBM (multi-tile CTAs)."""
    m = synth.bcn63_network()
    b = compute_basis(m)
    f = factor_step(b, m)
    for name, tiles_per_cta in (("W4k", 7), ("W16k", 28)):
        t = synth.paper_tree(*synth.PAPER_TREES[name])
        d = describe_sparse(m, t, f)
        assert d["wide"] == 1 and d["ctas"] == 148 and d["smem_bytes"] <= 232448, (name, d)
        assert d["chains"] == synth.PAPER_TREES[name][2] and d["tile_rows"] == 84
        assert d["tiles"] >= 148 * (tiles_per_cta - 1), (name, d)
        assert d["max_rows"] == 21 * -(-d["chains"] // 148), (name, d)
