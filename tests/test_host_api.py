"""Host-side data layer of the drop-in API: model / tree containers and their
invariants, synthetic inputs, configuration objects, the device planner."""

import dataclasses

import numpy as np
import pytest

from paper_1604_01074_b200 import (DemandForecast, DimensionError, ScenarioTree, SolverConfig,
                                   ValidationError, check_model, node_demands, synth,
                                   validate_model)
from paper_1604_01074_b200.plan import describe_tree


def test_model_validation():
    m = synth.three_tank_network()
    assert validate_model(m) == []
    bad = dataclasses.replace(m, u_min=np.array([50.0, 0, 0, 0]))
    assert any("u_min <= u_max" in v for v in validate_model(bad))
    with pytest.raises(ValidationError):
        check_model(dataclasses.replace(m, Wu=-np.eye(4)))
    assert any(v.startswith("B:") for v in validate_model(dataclasses.replace(m, B=np.eye(2))))


def test_tree_from_arrays_and_demands():
    t = synth.uniform_tree([3, 2], N=8, n_d=2, seed=11)
    assert t.n_s == 6 and t.n_edges == 3 + 6 + 6 * 6
    again = ScenarioTree.from_arrays(t.N, t.stage_starts, t.anc, t.prob, t.eps)
    for k in ("stage_starts", "anc", "child_start", "child_stop", "prob", "eps"):
        np.testing.assert_array_equal(getattr(again, k), getattr(t, k))
    # children ranges: contiguous runs of the next stage, leaves empty at n_nodes
    for node in range(t.n_nodes):
        kids = np.flatnonzero(t.anc == node)
        if kids.size:
            assert (t.child_start[node], t.child_stop[node]) == (kids[0], kids[-1] + 1)
        else:
            assert t.child_start[node] == t.child_stop[node] == t.n_nodes
    fc = DemandForecast(np.ones((8, 2)), k=3)
    np.testing.assert_allclose(node_demands(t, fc), 1.0 + t.edge_eps)
    with pytest.raises(DimensionError):
        node_demands(t, DemandForecast(np.ones((7, 2))))


def test_tree_validation_errors():
    t = synth.uniform_tree([2], N=2, n_d=1, seed=1)
    with pytest.raises(ValidationError):   # stage probabilities do not sum to 1
        ScenarioTree.from_arrays(t.N, t.stage_starts, t.anc, t.prob * 1.1, t.eps)
    anc = t.anc.copy()
    anc[4] = 0                             # a stage-2 node hanging from the root
    with pytest.raises(ValidationError):
        ScenarioTree.from_arrays(t.N, t.stage_starts, anc, t.prob, t.eps)
    with pytest.raises(ValidationError):   # bad stage offsets
        ScenarioTree.from_arrays(t.N, t.stage_starts[:-1], t.anc, t.prob, t.eps)


@pytest.mark.parametrize("name,edges", [("CE", 24), ("SMPC1", 136), ("SMPC3", 2431),
                                        ("SMPC8", 10486)])
def test_paper_trees_reproduce_table1_edge_counts(name, edges):
    # primal variables / (n_x + n_u) = edge count
    t = synth.paper_tree(*synth.PAPER_TREES[name])
    assert t.n_edges == edges and t.N == 24
    assert abs(t.prob[t.stage_slice(24)].sum() - 1.0) < 1e-12


def test_bcn63_network_dimensions():
    m = synth.bcn63_network()
    assert (m.n_x, m.n_u, m.n_d, m.n_e) == (63, 114, 88, 17)
    assert np.allclose(m.A, np.eye(63))


def test_device_decomposition_host_logic():
    """The planner (C++, host-only entry point) on the paper trees."""
    t = synth.paper_tree(*synth.PAPER_TREES["SMPC8"])
    d = describe_tree(t)
    assert d["segments"] == 493 and d["trunk_edges"] == 133      # leaf chains / trunk
    assert d["rows"] + d["trunk_edges"] == t.n_edges
    assert d["max_rows_per_cta"] == 84 and d["max_tiles_per_cta"] == 1
    lvl = describe_tree(t, collapse=False)                     # level-synchronous plan
    assert lvl["levels"] == 4 and lvl["rows"] == t.n_edges
    ce = describe_tree(synth.paper_tree(*synth.PAPER_TREES["CE"]))
    assert ce["ctas"] == 1 and ce["trunk_edges"] == 0 and ce["segments"] == 1
    # a chain longer than a segment is split into a trunk part and a leaf segment
    long = synth.paper_tree(1, 1, 1, N=40)
    dl = describe_tree(long)
    assert dl["rows"] + dl["trunk_edges"] == 40 and dl["rows"] <= 32


def test_solver_config_validation():
    with pytest.raises(ValidationError):
        SolverConfig(max_iters=0)
    with pytest.raises(ValidationError):
        SolverConfig(lam=-1.0)
    with pytest.raises(ValidationError):
        SolverConfig(threads=0)


def test_reference_style_solver_config_is_accepted():
    """A SolverConfig without the device / tol / check_every extensions (the
    reference's own class, engine.py:40-57) is read with defaults."""
    from paper_1604_01074_b200 import engine

    class RefConfig:  # the reference's fields only
        max_iters, lam, precondition, threads = 5, None, True, 1
        record_residuals, warm_start = False, False

    cfg = RefConfig()
    assert getattr(cfg, "device", 0) == 0 and getattr(cfg, "tol", None) is None
    with pytest.raises(ValidationError):
        SolverConfig(tol=1.0, record_residuals=True)
    assert engine.solve.__doc__
