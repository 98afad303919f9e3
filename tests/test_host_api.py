"""Host-side data layer of the drop-in API: loaders, validation, trees, synthetic
inputs and configuration objects (mirrors the reference's test_network_model.py /
test_scenario_tree.py expectations on the same behaviours)."""

import json

import numpy as np
import pytest

from paper_1604_01074_b200 import (DemandForecast, DimensionError, ParseError, SolverConfig,
                                   ValidationError, build_tree, load_network, load_tree,
                                   node_demands, scenario_paths, synth, tree_document)
from paper_1604_01074_b200.model import junction_residual, simulate_step, stage_cost
from paper_1604_01074_b200.plan import describe_tree


def _net_doc(m):
    d = {k: np.asarray(getattr(m, k)).tolist() for k in
         ("A", "B", "Gd", "E", "Ed", "u_min", "u_max", "x_min", "x_max", "x_s", "alpha1",
          "alpha2_schedule", "Wu")}
    d.update(W_alpha=m.W_alpha, Wx=m.Wx, gamma_d=m.gamma_d)
    return d


def test_network_roundtrip_and_validation():
    m = synth.three_tank_network()
    doc = _net_doc(m)
    back = load_network(json.dumps(doc))
    np.testing.assert_array_equal(back.B, m.B)
    assert back.n_x == 3 and back.n_u == 4 and back.n_e == 1 and back.n_d == 2
    with pytest.raises(ParseError):
        load_network("{not json")
    bad = dict(doc)
    del bad["Wu"]
    with pytest.raises(ParseError):
        load_network(json.dumps(bad))
    bad = dict(doc, u_min=[50.0, 0, 0, 0])
    with pytest.raises(ValidationError) as ei:
        load_network(json.dumps(bad))
    assert any("u_min > u_max" in v for v in ei.value.violations)
    bad = dict(doc, Wu=(-np.eye(4)).tolist())
    with pytest.raises(ValidationError):
        load_network(json.dumps(bad))


def test_plant_helpers():
    m = synth.three_tank_network()
    x = simulate_step(m, [250, 200, 200], [20, 50, 15, 15], [30, 20])
    np.testing.assert_allclose(x, [250 + 20 - 20, 200 + 15, 200 + 15])
    np.testing.assert_allclose(junction_residual(m, [0, 50, 10, 10], [30, 0]), [0.0])
    c = stage_cost(m, [50, 50, 50], [1, 1, 1, 1], [0, 0, 0, 0], 8)
    assert c.safety > 0 and c.smoothing == pytest.approx(0.5 + 0.3 + 0.2 + 0.2)
    with pytest.raises(DimensionError):
        simulate_step(m, [1, 2], [0, 0, 0, 0], [0, 0])


def test_tree_build_load_roundtrip():
    t = synth.uniform_tree([3, 2], N=8, n_d=2, seed=11)
    assert t.n_s == 6 and t.n_edges == 3 + 6 + 6 * 6
    back = load_tree(json.dumps(tree_document(t)))
    for k in ("stage_starts", "anc", "child_start", "child_stop"):
        np.testing.assert_array_equal(getattr(back, k), getattr(t, k))
    np.testing.assert_allclose(back.prob, t.prob)
    paths = scenario_paths(t)
    assert len(paths) == 6 and all(len(p) == 9 for p in paths)
    fc = DemandForecast(np.ones((8, 2)), k=3)
    d = node_demands(t, fc)
    np.testing.assert_allclose(d, 1.0 + t.edge_eps)
    with pytest.raises(DimensionError):
        node_demands(t, DemandForecast(np.ones((7, 2))))


def test_tree_validation_errors():
    with pytest.raises(ValidationError):
        build_tree([2], [np.zeros((2, 1))], [[1.0], [0.7, 0.7]], N=1)  # stage prob != 1
    with pytest.raises(ParseError):
        load_tree('{"N": 1, "stages": []}')
    with pytest.raises(ValidationError):
        build_tree([0], [np.zeros((1, 1))], [[1.0], [1.0]], N=1)


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
