"""GPU: the sharded solve machinery (phase 1 -> ncclAllReduce -> phase 2 per
iteration, streamed tiles) on one GPU with a one-rank NCCL communicator, and
the real multi-rank split (world 2..8) through tsmpc_solve_group: every shard's
kernels on one device, their head sums exchanged by an in-place device sum
between the phases, results assembled from each rank's owned rows.  The
partition logic is also covered on CPU by tests/test_shard_cpu.py (gloo)."""

import numpy as np
import pytest

from conftest import has_gpu, load_case, rel_err

pytestmark = pytest.mark.gpu

if not has_gpu():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1604_01074_b200 import engine  # noqa: E402
from paper_1604_01074_b200.errors import ValidationError  # noqa: E402
from paper_1604_01074_b200.plan import DevicePlan  # noqa: E402
from paper_1604_01074_b200.shard import LocalShardGroup, nccl_unique_id  # noqa: E402


@pytest.mark.parametrize("name", ["bcn63_SMPC1_N24", "tank3_tree30_N24", "tank3_tree_30_N8"])
def test_shard_world1_matches_reference(name):
    c = load_case(name)
    z = c.z
    plan = DevicePlan(c.model, c.tree, c.factor, c.scaling, shard=(0, 1, nccl_unique_id()))
    info = plan.info()
    assert info["sharded"] == 1 and info["world"] == 1 and info["sparse"] == 1
    assert np.array_equal(plan.edges(0), np.arange(c.tree.n_edges))
    plan.set_cache(c.cache, c.model)
    th, cf = engine.theta_schedule(c.iters)
    assert plan.solve(c.p, c.iters, c.lam, theta=th, coef=cf, skip_gap=True)["kernel_launches"] == 2 * c.iters
    out = plan.solve(c.p, c.iters, c.lam, theta=th, coef=cf)
    for f in ("u0", "x", "u", "x_avg", "u_avg"):
        assert rel_err(out[f], z[f"r_{f}"]) <= c.tol(f), (f, rel_err(out[f], z[f"r_{f}"]))
    for k in ("sig", "zeta", "psi"):
        assert rel_err(out[f"dual_{k}"], z[f"r_dual_{k}"]) <= c.tol("dual"), k
    r_ref = float(z["r_residual_inf"])
    assert abs(out["residual_inf"] - r_ref) <= c.tol("residual_inf") * max(1.0, abs(r_ref))
    # duality gap of the shard solve (assembled state, engine.py:458-480)
    g_ref = float(z["r_gap"])
    assert abs(out["gap"] - g_ref) <= c.tol("gap") * max(1.0, abs(g_ref)), (out["gap"], g_ref)


def test_shard_graph_replay_equals_direct_launches(monkeypatch):
    """The CUDA-graph replay of the 2 x iters launches + all-reduces gives the same
    bits as issuing them one by one (TSMPC_NO_GRAPH), twice in a row."""
    c = load_case("bcn63_SMPC1_N24")
    th, cf = engine.theta_schedule(c.iters)
    res = []
    for env in ("0", "1", "0"):
        if env == "1":
            monkeypatch.setenv("TSMPC_NO_GRAPH", "1")
        else:
            monkeypatch.delenv("TSMPC_NO_GRAPH", raising=False)
        plan = DevicePlan(c.model, c.tree, c.factor, c.scaling, shard=(0, 1, nccl_unique_id()))
        plan.set_cache(c.cache, c.model)
        res.append(plan.solve(c.p, c.iters, c.lam, theta=th, coef=cf))
        res.append(plan.solve(c.p, c.iters, c.lam, theta=th, coef=cf))
    for r in res[1:]:
        for f in ("u0", "x_avg", "u_avg", "dual_psi"):
            assert np.array_equal(r[f], res[0][f]), f
        assert r["gap"] == res[0]["gap"]


def test_shard_world1_matches_single_gpu_plan():
    c = load_case("bcn63_SMPC1_N24")
    th, cf = engine.theta_schedule(c.iters)
    single = DevicePlan(c.model, c.tree, c.factor, c.scaling)
    single.set_cache(c.cache, c.model)
    a = single.solve(c.p, c.iters, c.lam, theta=th, coef=cf, skip_gap=True)
    shard = DevicePlan(c.model, c.tree, c.factor, c.scaling, shard=(0, 1, nccl_unique_id()))
    shard.set_cache(c.cache, c.model)
    b = shard.solve(c.p, c.iters, c.lam, theta=th, coef=cf, skip_gap=True)
    for f in ("u0", "x_avg", "u_avg", "x", "u"):
        assert rel_err(b[f], a[f]) <= 10 * c.tol(f), f


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("name", ["bcn63_SMPC1_N24", "tank3_tree30_N24"])
def test_shard_group_matches_reference(name, world):
    c = load_case(name)
    z = c.z
    grp = LocalShardGroup(c.model, c.tree, c.factor, world, c.scaling)
    owned = np.concatenate(grp.edges)
    assert np.array_equal(np.unique(owned), np.arange(c.tree.n_edges))
    grp.set_cache(c.cache, c.model)
    th, cf = engine.theta_schedule(c.iters)
    outs = grp.solve(c.p, c.iters, c.lam, theta=th, coef=cf, skip_gap=False)
    assert all(o["kernel_launches"] >= 2 * c.iters for o in outs)
    g_ref = float(z["r_gap"])
    for o in outs:  # every rank evaluates the gap of the whole tree
        assert abs(o["gap"] - g_ref) <= c.tol("gap") * max(1.0, abs(g_ref)), (o["gap"], g_ref)
    assert len({o["residual_inf"] for o in outs}) == 1  # max over the group
    full = grp.assemble(outs)
    for f in ("u0", "x", "u", "x_avg", "u_avg"):
        assert rel_err(full[f], z[f"r_{f}"]) <= c.tol(f), (f, rel_err(full[f], z[f"r_{f}"]))
    for k in ("sig", "zeta", "psi"):
        assert rel_err(full[f"dual_{k}"], z[f"r_dual_{k}"]) <= c.tol("dual"), k
    r_ref = float(z["r_residual_inf"])
    assert abs(full["residual_inf"] - r_ref) <= c.tol("residual_inf") * max(1.0, abs(r_ref))


@pytest.mark.parametrize("tree_name,world", [("SMPC3", 2), ("SMPC3", 8), ("SMPC8", 3), ("SMPC8", 4), ("W4k", 8)])
def test_shard_group_matches_single_plan_paper_trees(tree_name, world):
    """Full-size paper trees: the w-way split reproduces the single-GPU plan's
    iterates to within the summation order of the chain-head sums."""
    import bench
    W = bench.build_workload(tree_name)
    iters = 60
    th, cf = engine.theta_schedule(iters)
    single = DevicePlan(W["model"], W["tree"], W["factor"], W["scaling"])
    single.set_cache(W["caches"][0], W["model"])
    lam = 0.05
    a = single.solve(W["p"], iters, lam, theta=th, coef=cf, record_residuals=True)
    grp = LocalShardGroup(W["model"], W["tree"], W["factor"], world, W["scaling"])
    sizes = [len(e) for e in grp.edges]
    assert min(sizes) > 0
    grp.set_cache(W["caches"][0], W["model"])
    outs = grp.solve(W["p"], iters, lam, theta=th, coef=cf, record_residuals=True, skip_gap=False)
    full = grp.assemble(outs)
    assert abs(outs[0]["gap"] - a["gap"]) <= 1e-9 * max(1.0, abs(a["gap"])), (outs[0]["gap"], a["gap"])
    for f in ("u0", "x", "u", "x_avg", "u_avg"):
        assert rel_err(full[f], a[f]) <= 1e-10, (f, rel_err(full[f], a[f]))
    for k in ("sig", "zeta", "psi"):
        assert rel_err(full[f"dual_{k}"], a[f"dual_{k}"]) <= 1e-10, k
    assert np.allclose(outs[0]["resid_trace"], a["resid_trace"], rtol=1e-8, atol=1e-12)


def test_shard_group_rejects_bad_members():
    c = load_case("tank3_tree30_N24")
    grp = LocalShardGroup(c.model, c.tree, c.factor, 2, c.scaling)
    grp.set_cache(c.cache, c.model)
    # an NCCL-less shard plan of a world-2 split cannot run alone
    with pytest.raises(ValidationError, match="tsmpc_solve_group"):
        grp.plans[0].solve(c.p, 5, c.lam, skip_gap=True)
    # members out of rank order are refused
    grp.plans.reverse()
    with pytest.raises(ValidationError, match="local shard plan of rank"):
        grp.solve(c.p, 5, c.lam)


def test_engine_solve_over_devices_matches_reference():
    """engine.solve(SolverConfig(devices=...)): the sharded solve behind the reference
    API (tsmpc_plans_create_multi + tsmpc_solve_multi; one GPU here, so one rank)."""
    c = load_case("bcn63_SMPC1_N24")
    z = c.z
    rep = engine.solve(c.model, c.tree, c.forecast, c.p, c.q,
                       engine.SolverConfig(max_iters=c.iters, devices=(0,)), basis=c.basis,
                       factor=c.factor, cache=c.cache, scaling=c.scaling, lam=c.lam)
    for f in ("u0", "x", "u", "x_avg", "u_avg"):
        assert rel_err(getattr(rep, f), z[f"r_{f}"]) <= c.tol(f), (f, rel_err(getattr(rep, f), z[f"r_{f}"]))
    for k in ("sig", "zeta", "psi"):
        assert rel_err(getattr(rep.dual, k), z[f"r_dual_{k}"]) <= c.tol("dual"), k
    g_ref = float(z["r_gap"])
    assert abs(rep.gap - g_ref) <= c.tol("gap") * max(1.0, abs(g_ref)), (rep.gap, g_ref)
    assert rep.iterations == c.iters


@pytest.mark.parametrize("tree_name,full", [("SMPC8", True), ("SMPC8", False), ("W4k", True)])
def test_peer_exchange_in_kernel_equals_nccl_launches(tree_name, full, monkeypatch):
    """The cut exchange inside the persistent kernel (tsmpc_plan_peer_open: receive
    rows and arrival counter mapped for every rank, both phases in one launch) gives
    the bits of the two-launch + ncclAllReduce path, over repeated solves (the
    arrival generations carry over).  One GPU: world 1, the plan is its own peer;
    TSMPC_SHARD_FULL makes every trunk position an exchanged one (n_xch > 0)."""
    import bench
    if full:
        monkeypatch.setenv("TSMPC_SHARD_FULL", "1")
    W = bench.build_workload(tree_name)
    iters = 30
    th, cf = engine.theta_schedule(iters)
    plan = DevicePlan(W["model"], W["tree"], W["factor"], W["scaling"], shard=(0, 1, nccl_unique_id()))
    plan.set_cache(W["caches"][0], W["model"])
    assert (plan.info()["exchange_doubles"] > 0) == full
    a = plan.solve(W["p"], iters, 0.05, theta=th, coef=cf, record_residuals=True)
    plan.peer_open([plan.peer_handles()])
    assert plan.info()["peer_exchange"] == 1
    outs = [plan.solve(W["p"], iters, 0.05, theta=th, coef=cf, record_residuals=True) for _ in range(2)]
    for b in outs:
        assert b["kernel_launches"] < a["kernel_launches"]
        for f in ("u0", "x", "u", "x_avg", "u_avg", "dual_sig", "dual_zeta", "dual_psi", "resid_trace"):
            assert np.array_equal(a[f], b[f]), f
        assert a["gap"] == b["gap"]
    plan.peer_close()
    c = plan.solve(W["p"], iters, 0.05, theta=th, coef=cf, record_residuals=True)
    assert np.array_equal(c["u_avg"], a["u_avg"]) and c["kernel_launches"] == a["kernel_launches"]
