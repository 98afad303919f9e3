"""GPU: the sharded solve machinery (phase 1 -> ncclAllReduce -> phase 2 per
iteration, streamed tiles) on one GPU with a one-rank NCCL communicator.  The
multi-rank data movement is NCCL's; the partition logic is covered on CPU by
tests/test_shard_cpu.py (gloo, world size 2)."""

import numpy as np
import pytest

from conftest import has_gpu, load_case, rel_err

pytestmark = pytest.mark.gpu

if not has_gpu():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1604_01074_b200 import engine  # noqa: E402
from paper_1604_01074_b200.plan import DevicePlan  # noqa: E402
from paper_1604_01074_b200.shard import nccl_unique_id  # noqa: E402


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
    out = plan.solve(c.p, c.iters, c.lam, theta=th, coef=cf, skip_gap=True)
    assert out["kernel_launches"] == 2 * c.iters
    for f in ("u0", "x", "u", "x_avg", "u_avg"):
        assert rel_err(out[f], z[f"r_{f}"]) <= c.tol(f), (f, rel_err(out[f], z[f"r_{f}"]))
    for k in ("sig", "zeta", "psi"):
        assert rel_err(out[f"dual_{k}"], z[f"r_dual_{k}"]) <= c.tol("dual"), k
    r_ref = float(z["r_residual_inf"])
    assert abs(out["residual_inf"] - r_ref) <= c.tol("residual_inf") * max(1.0, abs(r_ref))
    assert np.isnan(out["gap"])


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
