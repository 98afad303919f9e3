"""Full-size parity on the benchmark trees (BASELINE.json configs[1]-[3]) against
the CPU oracle, a few APG iterations each.

The golden fixtures stop at SMPC3; these cases exercise the plans that only the
large trees produce: SMPC8 runs the streamed tile slots with 3-4 chains per CTA
and two grid barriers per iteration (no split mode), W4k (86,561 edges) adds
multi-tile CTAs with trunk rows spread over every CTA, W16k (345,121 edges,
16,384 scenarios) CTAs of 28 tiles whose per-row meta is staged
tile by tile.  The oracle
(`oracle/tsmpc_oracle.py:122-169`, the reference loop `engine.py:519-600`) is
the checker only.

Tolerance: the device and the oracle sum in different orders (fp64); after a
handful of iterations the relative deviation stays at the 1e-12 level, so the
bound is 1e-9 relative to max(1, max|ref|) on every returned block.
"""

import numpy as np
import pytest

from conftest import has_gpu, rel_err

pytestmark = pytest.mark.gpu

if not has_gpu():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1604_01074_b200 import engine  # noqa: E402
from paper_1604_01074_b200.plan import DevicePlan  # noqa: E402
from oracle import tsmpc_oracle as O  # noqa: E402

TOL = 1e-9


@pytest.mark.parametrize("tree_name,iters,path", [("SMPC3", 6, "sparse"), ("SMPC8", 6, "sparse"),
                                                  ("SMPC8", 3, "dense"), ("W4k", 3, "sparse"),
                                                  ("W16k", 2, "sparse")])
def test_full_size_tree_matches_oracle(tree_name, iters, path, monkeypatch):
    import bench
    monkeypatch.setenv("TSMPC_FORCE_DENSE", "1" if path == "dense" else "0")
    W = bench.build_workload(tree_name)
    model, tree, cache = W["model"], W["tree"], W["caches"][0]
    plan = DevicePlan(model, tree, W["factor"], W["scaling"])
    plan.set_cache(cache, model)
    info = plan.info()
    assert info["sparse"] == (1 if path == "sparse" else 0), info["path"]
    if tree_name != "SMPC3" and path == "sparse":
        assert info["wide"] == 1 and info["resident_ctas"] == 0, info
    if tree_name == "W16k":  # 28 tiles per CTA: per-tile meta windows, fill rows through HBM
        assert info["tiles"] >= 28 * 148 - 148 and info["fill_rows_hbm"] == 1, info
    lam = 0.05
    th, cf = engine.theta_schedule(iters)
    out = plan.solve(W["p"], iters, lam, theta=th, coef=cf, skip_gap=True, record_residuals=True)
    ref = O.apg(O.factor_dict(W["factor"]), O.cache_dict(cache, model, tree), O.tree_dict(tree),
                O.model_dict(model), W["p"], lam, iters, scaling=O.scaling_tuple(W["scaling"]),
                record=True)
    for f in ("u0", "x", "u", "x_avg", "u_avg"):
        assert rel_err(out[f], ref[f]) <= TOL, (f, rel_err(out[f], ref[f]))
    for k, name in enumerate(("sig", "zeta", "psi")):
        assert rel_err(out[f"dual_{name}"], ref["dual"][k]) <= TOL, (name, rel_err(out[f"dual_{name}"], ref["dual"][k]))
    np.testing.assert_allclose(out["resid_trace"], ref["residual_trace"], rtol=1e-9, atol=1e-9)
