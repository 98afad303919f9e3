"""Bitwise comparison of two library builds on one solve (A/B experiments):
    TSMPC_LIB=<a.so> python tools/bitwise_variants.py --tree SMPC8 --out /tmp/a.npz
    TSMPC_LIB=<b.so> python tools/bitwise_variants.py --tree SMPC8 --out /tmp/b.npz --ref /tmp/a.npz"""
import argparse
import pathlib
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1604_01074_b200 import theta_schedule  # noqa: E402
from paper_1604_01074_b200.plan import DevicePlan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tree", default="SMPC8")
ap.add_argument("--iters", type=int, default=60)
ap.add_argument("--out", required=True)
ap.add_argument("--ref")
ap.add_argument("--record", action="store_true", help="record the residual trace (disables some fast paths)")
a = ap.parse_args()
W = bench.build_workload(a.tree)
plan = DevicePlan(W["model"], W["tree"], W["factor"], W["scaling"])
plan.set_cache(W["caches"][0], W["model"])
th, cf = theta_schedule(a.iters)
r = plan.solve(W["p"], a.iters, 0.4797, theta=th, coef=cf, record_residuals=a.record)
keys = ("u0", "x", "u", "x_avg", "u_avg", "dual_sig", "dual_zeta", "dual_psi") + (("resid_trace",) if a.record else ())
np.savez(a.out, **{k: r[k] for k in keys}, gap=r["gap"])
if a.ref:
    z = np.load(a.ref)
    diff = {k: float(np.max(np.abs(z[k] - r[k]))) for k in keys}
    print("bitwise" if all(v == 0 for v in diff.values()) and z["gap"] == r["gap"] else f"DIFF {diff}")
