"""Run one solve of a synthetic bcn63 case (profiling driver; no timing claims)."""
import argparse
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

from paper_1604_01074_b200 import (build_stage_cache, compute_basis, compute_preconditioner,  # noqa: E402
                                   factor_step, node_demands, synth, theta_schedule)
from paper_1604_01074_b200.plan import DevicePlan, tuned_plan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tree", default="CE")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--skip-gap", action="store_true")
ap.add_argument("--plain", action="store_true", help="no dual preconditioner (identity scaling)")
a = ap.parse_args()
m = synth.bcn63_network()
t = synth.paper_tree(*synth.PAPER_TREES[a.tree])
b = compute_basis(m)
f = factor_step(b, m)
s = compute_preconditioner(b, m, t.N, tree=t)
p, q = synth.initial_state(m)
fc = synth.forecast_for(t)
c = build_stage_cache(b, m, t, node_demands(t, fc), k=0, q=q)
plan = (DevicePlan if os.environ.get("PROF_UNTUNED") else tuned_plan)(m, t, f, None if a.plain else s)
plan.set_cache(c, m)
th, cf = theta_schedule(a.iters)
for _ in range(a.reps):
    r = plan.solve(p, a.iters, 0.48, theta=th, coef=cf, keep_device=True, skip_gap=a.skip_gap)
print(a.tree, plan.info(), f"loop {r['device_ms']:.3f} ms = {r['device_ms']*1e3/a.iters:.1f} us/iter")
tm = plan.debug_timers()
import os
if os.environ.get("TSMPC_DENSE_NAMES"):
    names = ["bwd fill", "bwd xiq scan", "bwd gemm1", "bwd g scan", "fwd t load", "fwd S scan",
             "fwd gemm2", "fwd x scan", "fwd epilogue", "grid.sync", "trunk sweep", "trunk gemm",
             "trunk rows"]
else:  # sparse kernel marks (tsmpc_sparse.cu)
    names = ["bwd fill", "bwd xiq scan", "bwd h=Ls'z", "bwd g scan", "fwd S scan", "bwd z=B'xiq",
             "fwd bv=B du", "fwd u, x scan", "fwd epilogue", "grid.sync", "trunk sweep", "fwd du=Lt S",
             "trunk needs+own", " sweep: stage", " sweep: loads", " sweep: levels"]
tot = float(tm.sum())
if tot > 0:
    n = a.iters * a.reps
    for k, nm in enumerate(names):
        print(f"  {nm:14s} {tm[k] / n / 1.965e3:8.2f} us/iter  {100 * tm[k] / tot:5.1f}%")
