"""Phase timers / trial time of one shard plan (profiling helper; no timing claims).

    TSMPC_TIMER_CTA=0 TSMPC_LIB=paper_1604_01074_b200/libtsmpc_timers.so \
        python tools/shard_prof.py --tree W4k --world 8 --rank 0 --iters 100
"""
import argparse
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import bench  # noqa: E402
from paper_1604_01074_b200.plan import DevicePlan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tree", default="W4k")
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--rank", type=int, default=0)
ap.add_argument("--iters", type=int, default=100)
a = ap.parse_args()
W = bench.build_workload(a.tree)
plan = DevicePlan(W["model"], W["tree"], W["factor"], W["scaling"], shard=(a.rank, a.world, None))
plan.set_cache(W["caches"][0], W["model"])
plan.trial(5)
plan.debug_timers()  # reset
ms = plan.trial(a.iters)
print(a.tree, f"rank {a.rank}/{a.world}", plan.info(), f"trial {ms * 1e3 / a.iters:.1f} us/iter")
tm = plan.debug_timers()
names = ["bwd fill", "bwd xiq scan", "bwd h=Ls'z", "bwd g scan", "fwd S scan", "bwd z=B'xiq",
         "fwd bv=B du", "fwd u, x scan", "fwd epilogue", "grid.sync", "trunk sweep", "fwd du=Lt S",
         "trunk needs+own", " sweep: stage", " sweep: loads", " sweep: levels"]
tot = float(tm.sum())
if tot > 0:
    for k, nm in enumerate(names):
        print(f"  {nm:14s} {tm[k] / a.iters / 1.965e3:8.2f} us/iter  {100 * tm[k] / tot:5.1f}%")
