"""Device-loop vs whole-call time of one SMPC8 solve with and without the result
read-back (profiling helper): how much of the SolveReport copy the gap hides."""
import pathlib
import statistics
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import bench  # noqa: E402
from paper_1604_01074_b200 import theta_schedule  # noqa: E402
from paper_1604_01074_b200.plan import plan_for  # noqa: E402

W = bench.build_workload("SMPC8")
plan = plan_for(W["model"], W["tree"], W["factor"], W["scaling"])
plan.set_cache(W["caches"][0], W["model"])
th, cf = theta_schedule(500)
for keep in (True, False, True, False):
    walls, tot = [], []
    for _ in range(5):
        t0 = time.perf_counter()
        r = plan.solve(W["p"], 500, 0.48, theta=th, coef=cf, keep_device=keep)
        walls.append((time.perf_counter() - t0) * 1e3)
        tot.append(r["device_total_ms"])
    print(f"keep_device={keep}: call {statistics.median(walls):.3f} ms, loop+gap {statistics.median(tot):.3f} ms")
