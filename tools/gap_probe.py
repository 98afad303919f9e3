"""Device time of the APG loop vs loop + duality gap (profiling helper; no timing claims)."""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import bench  # noqa: E402
from paper_1604_01074_b200 import theta_schedule  # noqa: E402
from paper_1604_01074_b200.plan import DevicePlan  # noqa: E402

tree = sys.argv[1] if len(sys.argv) > 1 else "SMPC3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 500
W = bench.build_workload(tree)
plan = DevicePlan(W["model"], W["tree"], W["factor"], W["scaling"])
plan.set_cache(W["caches"][0], W["model"])
th, cf = theta_schedule(iters)
for _ in range(4):
    r = plan.solve(W["p"], iters, 0.05, theta=th, coef=cf, keep_device=True)
    print(f"{tree}: loop {r['device_ms']:.3f} ms, loop+gap {r['device_total_ms']:.3f} ms, "
          f"gap {r['device_total_ms'] - r['device_ms']:.3f} ms")
