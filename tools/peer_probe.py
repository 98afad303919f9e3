"""Loop time of a world-1 shard plan: two launches + ncclAllReduce per iteration
vs both phases and the in-kernel exchange in one launch (profiling helper)."""
import pathlib
import statistics
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import bench  # noqa: E402
from paper_1604_01074_b200 import theta_schedule  # noqa: E402
from paper_1604_01074_b200.plan import DevicePlan  # noqa: E402
from paper_1604_01074_b200.shard import nccl_unique_id  # noqa: E402

tree = sys.argv[1] if len(sys.argv) > 1 else "W4k"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
W = bench.build_workload(tree)
th, cf = theta_schedule(iters)
plan = DevicePlan(W["model"], W["tree"], W["factor"], W["scaling"], shard=(0, 1, nccl_unique_id()))
plan.set_cache(W["caches"][0], W["model"])


def loop_ms():
    return statistics.median(plan.solve(W["p"], iters, 0.48, theta=th, coef=cf, skip_gap=True,
                                        keep_device=True)["device_ms"] for _ in range(4))


a = loop_ms()
plan.peer_open([plan.peer_handles()])
b = loop_ms()
print(f"{tree} world-1 shard, exchange doubles {plan.info()['exchange_doubles']}: "
      f"2 launches + all-reduce {a * 1e3 / iters:.1f} us/iter, one launch {b * 1e3 / iters:.1f} us/iter")
