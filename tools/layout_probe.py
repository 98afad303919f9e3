"""Loop time of identical SMPC8 plans at different device addresses / arena skews
(TSMPC_ARENA_PAD): is the kernel sensitive to the memory layout?
    python tools/layout_probe.py [pad_bytes ...]"""
import os
import pathlib
import statistics
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1604_01074_b200 import theta_schedule  # noqa: E402
from paper_1604_01074_b200.plan import DevicePlan  # noqa: E402

tree = os.environ.get("PROBE_TREE", "SMPC8")
W = bench.build_workload(tree)
lam = 0.47977
th, cf = theta_schedule(500)
pads = [int(a) for a in sys.argv[1:]] or [0]
keep = []
for pad in pads:
    os.environ["TSMPC_ARENA_PAD"] = str(pad)
    ts = []
    for i in range(4):
        plan = DevicePlan(W["model"], W["tree"], W["factor"], W["scaling"])
        plan.set_cache(W["caches"][0], W["model"])
        r = [plan.solve(W["p"], 500, lam, theta=th, coef=cf, keep_device=True, skip_gap=True)["device_ms"]
             for _ in range(3)]
        ts.append(statistics.median(r) * 1e3 / 500)
        keep.append(plan)
        keep.append(torch.empty((i + 1) * 3 * 1024 * 1024 // 8 + 4096, dtype=torch.float64, device="cuda"))
    print(f"{tree} pad {pad:8d}: " + " ".join(f"{t:6.1f}" for t in ts) + f"  us/iter  (mean {statistics.mean(ts):.1f})",
          flush=True)
