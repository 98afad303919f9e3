import sys, time, statistics
sys.path.insert(0, '.')
import torch, bench
from paper_1604_01074_b200 import theta_schedule
from paper_1604_01074_b200.plan import DevicePlan
W = bench.build_workload("SMPC8")
plan = DevicePlan(W["model"], W["tree"], W["factor"], W["scaling"])
plan.set_cache(W["caches"][0], W["model"])
lam = 0.47977
th, cf = theta_schedule(500)
dev = torch.device("cuda", 0)
def run(flush_mb):
    out = []
    for _ in range(6):
        if flush_mb:
            b = torch.empty(flush_mb * 1024 * 1024 // 4, dtype=torch.float32, device=dev); b.fill_(1.0); torch.cuda.synchronize()
        r = plan.solve(W["p"], 500, lam, theta=th, coef=cf, keep_device=True, skip_gap=True)
        out.append(r["device_ms"])
    return statistics.median(out[1:])
for f in (0, 256, 0, 512, 128, 0):
    print(f, run(f))
for iters in (50, 100, 500):
    th2, cf2 = theta_schedule(iters)
    rs=[plan.solve(W["p"], iters, lam, theta=th2, coef=cf2, keep_device=True, skip_gap=True)["device_ms"] for _ in range(4)]
    print("iters", iters, rs)
