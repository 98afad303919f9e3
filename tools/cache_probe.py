"""Device loop time of SMPC8 with the host-built stage cache (set_cache) vs the
device-built one (set_forecast), same plan, same step size (diagnostic)."""
import pathlib
import statistics
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1604_01074_b200 import engine, theta_schedule  # noqa: E402
from paper_1604_01074_b200.plan import DevicePlan  # noqa: E402

W = bench.build_workload("SMPC8")
plan = DevicePlan(W["model"], W["tree"], W["factor"], W["scaling"])
lam = 0.47977
th, cf = theta_schedule(500)


def t(label):
    r = [plan.solve(W["p"], 500, lam, theta=th, coef=cf, keep_device=True, skip_gap=True)["device_ms"]
         for _ in range(4)]
    print(f"{label:34s} {statistics.median(r[1:]):8.3f} ms", flush=True)


for rep in range(2):
    plan.set_cache(W["caches"][0], W["model"])
    t("host cache k=0 (set_cache)")
    plan.set_forecast(W["forecasts"][0], W["q"], W["basis"], W["model"])
    t("device cache k=0 (set_forecast)")
    plan.set_forecast(W["forecasts"][1], W["q"], W["basis"], W["model"])
    t("device cache k=1 (set_forecast)")
    plan.set_cache(W["caches"][1], W["model"])
    t("host cache k=1 (set_cache)")
rep = engine.solve(W["model"], W["tree"], W["forecasts"][0], W["p"], W["q"], engine.SolverConfig(max_iters=500),
                   basis=W["basis"], factor=W["factor"], scaling=W["scaling"], lam=lam)
print("engine.solve device_ms", rep.device_ms, "wall", rep.wall_time_s * 1e3)
import time  # noqa: E402
for k in range(6):
    t0 = time.perf_counter()
    rep = engine.solve(W["model"], W["tree"], W["forecasts"][k % 2], W["p"], W["q"],
                       engine.SolverConfig(max_iters=500), basis=W["basis"], factor=W["factor"],
                       scaling=W["scaling"], lam=lam)
    print(f"engine.solve call {k}: wall {1e3 * (time.perf_counter() - t0):.2f} ms, device loop {rep.device_ms:.2f} ms, "
          f"iterations {rep.iterations}")
