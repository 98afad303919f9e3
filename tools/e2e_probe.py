"""Wall-clock split of one engine.solve call on SMPC8 (profiling helper): the device
stage cache (set_forecast) vs the whole call."""
import sys, time, pathlib
sys.path.insert(0, "/root/repo")
import numpy as np
import bench
from paper_1604_01074_b200 import engine, theta_schedule
from paper_1604_01074_b200.plan import plan_for
W = bench.build_workload("SMPC8")
cfg = engine.SolverConfig(max_iters=500, lam=0.4797702477755166)
args = dict(basis=W["basis"], factor=W["factor"], scaling=W["scaling"], lam=0.4797702477755166)
for _ in range(3):
    engine.solve(W["model"], W["tree"], W["forecasts"][0], W["p"], W["q"], cfg, **args)
import torch
plan = plan_for(W["model"], W["tree"], W["factor"], W["scaling"])
ts = {"set_forecast": [], "solve_call": [], "total": []}
for _ in range(10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan.set_forecast(W["forecasts"][0], W["q"], W["basis"], W["model"])
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    rep = engine.solve(W["model"], W["tree"], W["forecasts"][0], W["p"], W["q"], cfg, **args)
    t2 = time.perf_counter()
    ts["set_forecast"].append((t1 - t0) * 1e3)
    ts["total"].append((t2 - t1) * 1e3)
print({k: round(float(np.median(v)), 3) for k, v in ts.items() if v})
