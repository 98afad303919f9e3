"""Timeline of one steady-state SMPC8 iteration across CTAs (timer build):
    TSMPC_LIB=paper_1604_01074_b200/libtsmpc_timers.so python tools/trace_probe.py
Chain CTAs: 0 start, 5 heads published, 1 backward done, 2 zero-input forward done,
3 TR received, 4 finish done.  Trunk CTAs: 0 start, 1 own terms done, 2 heads
received, 3 sweep done, 4 trunk barrier passed, 5 TR published, 6 trunk-row epilogues
done.  Times in us from the earliest start."""
import os
import pathlib
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
os.environ.setdefault("PROF_UNTUNED", "1")

import bench  # noqa: E402
from paper_1604_01074_b200 import theta_schedule  # noqa: E402
from paper_1604_01074_b200.plan import DevicePlan  # noqa: E402

W = bench.build_workload(sys.argv[1] if len(sys.argv) > 1 else "SMPC8")
plan = DevicePlan(W["model"], W["tree"], W["factor"], W["scaling"])
plan.set_cache(W["caches"][0], W["model"])
th, cf = theta_schedule(100)
plan.solve(W["p"], 100, 0.48, theta=th, coef=cf, keep_device=True, skip_gap=True)
buf = (np.zeros(16 + 8 * 256, dtype=np.uint64))
import ctypes  # noqa: E402
nat_buf = buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
plan._lib.tsmpc_debug_timers(plan._h, nat_buf, buf.size)
info = plan.info()
C, tc = info["ctas"], info["trunk_ctas"]
st = buf[16:16 + 8 * C].reshape(C, 8).astype(np.float64)
t0 = st[:, 0][st[:, 0] > 0].min()
rel = np.where(st > 0, (st - t0) / 1e3, np.nan)
chain, trunk = rel[:C - tc], rel[C - tc:]
names_c = {0: "start", 6: "backward entered", 7: "head sums phase 1", 5: "heads published", 1: "backward done", 2: "zero-input fwd done", 3: "TR received",
           4: "finish done"}
names_t = {0: "start", 1: "own terms done", 2: "heads received", 3: "sweep done", 4: "trunk barrier",
           5: "TR published", 6: "trunk-row epilogues done"}
print(f"{C - tc} chain CTAs, {tc} trunk CTAs (us from the earliest iteration start; min / median / max)")
for k, nm in names_c.items():
    v = chain[:, k]
    print(f"  chain {nm:24s} {np.nanmin(v):7.2f} {np.nanmedian(v):7.2f} {np.nanmax(v):7.2f}")
for k, nm in names_t.items():
    v = trunk[:, k]
    print(f"  trunk {nm:24s} {np.nanmin(v):7.2f} {np.nanmedian(v):7.2f} {np.nanmax(v):7.2f}")
