"""Closed-loop golden vectors from the REAL reference (run in this container).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_closed_loop_golden.py

Runs ``treesmpc.closed_loop.run_closed_loop`` (``pkg/src/treesmpc/
closed_loop.py:107-208``) on self-contained inputs and stores inputs and
outputs (states, controls, per-step residuals / gaps, KPIs) as
``tests/golden/cl_<name>.npz`` for tests/test_closed_loop_gpu.py.  Each case is
also re-run with the reference's solve-step outputs perturbed at the ulp level
(as in make_golden.py) to calibrate the tolerance of the closed-loop outputs,
where controls feed back into the next solve.
"""

from __future__ import annotations

import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
from make_golden import OUT, _Perturb, pack_inputs, ref_model, ref_tree  # noqa: E402

from paper_1604_01074_b200 import DemandForecast, synth  # noqa: E402
from treesmpc import closed_loop as R_cl  # noqa: E402
from treesmpc import engine as R_engine  # noqa: E402


_LAM = []
_orig_lambda = R_engine.compute_lambda


def _recording_lambda(*a, **k):
    v = _orig_lambda(*a, **k)
    _LAM.append(v)
    return v


R_cl.engine.compute_lambda = _recording_lambda


def run(model, tree, realized, nominal, x0, u_prev, iters, warm, precondition, perturb=False):
    cfg = R_cl.SimulationConfig(
        network=ref_model(model), tree=ref_tree(tree), demands=realized, forecast=nominal,
        h_s=realized.shape[0], x0=x0, u_prev=u_prev, k0=0,
        solver=R_engine.SolverConfig(max_iters=iters, warm_start=warm, precondition=precondition))
    if not perturb:
        return R_cl.run_closed_loop(cfg)
    with _Perturb(seed=3):
        return R_cl.run_closed_loop(cfg)


def case(name, model, tree, h_s, iters, warm, precondition, seed):
    rng = np.random.default_rng(seed)
    N = tree.N
    base = rng.uniform(0.5, 1.5, model.n_d) * (30.0 if model.n_d == 2 else 8.0)
    kk = np.arange(h_s + N)
    nominal = base[None, :] * (1.0 + 0.3 * np.sin(2 * np.pi * (kk[:, None] - 7) / 24.0))
    realized = nominal[:h_s] + rng.normal(0.0, 0.05, (h_s, model.n_d)) * base[None, :]
    x0 = 0.5 * (model.x_min + model.x_max)
    u_prev = np.clip(np.full(model.n_u, 5.0), model.u_min, model.u_max)
    _LAM.clear()
    res = run(model, tree, realized, nominal, x0, u_prev, iters, warm, precondition)
    lam = _LAM[0]
    per = run(model, tree, realized, nominal, x0, u_prev, iters, warm, precondition, perturb=True)
    d = {}
    pack_inputs(d, model, tree, DemandForecast(nominal[:N], k=0), x0, u_prev)
    d.update(cl_realized=realized, cl_nominal=nominal, cl_iters=np.array(iters),
             cl_warm=np.array(warm), cl_precondition=np.array(precondition), lam=np.array(lam),
             r_states=res.states, r_controls=res.controls, r_residuals=res.residuals,
             r_gaps=res.gaps, r_kpis=np.array([res.kpis.economic, res.kpis.smoothness,
                                               res.kpis.safety_shortfall,
                                               res.kpis.network_utility]),
             r_economic=res.economic, r_smoothing=res.smoothing, r_safety=res.safety)
    for f, a, b in (("states", res.states, per.states), ("controls", res.controls, per.controls),
                    ("residuals", res.residuals, per.residuals), ("gaps", res.gaps, per.gaps)):
        d[f"ulp_{f}"] = np.array(np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(a))))
    np.savez_compressed(OUT / f"cl_{name}.npz", **d)
    print(name, {k: float(v) for k, v in d.items() if k.startswith("ulp_")},
          res.kpis.to_dict(), f"{res.wall_times['per_step_s']:.2f} s/step")


if __name__ == "__main__":
    m3 = synth.three_tank_network()
    case("tank3_tree6_warm", m3, synth.uniform_tree([3, 2], N=8, n_d=2, seed=5), h_s=8, iters=300,
         warm=True, precondition=True, seed=1)
    case("tank3_tree6_cold", m3, synth.uniform_tree([3, 2], N=8, n_d=2, seed=5), h_s=6, iters=300,
         warm=False, precondition=False, seed=2)
    mb = synth.bcn63_network()
    case("bcn63_CE_warm", mb, synth.paper_tree(1, 1, 1, N=24), h_s=4, iters=200, warm=True,
         precondition=True, seed=3)
