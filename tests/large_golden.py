"""Loader / comparison helpers for the benchmark-tree goldens of
tests/golden/make_golden_large.py (the real reference's engine.solve on bcn63
CE / SMPC1 / SMPC3 / SMPC8 / W4k / W16k).

Inputs are regenerated with ``synth`` and checked against the sha256 digest the
generator stored; results are compared on the stored row sample, on the
per-column sums and maxima of the full arrays, and on u0 / residual / gap.
Tolerance per field and metric: 10x the reference's own ulp-perturbation
deviation in that metric, floored at 1e-11.
"""

from __future__ import annotations

import hashlib
import pathlib

import numpy as np

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"
FIELDS = ("x", "u", "x_avg", "u_avg", "dual_sig", "dual_zeta", "dual_psi")
LARGE_CASES = ["L_bcn63_CE_i500", "L_bcn63_CE_i2000", "L_bcn63_SMPC1_i2000", "L_bcn63_SMPC3_i500",
               "L_bcn63_SMPC3_i2000", "L_bcn63_SMPC8_i500", "L_bcn63_W4k_i100", "L_bcn63pw_SMPC3_i500",
               "L_bcn63_W16k_i20"]
TRACE_CASES = ["L_bcn63_CE_trace_i150", "L_bcn63_SMPC1_trace_i60"]
FLOOR = 1e-11


def load(name: str) -> dict:
    raw = np.load(GOLDEN / f"{name}.npz")
    return {k: raw[k] for k in raw.files}


def workload(z: dict) -> dict:
    """Regenerate the inputs the reference was fed and check their digest."""
    from paper_1604_01074_b200 import (build_stage_cache, compute_basis, compute_preconditioner,
                                       factor_step, node_demands, synth)
    model = synth.bcn63_network(paper_weights=bool(z.get("paper_weights", False)))
    tree = synth.paper_tree(*synth.PAPER_TREES[str(z["tree_name"])])
    fc = synth.forecast_for(tree, k=0)
    p, q = synth.initial_state(model)
    h = hashlib.sha256()
    for a in synth.input_arrays(model, tree, fc, p, q):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == str(z["input_sha256"]), "regenerated inputs differ from the fixture's"
    basis = compute_basis(model)
    factor = factor_step(basis, model)
    scaling = compute_preconditioner(basis, model, tree.N, tree=tree)
    cache = build_stage_cache(basis, model, tree, node_demands(tree, fc), k=0, q=q)
    return dict(model=model, tree=tree, forecast=fc, p=p, q=q, basis=basis, factor=factor,
                scaling=scaling, cache=cache)


def tol(z: dict, key: str) -> float:
    return max(10.0 * float(z[key]), FLOOR) if key in z else FLOOR


def col_scale(ref_colmax: np.ndarray, blockmax: float) -> np.ndarray:
    return np.maximum(ref_colmax, 1e-3 * max(1.0, blockmax))


def compare(z: dict, got: dict) -> dict:
    """Deviation of the device results from the golden, per field and metric, next
    to the allowed tolerance: {name: (deviation, tolerance)}."""
    out = {}
    rows_e, rows_n = z["rows_e"], z["rows_n"]
    for f in FIELDS:
        a = np.asarray(got[f], dtype=float)
        ref_rows = z[f"r_{f}_rows"]
        mine = a[rows_n if f in ("x", "x_avg") else rows_e]
        blk = float(z[f"r_{f}_max"])
        out[f"{f}:rows_block"] = (float(np.max(np.abs(mine - ref_rows)) / max(1.0, blk)), tol(z, f"ulp_{f}"))
        scale = col_scale(z[f"r_{f}_colmax"], blk)
        out[f"{f}:rows_column"] = (float(np.max(np.max(np.abs(mine - ref_rows), axis=0) / scale)),
                                   tol(z, f"ulpc_{f}"))
        out[f"{f}:colmax"] = (float(np.max(np.abs(np.max(np.abs(a), axis=0) - z[f"r_{f}_colmax"]) / scale)),
                              tol(z, f"ulpc_{f}"))
        cs = z[f"r_{f}_colsum"]
        sab = np.maximum(np.abs(cs), 1e-3 * max(1.0, float(np.max(np.abs(cs)))))
        # column sums are checked against |sum| (the generator calibrated against sum |.|,
        # which is >= |sum|): take the larger of the two scales per column
        out[f"{f}:colsum"] = (float(np.max(np.abs(a.sum(axis=0) - cs) / np.maximum(sab, scale))),
                              tol(z, f"ulps_{f}") + tol(z, f"ulpc_{f}"))
    out["u0"] = (float(np.max(np.abs(got["u0"] - z["r_u0"])) / max(1.0, float(np.max(np.abs(z["r_u0"]))))),
                 tol(z, "ulp_u0"))
    r = float(z["r_residual_inf"])
    out["residual_inf"] = (abs(got["residual_inf"] - r) / max(1.0, abs(r)), tol(z, "ulp_residual_inf"))
    if "gap" in got and got["gap"] is not None and np.isfinite(got["gap"]):
        g = float(z["r_gap"])
        out["gap"] = (abs(got["gap"] - g) / max(1.0, abs(g)), tol(z, "ulp_gap"))
    return out


def failures(cmp: dict) -> dict:
    return {k: v for k, v in cmp.items() if not v[0] <= v[1]}
