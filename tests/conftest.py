"""Shared test helpers: golden-case loader and the `gpu` marker.

Golden fixtures (``tests/golden/*.npz``) are produced by the real reference
(``tests/golden/make_golden.py``) and are self-contained: they carry every
input so tests never read /root/reference at run time.
"""

from __future__ import annotations

import pathlib
import sys
from dataclasses import dataclass

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1604_01074_b200 import (DemandForecast, DualScaling, NetworkModel)  # noqa: E402
from paper_1604_01074_b200.precompute import (EliminationBasis, FactorCache,  # noqa: E402
                                              StageCache)
from paper_1604_01074_b200.tree import _finish  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"
SMALL_CASES = ["tank3_tree_1_N8", "tank3_tree_6_N8", "tank3_tree_30_N8", "small_s0", "small_s1",
               "small_s2", "small_s3", "small_s4", "small_s5", "small_denseA", "small_s6_plain"]
N24_CASES = ["tank3_tree30_N24", "bcn63_CE_N24", "bcn63_SMPC1_N24"]
ALL_CASES = SMALL_CASES + N24_CASES


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def has_gpu() -> bool:
    try:
        from paper_1604_01074_b200 import _native
        return _native.LIB_PATH.exists() and _native.device_count() > 0
    except Exception:
        return False


@dataclass
class Case:
    name: str
    z: dict
    model: NetworkModel
    tree: object
    forecast: DemandForecast
    p: np.ndarray
    q: np.ndarray
    basis: EliminationBasis
    factor: FactorCache
    cache: StageCache
    scaling: DualScaling | None
    lam: float
    iters: int

    def tol(self, field: str, floor: float = 1e-11) -> float:
        """10x the reference's own ulp-perturbation deviation, floored."""
        key = f"ulp_{field}"
        return max(10.0 * float(self.z[key]), floor) if key in self.z else floor


_CACHE: dict = {}


def load_case(name: str) -> Case:
    if name in _CACHE:
        return _CACHE[name]
    raw = np.load(GOLDEN / f"{name}.npz")
    z = {k: raw[k] for k in raw.files}
    keys = ("A", "B", "Gd", "E", "Ed", "u_min", "u_max", "x_min", "x_max", "x_s", "alpha1",
            "alpha2_schedule", "Wu")
    sc = z["m_scalars"]
    model = NetworkModel(**{k: z[f"m_{k}"] for k in keys}, W_alpha=float(sc[0]),
                         Wx=float(sc[1]), gamma_d=float(sc[2]))
    tree = _finish(int(z["t_N"]), z["t_stage_starts"], z["t_anc"], z["t_prob"], z["t_eps"])
    forecast = DemandForecast(z["f_dhat"], k=int(z["f_k"]))
    L = z["L"]
    basis = EliminationBasis(L=L, part_map=z["part_map"], Rhat=model.Wu @ L, Rbar=z["Rbar"],
                             Rbar_chol=z["Rbar_chol"], sigma=float(z["sigma"]))
    factor = FactorCache(Bbar=z["Bbar"], Phi=z["Phi"], Psi=z["Psi"], Rbar_chol=z["Rbar_chol"],
                         A=model.A, L=L)
    cache = StageCache(k=int(z["f_k"]), q=z["q"], demands=z["demands"], uhat=z["uhat"],
                       evec=z["evec"], beta=z["beta"], alpha_bar=z["alpha_bar"], pbar=z["pbar"])
    scaling = (DualScaling(z["sig_stage"], z["zeta_stage"], z["psi_stage"])
               if bool(z["precondition"]) else None)
    case = Case(name, z, model, tree, forecast, z["p"], z["q"], basis, factor, cache, scaling,
                float(z["lam"]), int(z["iters"]))
    _CACHE[name] = case
    return case


def rel_err(got, ref) -> float:
    got, ref = np.asarray(got, dtype=float), np.asarray(ref, dtype=float)
    return float(np.max(np.abs(got - ref)) / max(1.0, float(np.max(np.abs(ref)))))


@pytest.fixture(params=ALL_CASES)
def golden_case(request):
    return load_case(request.param)


@pytest.fixture(params=SMALL_CASES)
def small_case(request):
    return load_case(request.param)
