"""The C-ABI library: builds for sm_100a, loads, exports every symbol declared in
include/tsmpc.h, and fails loudly (DeviceError) when no CUDA device is present."""

import pathlib
import re

import pytest

from conftest import ROOT, has_gpu
from paper_1604_01074_b200 import _native
from paper_1604_01074_b200.errors import DeviceError


def _declared():
    text = (ROOT / "include" / "tsmpc.h").read_text()
    return sorted(set(re.findall(r"\b(tsmpc_[a-z_]+)\s*\(", text)))


def test_library_builds_and_exports_every_declared_symbol():
    _native.build_library()
    lib = _native.load_library()
    names = _declared()
    assert len(names) >= 12
    for name in names:
        assert hasattr(lib, name), name
    assert set(_native.SIGNATURES) >= set(names)


def test_sass_contains_fp64_tensor_instructions():
    import subprocess
    lib = pathlib.Path(_native.LIB_PATH)
    out = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in out                    # fp64 tensor-core MMA (mma.sync f64)
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", str(lib)], capture_output=True,
                                       text=True).stdout


@pytest.mark.skipif(has_gpu(), reason="checks the no-device behaviour")
def test_fails_loudly_without_device():
    from paper_1604_01074_b200 import synth
    from paper_1604_01074_b200.plan import DevicePlan
    from paper_1604_01074_b200.precompute import compute_basis, factor_step
    assert _native.device_count() == 0
    m = synth.three_tank_network()
    t = synth.uniform_tree([2], N=3, n_d=2, seed=1)
    f = factor_step(compute_basis(m), m)
    with pytest.raises(DeviceError):
        DevicePlan(m, t, f)
