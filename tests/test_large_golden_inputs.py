"""CPU check of the benchmark-tree goldens: the synthetic inputs regenerate
bit-identically (sha256 stored by tests/golden/make_golden_large.py), so the GPU
box compares against exactly what the reference was fed."""

import pytest

from large_golden import LARGE_CASES, TRACE_CASES, load, workload


@pytest.mark.parametrize("name", LARGE_CASES + TRACE_CASES)
def test_regenerated_inputs_match_fixture_digest(name):
    z = load(name)
    W = workload(z)  # asserts the digest
    assert W["tree"].n_edges == int(z["edges"])
    assert z["r_u0"].shape == (W["model"].n_u,)
