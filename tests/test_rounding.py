"""Rounding (rounding.py): device maxcut_round and host qap_round against the
reference's outputs recorded in tests/golden/rounding.npz
(oracle/make_golden.py rounding_cases).  Cut values of integer-weight
graphs and assignment objectives of integer QAP data are exact, so the
comparisons are bit-exact."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import cuda_ok
from helpers import load_npz
from paper_2312_11801_b200 import instances as inst
from paper_2312_11801_b200 import rounding as R


@pytest.mark.parametrize("key", ["qap4", "qap6"])
def test_qap_round_matches_reference(key):
    z = load_npz("rounding.npz")
    q = inst.Qap(z[f"{key}/W"], z[f"{key}/D"])
    r = R.qap_round(z[f"{key}/u"], q)
    np.testing.assert_array_equal(r.perm, z[f"{key}/perm"])
    assert r.objective == float(z[f"{key}/objective"][0])
    r2 = R.qap_round(z[f"{key}/u"], q, known_optimum=r.objective / 2)
    assert r2.relative_gap == pytest.approx(1.0)
    t = R.GapTracker()
    assert t.update(r2) == pytest.approx(1.0) and t.update(0.5) == 0.5 and t.update(0.7) == 0.5


def test_hungarian_rejects_bad_input():
    with pytest.raises(ValueError):
        R.hungarian(np.ones((2, 3)))
    with pytest.raises(ValueError):
        R.hungarian(np.array([[0.0, np.inf], [1.0, 0.0]]))
    np.testing.assert_array_equal(R.hungarian(np.array([[4.0, 1.0], [2.0, 8.0]])), [1, 0])


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")
@pytest.mark.parametrize("name", ["er", "torus"])
def test_maxcut_round_bit_exact(name):
    z = load_npz("rounding.npz")
    g = inst.Graph(int(z[f"{name}/u"].shape[0]), z[f"{name}/eu"], z[f"{name}/ev"], z[f"{name}/ew"])
    r = R.maxcut_round(z[f"{name}/u"], g)
    assert r.value == float(z[f"{name}/value"][0])
    np.testing.assert_array_equal(r.values, z[f"{name}/all"])
    np.testing.assert_array_equal(r.assignment, z[f"{name}/x"])


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")
def test_maxcut_round_device_factor_and_errors():
    """A device tensor factor, a single column, and the reference's shape errors."""
    from paper_2312_11801_b200.runtime import runtime
    rt = runtime()
    g = inst.erdos_renyi(200, 0.05, 1)
    u = np.random.default_rng(3).standard_normal((200, 4))
    r_host = R.maxcut_round(u, g)
    r_dev = R.maxcut_round(rt.upload(u), g)
    assert r_host.value == r_dev.value
    x = np.where(u[:, int(np.argmax(r_host.values))] >= 0, 1, -1)
    np.testing.assert_array_equal(r_dev.assignment, x)
    lap = g.laplacian()
    assert r_host.value == 0.25 * float(x @ (lap @ x))
    with pytest.raises(ValueError):
        R.maxcut_round(np.zeros((199, 2)), g)
