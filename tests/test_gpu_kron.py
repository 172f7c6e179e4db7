"""K1q: the QAP cost applied as the dense contraction coef * D X W^T on the
FP64 tensor cores (usbs_kron.cu; problem.py:364-371, 462-477) -- C V and
Z V = C V - A*(y) V against the oracle's scipy CSR products, with the
Kronecker factors from the builder and detected from a reference-style CSR,
and against the sparse path (USBS_KRON=0)."""
from __future__ import annotations

import dataclasses

import numpy as np
import pytest

from helpers import random_qap
from oracle import usbs_cpu as O
from paper_2312_11801_b200 import instances as inst

pytestmark = pytest.mark.gpu

EPS = 2.0 ** -53


def _cases():
    c3 = inst.baseline_config("C3").problem
    q5 = inst.qap_problem(random_qap(5, 3))
    return {"C3": c3, "C3_detected": dataclasses.replace(c3, kron_factors=None), "qap5": q5,
            "qap3_detected": dataclasses.replace(inst.qap_problem(random_qap(3, 1)), kron_factors=None)}


CASES = _cases()


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("k", [1, 11, 20])
def test_kron_apply_matches_oracle(name, k, monkeypatch):
    from paper_2312_11801_b200 import runtime
    p = CASES[name]
    rng = np.random.default_rng(k)
    y = rng.standard_normal(p.m) * 1e-3
    y[p.ineq_mask] = np.abs(y[p.ineq_mask])
    v, _ = np.linalg.qr(rng.standard_normal((p.n, k)))
    dp = runtime.DeviceProblem(p)
    assert dp.kron is not None
    rt = dp.rt
    V = rt.upload(v)
    z = (p.cost - O.adjoint_csr(p.constraints, y, p.n)).tocsr()
    for which, mat in ((0, p.cost.tocsr()), (1, z)):
        if which:
            dp.assemble(rt.upload(y))
        got = rt.download(dp.apply(which, V))
        want = mat @ v
        lim = 8.0 * (np.diff(mat.indptr)[:, None] + 2) * EPS * (abs(mat) @ np.abs(v)) + 1e-300
        assert np.max(np.abs(got - want) / lim) <= 1.0, (name, which, k)
        # same result as the sparse path to rounding
        monkeypatch.setenv("USBS_KRON", "0")
        sparse = rt.download(dp.apply(which, V))
        monkeypatch.delenv("USBS_KRON")
        scale = np.abs(want).max()
        assert np.max(np.abs(got - sparse)) <= 1e-13 * scale, (name, which, k)


def test_kron_gram_epilogue_cost_quad():
    """cost_quad = sym(V^T C V) (problem.py:284-286) through the Kronecker path."""
    from paper_2312_11801_b200 import runtime
    p = CASES["C3"]
    v, _ = np.linalg.qr(np.random.default_rng(3).standard_normal((p.n, 20)))
    dp = runtime.DeviceProblem(p)
    g = dp.rt.empty(20, 20)
    dp.apply(0, dp.rt.upload(v), gram=g)
    want = O.cost_gram(p, v)
    np.testing.assert_allclose(dp.rt.download(g), want, rtol=1e-12, atol=1e-13 * np.abs(want).max())


def test_non_kron_problems_are_not_detected():
    from paper_2312_11801_b200 import runtime
    assert runtime.kron_structure(inst.baseline_config("C1").problem) is None
    p = CASES["qap5"]
    cost = p.cost.tolil()
    cost[3, 7] = cost[3, 7] * 1.5  # breaks the product structure
    assert runtime.kron_structure(dataclasses.replace(p, cost=cost.tocsr(), kron_factors=None)) is None
