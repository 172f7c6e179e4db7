"""The device constraint-bundle surface (constraints.DeviceConstraints, the
duck type of problem.py:144-243) against the oracle restatement, for the
diagonal family (MaxCut) and entry families (QAP, correlation, mixed)."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import cuda_ok
from helpers import mixed40, random_graph, random_qap
from oracle import usbs_cpu as O
from paper_2312_11801_b200 import instances as inst

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


def _problem(name):
    if name == "maxcut":
        return inst.maxcut_problem(random_graph(150, 0.08, 2))
    if name == "qap":
        return inst.qap_problem(random_qap(4, 3))
    if name == "corr":
        return inst.correlation_problem(*inst.knn_correlation(n=200, clusters=8, dim=8, knn=5, seed=4))
    return mixed40()


@pytest.mark.parametrize("name", ["maxcut", "qap", "corr", "mixed"])
def test_device_constraints_match_oracle(name):
    from paper_2312_11801_b200.constraints import device_constraints
    p = _problem(name)
    c = p.constraints
    dc = device_constraints(p)
    assert (dc.n, dc.m) == (p.n, p.m)
    rng = np.random.default_rng(7)
    k = 5
    v = rng.standard_normal((p.n, k))
    s = rng.standard_normal((k, k))
    s = s + s.T
    lams = rng.random(k)
    y = rng.standard_normal(p.m)
    x = rng.standard_normal((p.n, p.n))
    x = x + x.T

    def close(a, b, rtol=1e-11):
        np.testing.assert_allclose(a, b, rtol=rtol, atol=rtol * max(1.0, np.abs(b).max()))

    close(dc.primal_image_lowrank(v, s), O.image_lowrank(c, v, s))
    close(dc.primal_image_factor(v, lams), O.image_factor(c, v, lams))
    if hasattr(c, "idx"):
        eff = np.where(c.rows == c.cols, 1.0, 2.0) * c.vals
        want_dense = np.bincount(c.idx, weights=x[c.rows, c.cols] * eff, minlength=p.m)
    else:
        want_dense = np.diag(x)
    close(dc.primal_image_dense(x), want_dense)
    adj = O.adjoint_csr(c, y, p.n)
    np.testing.assert_allclose(dc.adjoint_matrix(y).toarray(), adj.toarray(), rtol=1e-14, atol=1e-14)
    close(dc.adjoint_matvec(y, v[:, 0]), adj @ v[:, 0])
    close(dc.adjoint_matvec(y, v), adj @ v)
    close(dc.adjoint_inner_lowrank(y, v), O.adjoint_gram(c, y, v, p.n), rtol=1e-10)
    close(dc.compressed_rows(v), O.compressed(c, v))
    want_fro = c.frob_norms() if hasattr(c, "frob_norms") else np.ones(p.m)
    np.testing.assert_allclose(dc.frob_norms(), want_fro, rtol=1e-15)
    if hasattr(c, "idx"):
        f = rng.random(p.m) + 0.5
        ds = dc.scaled(f)
        close(ds.primal_image_lowrank(v, s), O.image_lowrank(c.scaled(f), v, s))
