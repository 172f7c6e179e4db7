"""Standalone device orthonormalize / Nystrom sketch (linalg.py) against the
oracle restatements of symlin.orthonormalize and sketch.py."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import cuda_ok
from helpers import random_graph
from oracle import usbs_cpu as O
from paper_2312_11801_b200 import instances as inst

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


def _proj(q):
    return q @ q.T


@pytest.mark.parametrize("case", ["full", "dependent", "tiny"])
def test_orthonormalize_matches_oracle(case):
    from paper_2312_11801_b200 import linalg as L
    rng = np.random.default_rng(3)
    a = rng.standard_normal((300, 9))
    if case == "dependent":
        a[:, 4] = a[:, 1] - 2 * a[:, 2]
        a[:, 7] = 0.0
    if case == "tiny":
        a[:, 5] = a[:, 0] + 1e-10 * rng.standard_normal(300)  # residual below the CholQR cut-over
    q = L.orthonormalize(a)
    qo = O.gs_pivoted(a)
    assert q.shape == qo.shape
    np.testing.assert_allclose(q.T @ q, np.eye(q.shape[1]), atol=1e-12)
    # the 'tiny' column's direction is a 1e-10-relative residual: any two
    # Gram-Schmidt orders agree on it only to ~eps |a| / |residual| ~ 1e-6
    np.testing.assert_allclose(_proj(q), _proj(qo), atol=1e-6 if case == "tiny" else 1e-9)


def test_orthonormalize_errors():
    from paper_2312_11801_b200 import linalg as L
    from paper_2312_11801_b200.errors import EmptyBasisError
    with pytest.raises(EmptyBasisError):
        L.orthonormalize(np.zeros((50, 3)))
    with pytest.raises(EmptyBasisError):
        L.orthonormalize(np.zeros((50, 0)))


def test_sketch_update_and_reconstruct_match_oracle():
    from paper_2312_11801_b200 import linalg as L
    rng = np.random.default_rng(5)
    n, r, k = 400, 8, 5
    s = L.sketch_init(n, r, 17)
    so = O.sketch_new(n, r, 17)
    np.testing.assert_array_equal(s.psi(), so.psi)
    for step in range(3):
        v, _ = np.linalg.qr(rng.standard_normal((n, k)))
        qm, _ = np.linalg.qr(rng.standard_normal((k, k)))
        lams = rng.random(k)
        eta = 0.7
        s = L.sketch_update(s, eta, v, qm, lams)
        so = O.sketch_apply(so, eta, v @ qm, lams)
        np.testing.assert_allclose(s.sketch_mat, so.p, rtol=1e-12, atol=1e-12 * np.abs(so.p).max())
    u, lam = L.reconstruct(s)
    uo, lamo = O.sketch_factor(so)
    np.testing.assert_allclose(lam, lamo, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(u @ np.diag(lam) @ u.T, uo @ np.diag(lamo) @ uo.T, atol=1e-9 * lamo.max())
    with pytest.raises(ValueError):
        L.sketch_update(s, -1.0, v, qm, lams)
    with pytest.raises(ValueError):
        L.sketch_update(s, 1.0, v, qm, -lams)


@pytest.mark.parametrize("kappa", [1e2, 1e6])
def test_thin_svd_device_vs_lapack(kappa):
    """Exit-time thin SVD of a tall factor on the device (CholQR2 + the c x c
    SVD on the host, solver.thin_svd_device) against LAPACK on the whole
    matrix: singular values to rounding, U orthonormal, each singular
    vector equal up to sign."""
    from paper_2312_11801_b200 import solver as S
    from paper_2312_11801_b200.engine import Engine
    from paper_2312_11801_b200.runtime import DeviceProblem
    rng = np.random.default_rng(5)
    n, c = 100_000, 10
    qa, _ = np.linalg.qr(rng.standard_normal((n, c)))
    qb, _ = np.linalg.qr(rng.standard_normal((c, c)))
    sv = np.logspace(0, -np.log10(kappa), c)
    b = (qa * sv) @ qb.T
    dp = DeviceProblem(inst.maxcut_problem(random_graph(50, 0.2, 1)))
    eng = Engine(dp)
    u, s = S.thin_svd_device(eng, dp.rt.upload(b))
    u0, s0, _ = np.linalg.svd(b, full_matrices=False)
    np.testing.assert_allclose(s, s0, rtol=1e-10, atol=1e-15 * s0[0])
    assert np.abs(u.T @ u - np.eye(c)).max() <= 1e-12
    np.testing.assert_allclose(np.abs(np.sum(u * u0, axis=0)), np.ones(c), atol=1e-9)
