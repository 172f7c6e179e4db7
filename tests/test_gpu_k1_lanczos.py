"""GPU parity: K1 operator apply and the device Lanczos against the CPU
oracle (oracle/usbs_cpu.py, itself pinned bit-exact to the reference)."""
from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import cuda_ok
from helpers import load_npz, mixed40, random_graph, random_qap
from oracle import usbs_cpu as O
from paper_2312_11801_b200 import instances as inst

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

EPS = 2.0 ** -53


def dev():
    from paper_2312_11801_b200 import eigen, runtime
    return eigen, runtime


def dense_problem(a):
    """SdpProblem-like wrapper whose cost is the dense matrix a (diag constraints)."""
    n = a.shape[0]
    return inst.Problem(n=n, m=n, cost=sp.csr_matrix(a), constraints=inst.DiagonalFamily(n),
                        b=np.ones(n) / n, ineq_mask=np.zeros(n, bool), alpha=2.0, scale_c=1.0, scale_x=float(n))


def bound_check(got, want, z_abs, v_abs, rownnz, factor=8.0):
    """|dY| <= factor * (row nnz + 2) * eps * (|Z||V|)  (minimum slice)."""
    lim = factor * (rownnz[:, None] + 2) * EPS * (z_abs @ v_abs) + 1e-300
    err = np.abs(got - want)
    assert np.all(err <= lim), float(np.max(err / lim))


CASES = ["C1", "C2", "qap3", "mixed40", "C5s", "C4s"]


def case_problem(name):
    if name in ("C1", "C2"):
        return inst.baseline_config(name).problem
    if name == "qap3":
        return inst.qap_problem(random_qap(3, 1))
    if name == "mixed40":
        return mixed40()
    if name == "C5s":
        return inst.baseline_config("C5", small=True).problem
    if name == "C4s":
        return inst.baseline_config("C4", small=True).problem
    raise KeyError(name)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("k", [1, 11, 20])
def test_op_apply_matches_oracle(name, k):
    eigen, runtime = dev()
    p = case_problem(name)
    rng = np.random.default_rng(1234)
    y = rng.standard_normal(p.m) * 1e-3
    v, _ = np.linalg.qr(rng.standard_normal((p.n, k)))
    k = v.shape[1]
    dp = runtime.DeviceProblem(p)
    rt = dp.rt
    z = (p.cost - O.adjoint_csr(p.constraints, y, p.n)).tocsr()
    rownnz = np.diff(z.indptr)
    # Z V with the gram epilogue
    dp.assemble(rt.upload(y))
    V = rt.upload(v)
    g = rt.empty(k, k)
    out = rt.download(dp.apply(1, V, gram=g))
    want = z @ v
    bound_check(out, want, abs(z), np.abs(v), rownnz)
    gw = v.T @ want
    np.testing.assert_allclose(rt.download(g), 0.5 * (gw + gw.T), rtol=1e-12, atol=1e-14 * np.abs(gw).max())
    # C V (cost only) and sym(V^T C V) = cost_quad
    out_c = rt.download(dp.apply(0, V, gram=g))
    bound_check(out_c, p.cost @ v, abs(p.cost), np.abs(v), np.diff(p.cost.indptr))
    cq = O.cost_gram(p, v)
    np.testing.assert_allclose(rt.download(g), cq, rtol=1e-12, atol=1e-14 * max(1e-300, np.abs(cq).max()))


@pytest.mark.parametrize("name", ["C4s", "C5s", "mixed40"])
def test_spmm_grouped_gather_any_k_and_view(name, monkeypatch):
    """K1 for 2 <= k <= 15 (grouped 16-byte gathers, usbs_sparse.cu k_spmm_g):
    every group width (k = 2 .. 15), V a contiguous tensor, a strided view
    with an odd row stride (row starts alternate 8-byte parity) and an
    offset view (8-byte base: the launcher falls back to the half-warp
    kernel), within the dot-product bound and equal to the half-warp kernel
    up to summation order."""
    eigen, runtime = dev()
    p = case_problem(name)
    rng = np.random.default_rng(77)
    dp = runtime.DeviceProblem(p)
    rt = dp.rt
    c_abs = abs(p.cost)
    rownnz = np.diff(p.cost.indptr)
    for k in (2, 3, 5, 6, 7, 9, 11, 12, 15):
        v = rng.standard_normal((p.n, k))
        want = p.cost @ v
        big = rt.upload(np.zeros((p.n, k + 3)))
        view = big[:, 1:k + 1]  # 8-byte base offset: the launcher takes the half-warp kernel
        view.copy_(rt.upload(v))
        ldo = k + 2 if k % 2 else k + 3  # odd row stride: row starts alternate 8-byte parity
        big2 = rt.upload(np.zeros((p.n, ldo)))
        view2 = big2[:, :k]
        view2.copy_(rt.upload(v))
        for V in (rt.upload(v), view, view2):
            monkeypatch.delenv("USBS_SPMM_16X2", raising=False)
            got = rt.download(dp.apply(0, V))
            bound_check(got, want, c_abs, np.abs(v), rownnz)
            monkeypatch.setenv("USBS_SPMM_16X2", "1")
            ref = rt.download(dp.apply(0, V))
            bound_check(ref, want, c_abs, np.abs(v), rownnz)
            np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-13 * np.abs(want).max())
        monkeypatch.delenv("USBS_SPMM_16X2", raising=False)


def test_slack_pattern_holds_cost_bit_exact():
    """The uploaded cost values/columns equal prob.cost (bit-exact), checked
    through C e_j products on a few columns."""
    eigen, runtime = dev()
    p = inst.baseline_config("C1").problem
    dp = runtime.DeviceProblem(p)
    info = dp.info()
    assert info.nnz_c == p.cost.nnz
    cols = [0, 5, 399, 799]
    e = np.zeros((p.n, len(cols)))
    e[cols, range(len(cols))] = 1.0
    got = dp.rt.download(dp.apply(0, dp.rt.upload(e)))
    np.testing.assert_array_equal(got, p.cost.toarray()[:, cols])


def _projector_err(a, b):
    return np.linalg.norm(a @ a.T - b @ b.T)


@pytest.mark.parametrize("name", ["dense200", "dense300", "degenerate62"])
def test_lanczos_dense_golden(name):
    eigen, runtime = dev()
    z = load_npz("lanczos.npz")
    a = z[f"{name}/A"]
    kc, inner, rst, seed = (int(x) for x in z[f"{name}/args"])
    dp = runtime.DeviceProblem(dense_problem(a))
    r = eigen.lanczos_top(eigen.cost_operator(dp), kc, inner, rst, None, seed)
    ref_vals = z[f"{name}/vals"]
    scale = np.abs(ref_vals).max()
    assert np.max(np.abs(r.eigenvalues - ref_vals)) <= 1e-10 * scale
    vecs = r.eigenvectors
    np.testing.assert_allclose(vecs.T @ vecs, np.eye(kc), atol=1e-10)
    conv_ref, rst_ref = z[f"{name}/meta"]
    assert r.converged == bool(conv_ref)
    assert r.restarts == int(rst_ref)
    # leading eigenvalue vs dense eigvalsh (reference test_eigsolve.py:24-33)
    dense = np.linalg.eigvalsh(a)[::-1][:kc]
    if name != "dense300":
        np.testing.assert_allclose(r.eigenvalues, dense, atol=1e-8)
    if name == "degenerate62":
        assert _projector_err(vecs, z[f"{name}/vecs"]) <= 1e-6


def test_lanczos_c1_slack_vs_oracle():
    """C1 slack operator at the golden dual: eigenvalues and the Ritz-block
    projector against the reference/oracle result."""
    eigen, runtime = dev()
    z = load_npz("lanczos.npz")
    p = inst.baseline_config("C1").problem
    dp = runtime.DeviceProblem(p)
    op = eigen.dual_slack_operator(dp, z["c1/y"])
    r = eigen.lanczos_top(op, 10, seed=0)
    ref = z["c1/vals"]
    rel = np.abs(r.eigenvalues - ref) / np.abs(ref)
    assert rel[0] <= 1e-12, rel
    assert np.max(rel) <= 1e-6, rel
    assert r.restarts == int(z["c1/meta"][1])
    pe = _projector_err(r.eigenvectors, z["c1/vecs"])
    assert pe <= 1e-6, pe


@pytest.mark.parametrize("name", ["C2", "C5s", "C4s", "qap3"])
def test_lanczos_vs_oracle(name):
    eigen, runtime = dev()
    p = case_problem(name)
    y = np.random.default_rng(7).standard_normal(p.m) * 1e-3
    if p.ineq_mask.any():
        y[p.ineq_mask] = np.abs(y[p.ineq_mask])
    kc = 10
    ro = O.lanczos(O.slack_op(p, y), kc, seed=0)
    dp = runtime.DeviceProblem(p)
    r = eigen.lanczos_top(eigen.dual_slack_operator(dp, y), kc, seed=0)
    assert abs(r.eigenvalues[0] - ro.eigenvalues[0]) <= 1e-10 * max(1.0, abs(ro.eigenvalues[0]))
    assert r.restarts == ro.restarts
    assert r.matvecs == ro.matvecs
    np.testing.assert_allclose(r.eigenvalues, ro.eigenvalues, rtol=1e-5, atol=1e-9)


@pytest.mark.parametrize("name", ["C2", "C1", "C5s", "qap3"])
def test_lanczos_cluster_matches_grid(name, monkeypatch):
    """The cluster (Q in shared memory) and grid-wide kernels run the same
    recurrence: same restarts/matvecs, eigenvalues to rounding."""
    eigen, runtime = dev()
    p = case_problem(name)
    y = np.random.default_rng(11).standard_normal(p.m) * 1e-3
    if p.ineq_mask.any():
        y[p.ineq_mask] = np.abs(y[p.ineq_mask])
    dp_c = runtime.DeviceProblem(p)
    monkeypatch.setenv("USBS_LZ_CLUSTER", "0")
    dp_g = runtime.DeviceProblem(p)
    assert dp_g.lanczos_plan(32) == (0, 0)
    monkeypatch.delenv("USBS_LZ_CLUSTER")
    cs, rows = dp_c.lanczos_plan(32)
    if p.n >= 512:
        assert cs in (8, 16) and cs * rows >= p.n
    rc = eigen.lanczos_top(eigen.dual_slack_operator(dp_c, y), 10, seed=3)
    rg = eigen.lanczos_top(eigen.dual_slack_operator(dp_g, y), 10, seed=3)
    assert rc.restarts == rg.restarts and rc.matvecs == rg.matvecs
    np.testing.assert_allclose(rc.eigenvalues, rg.eigenvalues, rtol=1e-11, atol=1e-13)
    assert _projector_err(rc.eigenvectors, rg.eigenvectors) <= 1e-7


@pytest.mark.parametrize("cluster", [True, False])
def test_lanczos_breakdown_three_levels(cluster, monkeypatch):
    """Diagonal operator with 3 distinct values at n=3000: the Krylov space
    has dimension 3, so every cycle breaks down and reseeds (eigsolve.py:136-147)
    — on the cluster kernel this exercises the Q spill / host reseed / resume."""
    eigen, runtime = dev()
    n = 3000
    d = np.array([3.0, 2.0, 1.0])[np.arange(n) % 3]
    if not cluster:
        monkeypatch.setenv("USBS_LZ_CLUSTER", "0")
    dp = runtime.DeviceProblem(dense_problem(np.diag(d)))
    assert (dp.lanczos_plan(32)[0] > 0) == cluster
    r = eigen.lanczos_top(eigen.cost_operator(dp), 2, seed=0)
    ro = O.lanczos(O.Op(n, lambda v: d * v if v.ndim == 1 else d[:, None] * v), 2, seed=0)
    np.testing.assert_allclose(r.eigenvalues, ro.eigenvalues, atol=1e-10)
    assert r.converged == ro.converged
    assert r.matvecs == ro.matvecs


def test_lanczos_breakdown_diag_spike():
    """eigsolve breakdown path (reference test_eigsolve.py:11-15)."""
    eigen, runtime = dev()
    dp = runtime.DeviceProblem(dense_problem(np.diag([5.0, 1.0, 1.0, 1.0])))
    r = eigen.lanczos_top(eigen.cost_operator(dp), 1, inner_iters=3, seed=0)
    ro = O.lanczos(O.Op(4, lambda v: np.array([5.0, 1, 1, 1]) * v), 1, inner_iters=3, seed=0)
    assert r.eigenvalues[0] == pytest.approx(5.0, abs=1e-10)
    np.testing.assert_allclose(np.abs(r.eigenvectors[:, 0]), [1, 0, 0, 0], atol=1e-8)
    assert r.matvecs == ro.matvecs


def test_lanczos_breakdown_low_rank():
    """Rank-3 operator in n=60 forces repeated fresh directions."""
    eigen, runtime = dev()
    rng = np.random.default_rng(3)
    u, _ = np.linalg.qr(rng.standard_normal((60, 3)))
    a = (u * np.array([3.0, 2.0, 1.0])) @ u.T
    dp = runtime.DeviceProblem(dense_problem(a))
    r = eigen.lanczos_top(eigen.cost_operator(dp), 2, seed=0)
    ro = O.lanczos(O.Op(60, lambda v: a @ v, lambda b: a @ b), 2, seed=0)
    np.testing.assert_allclose(r.eigenvalues, ro.eigenvalues, atol=1e-10)
    assert r.converged == ro.converged


def test_lanczos_negative_definite_and_dense_fallback():
    eigen, runtime = dev()
    dp = runtime.DeviceProblem(dense_problem(-2.0 * np.eye(50)))
    r = eigen.lanczos_top(eigen.cost_operator(dp), 1, seed=0)
    assert r.eigenvalues[0] == pytest.approx(-2.0, abs=1e-10)
    a = np.random.default_rng(6).standard_normal((6, 6))
    a = 0.5 * (a + a.T)
    dp = runtime.DeviceProblem(dense_problem(a))
    r = eigen.lanczos_top(eigen.cost_operator(dp), 6, seed=0)
    np.testing.assert_allclose(r.eigenvalues, np.linalg.eigvalsh(a)[::-1], atol=1e-12)
    assert r.converged


def test_lanczos_nonfinite_raises():
    eigen, runtime = dev()
    from paper_2312_11801_b200.errors import NumericError
    a = np.eye(40)
    a[3, 3] = np.nan
    dp = runtime.DeviceProblem(dense_problem(a))
    with pytest.raises(NumericError):
        eigen.lanczos_top(eigen.cost_operator(dp), 1, seed=0)


def test_lanczos_determinism():
    eigen, runtime = dev()
    p = inst.baseline_config("C2").problem
    dp = runtime.DeviceProblem(p)
    y = np.random.default_rng(2).standard_normal(p.m) * 1e-3
    r1 = eigen.lanczos_top(eigen.dual_slack_operator(dp, y), 10, seed=7)
    r2 = eigen.lanczos_top(eigen.dual_slack_operator(dp, y), 10, seed=7)
    assert np.array_equal(r1.eigenvalues, r2.eigenvalues)
    assert np.array_equal(r1.eigenvectors, r2.eigenvectors)


@pytest.mark.parametrize("k", [1, 2, 11, 20, 32, 33])
def test_small_eigh_matches_lapack(k):
    eigen, runtime = dev()
    rng = np.random.default_rng(k)
    a = rng.standard_normal((k, k))
    a = a + a.T
    vals, vecs = eigen.small_eigh(a)
    lv, _ = O.eigh_desc(a)
    np.testing.assert_allclose(vals, lv, atol=1e-13 * max(1, np.abs(lv).max()))
    np.testing.assert_allclose(vecs @ np.diag(vals) @ vecs.T, 0.5 * (a + a.T), atol=1e-12 * np.abs(a).max())
    np.testing.assert_allclose(vecs.T @ vecs, np.eye(k), atol=1e-13)


def _star_problem(n=6000, hubs=(0, 2500), seed=9):
    """Graph with hub rows far above the SpMV tile (1024) and the grid-Lanczos
    segment (4096) sizes plus a random sparse rest: exercises the block-per-row
    paths of the fused SpMV and of the grid kernel's segments."""
    rng = np.random.default_rng(seed)
    eu, ev = [], []
    for h in hubs:
        leaves = rng.choice(n, size=4500, replace=False)
        leaves = leaves[leaves != h]
        eu += [h] * leaves.size
        ev += list(leaves)
    m = 20000
    a, b = rng.integers(0, n, m), rng.integers(0, n, m)
    eu += list(a)
    ev += list(b)
    g = inst.Graph.from_arrays(n, np.array(eu), np.array(ev), rng.choice([-1.0, 1.0], len(eu)))
    return inst.maxcut_problem(g)


@pytest.mark.parametrize("k", [1, 3, 11])
def test_op_apply_hub_rows(k):
    eigen, runtime = dev()
    p = _star_problem()
    assert np.diff(p.cost.indptr).max() > 4096
    rng = np.random.default_rng(2)
    y = rng.standard_normal(p.m) * 1e-3
    v, _ = np.linalg.qr(rng.standard_normal((p.n, k)))
    dp = runtime.DeviceProblem(p)
    dp.assemble(dp.rt.upload(y))
    out = dp.rt.download(dp.apply(1, dp.rt.upload(v)))
    z = (p.cost - O.adjoint_csr(p.constraints, y, p.n)).tocsr()
    bound_check(out, z @ v, abs(z), np.abs(v), np.diff(z.indptr))


@pytest.mark.parametrize("cluster", [True, False])
def test_lanczos_hub_rows(cluster, monkeypatch):
    """Grid kernel (hub rows above one segment, split across the nonzero
    partition) and cluster kernel against the oracle."""
    eigen, runtime = dev()
    if not cluster:
        monkeypatch.setenv("USBS_LZ_CLUSTER", "0")
    p = _star_problem()
    y = np.random.default_rng(4).standard_normal(p.m) * 1e-3
    dp = runtime.DeviceProblem(p)
    assert (dp.lanczos_plan(32)[0] > 0) == cluster
    r = eigen.lanczos_top(eigen.dual_slack_operator(dp, y), 8, seed=0)
    ro = O.lanczos(O.slack_op(p, y), 8, seed=0)
    assert abs(r.eigenvalues[0] - ro.eigenvalues[0]) <= 1e-10 * abs(ro.eigenvalues[0])
    assert r.restarts == ro.restarts and r.matvecs == ro.matvecs
    np.testing.assert_allclose(r.eigenvalues, ro.eigenvalues, rtol=1e-7, atol=1e-10)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_lanczos_halo_matches_dsmem_gather(name, monkeypatch):
    """The cluster kernel's two SpMV paths -- the per-step halo fetch and the
    DSMEM gather inside the row loop (USBS_LZ_HALO=0, the fallback when the
    halo does not fit) -- multiply the same operands in the same order: the
    whole call is bit-identical."""
    eigen, runtime = dev()
    p = case_problem(name)
    y = np.random.default_rng(12).standard_normal(p.m) * 1e-3
    dp_h = runtime.DeviceProblem(p)
    monkeypatch.setenv("USBS_LZ_HALO", "0")
    dp_g = runtime.DeviceProblem(p)
    assert dp_g.lanczos_plan(32)[0] > 0
    monkeypatch.delenv("USBS_LZ_HALO")
    assert dp_h.lanczos_plan(32)[0] > 0
    rh = eigen.lanczos_top(eigen.dual_slack_operator(dp_h, y), 10, seed=5)
    rg = eigen.lanczos_top(eigen.dual_slack_operator(dp_g, y), 10, seed=5)
    assert rh.restarts == rg.restarts and rh.matvecs == rg.matvecs
    np.testing.assert_array_equal(rh.eigenvalues, rg.eigenvalues)
    np.testing.assert_array_equal(rh.eigenvectors, rg.eigenvectors)
