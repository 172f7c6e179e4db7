"""Device-path properties that the reference's own tests assert (SURVEY.md
section 4), restated against the B200 implementation:

* convergence invariants of seeded random MaxCut runs (test_acceptance.py
  criteria 2 and 10): converged status, dual feasibility by an independent
  dense eigensolve, infeasibility and gap bounds, monotone f(y), the model
  minorant and the trace budget at every iteration;
* the inequality path (criterion 6): clipped candidates stay nonnegative and
  complementary to the slack;
* bookkeeping (test_bundle.py:147-204): tracked statistics equal the dense
  shadow, the basis stays orthonormal;
* the sketch does not perturb the dual path (test_bundle.py:303-319);
* Nystrom sketch algebra (test_sketch.py): exact low-rank recovery, PSD,
  linearity;
* Lanczos (test_eigsolve.py, acceptance criterion 9): dense agreement over
  random matrices, monotone Ritz history, degenerate top eigenspace, budget
  reporting, defaults;
* the IPM exit certificate and warm starts (test_subqp.py:418-488).
"""
from __future__ import annotations

import inspect
from types import SimpleNamespace

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import cuda_ok
from helpers import mixed40, random_graph
from paper_2312_11801_b200 import instances as inst

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

EPS = 1e-3


def _solver():
    from paper_2312_11801_b200 import solver as S
    return S


# ---------------------------------------------------------------- solve
def test_convergence_invariants_random_maxcut():
    S = _solver()
    rng = np.random.default_rng(2024)
    for trial in range(8):
        n = int(rng.integers(30, 101))
        p = float(rng.uniform(0.08, 0.3))
        prob = inst.maxcut_problem(random_graph(n, p, trial))
        cfg = S.SolverConfig(rho=0.01, beta=0.25, k_c=10, k_p=1, eps=EPS, max_iters=3000, seed=trial)
        rows = []
        state, _ = S.solve(prob, cfg, callback=lambda i: rows.append(
            (i.f_y, i.model_val, i.f_cand, i.primal.trace)))
        assert state.status == "converged", trial
        z = prob.cost.toarray() - np.diag(state.y)
        assert float(np.linalg.eigvalsh(z).max()) <= EPS + 1e-10
        assert state.residuals.rel_infeas <= EPS
        c_x = state.last_primal.cost_ip
        b_y = float(prob.b @ state.y)
        assert abs(b_y - c_x) <= np.sqrt(EPS) * (1.0 + abs(c_x) + abs(b_y))
        f = [r[0] for r in rows]
        assert all(b <= a + 1e-12 for a, b in zip(f, f[1:]))
        for _, model_val, f_cand, trace in rows:
            assert model_val <= f_cand + 1e-8 * (1.0 + abs(f_cand))
            assert trace <= prob.alpha + 1e-9


def test_inequality_candidates_clipped_and_complementary():
    S = _solver()
    prob = mixed40()
    idx = np.flatnonzero(prob.ineq_mask)
    worst = {"sign": 0.0, "comp": 0.0}

    def cb(info):
        yc = info.y_cand
        worst["sign"] = min(worst["sign"], float(np.min(yc[idx])))
        worst["comp"] = max(worst["comp"], abs(float(yc @ info.nu_cand)))

    cfg = S.SolverConfig(rho=0.1, beta=0.25, k_c=5, k_p=1, eps=EPS, max_iters=60, seed=0)
    S.solve(prob, cfg, callback=cb)
    assert worst["sign"] >= 0.0
    assert worst["comp"] <= 1e-10


def test_statistics_track_dense_shadow():
    """The explicit store is the dense shadow X = sum of the updates; the
    tracked trace, <C, X> and diag(X) = A(X) must equal it at every
    iteration, and the basis must stay orthonormal."""
    S = _solver()
    prob = inst.maxcut_problem(random_graph(40, 0.2, 11))
    cfg = S.SolverConfig(k_c=4, k_p=2, sketch_rank=0, max_iters=25, eps=1e-12, seed=0)
    cost = prob.cost.toarray()
    checked = 0

    def cb(info):
        nonlocal checked
        x = info.model.store.xbar
        st = info.model.stats
        assert abs(st.trace - np.trace(x)) <= 1e-9
        assert abs(st.cost_ip - np.sum(cost * x)) <= 1e-9
        np.testing.assert_allclose(st.constr_image, np.diag(x), atol=1e-9)
        v = info.model.basis
        np.testing.assert_allclose(v.T @ v, np.eye(v.shape[1]), atol=1e-10)
        checked += 1

    S.solve(prob, cfg, callback=cb)
    assert checked == 25


def test_sketch_does_not_perturb_dual_path():
    S = _solver()
    prob = inst.maxcut_problem(random_graph(50, 0.15, 5))
    ys = {}
    for r in (0, 6):
        cfg = S.SolverConfig(sketch_rank=r, eps=1e-3, max_iters=300, seed=1)
        st, _ = S.solve(prob, cfg)
        ys[r] = (st.iterations, st.y)
    assert ys[0][0] == ys[6][0]
    np.testing.assert_allclose(ys[6][1], ys[0][1], rtol=0, atol=1e-12)


# ---------------------------------------------------------------- sketch
def test_sketch_recovers_low_rank_exactly_and_is_linear():
    from paper_2312_11801_b200 import linalg as L
    rng = np.random.default_rng(7)
    n = 60
    for rank, r in ((1, 4), (3, 6)):
        f, _ = np.linalg.qr(rng.standard_normal((n, rank)))
        lams = np.sort(rng.uniform(0.5, 2.0, rank))[::-1]
        sk = L.sketch_update(L.sketch_init(n, r, seed=3), 0.0, f, np.eye(rank), lams)
        u, lam = L.reconstruct(sk)
        x = (f * lams) @ f.T
        xr = (u * lam) @ u.T
        assert np.all(lam >= 0.0)
        assert np.linalg.norm(xr - x) <= 1e-8 * np.linalg.norm(x)
    # linearity of the sketch in the tracked matrix
    f1, f2 = rng.standard_normal((n, 2)), rng.standard_normal((n, 3))
    l1, l2 = np.array([1.0, 0.5]), np.array([2.0, 0.3, 0.1])
    s0 = L.sketch_init(n, 5, seed=9)
    a = L.sketch_update(L.sketch_update(s0, 0.0, f1, np.eye(2), l1), 0.7, f2, np.eye(3), l2)
    b1 = L.sketch_update(s0, 0.0, f1, np.eye(2), l1)
    b2 = L.sketch_update(s0, 0.0, f2, np.eye(3), l2)
    np.testing.assert_allclose(a.sketch_mat, 0.7 * b1.sketch_mat + b2.sketch_mat, atol=1e-12)


# ---------------------------------------------------------------- Lanczos
def _op(cost):
    from paper_2312_11801_b200 import eigen
    from paper_2312_11801_b200.runtime import DeviceProblem
    n = cost.shape[0]
    prob = inst.Problem(n=n, m=n, cost=sp.csr_matrix(cost), constraints=inst.DiagonalFamily(n), b=np.ones(n),
                        ineq_mask=np.zeros(n, dtype=bool), alpha=1.0, scale_c=1.0, scale_x=1.0, sense=1)
    dp = DeviceProblem(prob)
    return eigen, eigen.dual_slack_operator(dp, np.zeros(n))


def test_lanczos_matches_dense_over_random_matrices():
    rng = np.random.default_rng(9)
    worst = 0.0
    for t in range(25):
        n = int(rng.integers(60, 200))
        a = sp.random(n, n, density=0.08, random_state=int(rng.integers(1 << 30)), format="csr")
        a = (a + a.T) * 0.5 + sp.diags(rng.standard_normal(n) * 0.1)
        eigen, op = _op(a.toarray())
        r = eigen.lanczos_top(op, 5, max_restarts=60, seed=t)
        want = float(np.linalg.eigvalsh(a.toarray()).max())
        worst = max(worst, abs(r.eigenvalues[0] - want) / max(1.0, abs(want)))
    assert worst <= 1e-8


def test_lanczos_history_monotone_and_budget_reported():
    rng = np.random.default_rng(3)
    n = 300
    a = sp.random(n, n, density=0.05, random_state=4, format="csr")
    a = ((a + a.T) * 0.5).toarray()
    eigen, op = _op(a)
    r = eigen.lanczos_top(op, 10, inner_iters=32, max_restarts=2, tol=1e-15, seed=0)
    h = list(r.ritz_history)
    assert all(b >= a_ - 1e-12 * max(1.0, abs(a_)) for a_, b in zip(h, h[1:]))
    assert not r.converged and r.restarts == 2


def test_lanczos_degenerate_top_eigenspace():
    n = 120
    d = np.linspace(-1.0, 1.0, n)
    d[:3] = 5.0  # a threefold top eigenvalue
    eigen, op = _op(np.diag(d))
    r = eigen.lanczos_top(op, 3, seed=2)
    np.testing.assert_allclose(r.eigenvalues[:3], 5.0, atol=1e-10)
    v = r.eigenvectors
    # the three vectors span e_0, e_1, e_2
    assert np.linalg.norm(v[3:, :]) <= 1e-6
    np.testing.assert_allclose(v.T @ v, np.eye(3), atol=1e-10)


def test_lanczos_defaults_match_reference():
    from paper_2312_11801_b200 import eigen
    sig = inspect.signature(eigen.lanczos_top)
    assert sig.parameters["inner_iters"].default == 32
    assert sig.parameters["max_restarts"].default == 10
    assert sig.parameters["seed"].default == 0


# ---------------------------------------------------------------- IPM
def _random_quad(rng, k):
    d = k * (k + 1) // 2
    a = rng.standard_normal((d + 2, d))
    z = rng.standard_normal(d + 2)
    return SimpleNamespace(quad_ss=a.T @ a / (d + 2), quad_s_eta=a.T @ z / (d + 2), quad_eta=float(z @ z / (d + 2)),
                           lin_s=rng.standard_normal(d), lin_eta=float(rng.standard_normal()), has_eta=True, k=k)


def _svec(x):
    k = x.shape[0]
    out = []
    for j in range(k):
        for i in range(j, k):
            out.append(x[i, j] * (1.0 if i == j else np.sqrt(2.0)))
    return np.array(out)


def test_ipm_exit_certificate():
    from paper_2312_11801_b200 import subproblem as Q
    rng = np.random.default_rng(31)
    for _ in range(10):
        k = int(rng.integers(2, 6))
        c = _random_quad(rng, k)
        res = Q.ipm_quad(c)
        assert res.exact
        st = res.state
        s_mat, t_mat = st.s_mat, st.t_mat
        scale = 1.0 + max(np.abs(c.lin_s).max(), abs(c.lin_eta), np.abs(c.quad_ss).max())
        s_vec = _svec(s_mat)
        f1 = c.quad_ss @ s_vec + st.eta * c.quad_s_eta + c.lin_s - _svec(t_mat) + st.omega * _svec(np.eye(k))
        f2 = c.quad_s_eta @ s_vec + st.eta * c.quad_eta + c.lin_eta - st.zeta + st.omega
        assert np.abs(f1).max() <= 1e-6 * scale
        assert abs(f2) <= 1e-6 * scale
        assert np.abs(s_mat @ t_mat).max() <= 1e-6 * scale
        assert st.eta * st.zeta <= 1e-6 * scale
        assert st.omega * (1.0 - np.trace(s_mat) - st.eta) <= 1e-6 * scale


def test_ipm_warm_start_beats_cold_in_aggregate():
    from paper_2312_11801_b200 import subproblem as Q
    rng = np.random.default_rng(123)
    wins = total = 0
    for _ in range(12):
        c = _random_quad(rng, int(rng.integers(2, 5)))
        warm = None
        for call in range(5):
            c.lin_s = c.lin_s + 0.02 * rng.standard_normal(c.lin_s.shape)
            c.lin_eta = c.lin_eta + 0.02 * float(rng.standard_normal())
            cold = Q.ipm_quad(c)
            w = Q.ipm_quad(c, warm=warm)
            if call > 0:
                total += 1
                wins += w.newton_iters <= cold.newton_iters
            warm = w.state
    assert wins / total >= 0.9


def test_warm_start_from_subgraph_saves_descent_steps():
    """Acceptance criterion 7 (test_acceptance.py:320-347): a state solved on
    the induced subgraph of the first 99 vertices, padded into the full
    graph, needs no more descent steps than a cold start in >= 4 of 5 runs."""
    S = _solver()
    from paper_2312_11801_b200 import state as ST
    wins = 0
    for seed in range(5):
        g = random_graph(100, 0.08, 900 + seed)
        keep = (g.eu < 99) & (g.ev < 99)
        sub = inst.Graph.from_arrays(99, g.eu[keep], g.ev[keep], g.ew[keep])
        prob, sub_prob = inst.maxcut_problem(g), inst.maxcut_problem(sub)
        cfg = S.SolverConfig(rho=0.01, beta=0.25, k_c=10, k_p=1, eps=1e-3, max_iters=3000, seed=seed)
        cold, _ = S.solve(prob, cfg)
        assert cold.status == "converged"
        sub_state, _ = S.solve(sub_prob, cfg)
        padded = ST.warm_start_pad(sub_state, prob, ST.Mapping(np.arange(99), np.arange(99)), sketch_seed=seed)
        warm, _ = S.solve(prob, cfg, init=padded)
        assert warm.status == "converged"
        wins += warm.descent_steps <= cold.descent_steps
    assert wins >= 4


def test_diagonal_fast_path_equals_generic_entries():
    """problem.py's diagonal family and the same constraints written as
    generic entries give the same device images and adjoints
    (test_problem.py:228-256)."""
    from paper_2312_11801_b200.constraints import DeviceConstraints
    rng = np.random.default_rng(12)
    n, k = 300, 7
    ent = SimpleNamespace(idx=np.arange(n), rows=np.arange(n), cols=np.arange(n), vals=np.ones(n))
    diag = DeviceConstraints(n, n, inst.DiagonalFamily(n))
    gen = DeviceConstraints(n, n, ent)
    v = rng.standard_normal((n, k))
    s = rng.standard_normal((k, k))
    s = s + s.T
    y = rng.standard_normal(n)
    np.testing.assert_allclose(diag.primal_image_lowrank(v, s), gen.primal_image_lowrank(v, s), rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(diag.adjoint_matvec(y, v), gen.adjoint_matvec(y, v), rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(diag.adjoint_inner_lowrank(y, v), gen.adjoint_inner_lowrank(y, v), rtol=1e-12,
                               atol=1e-12)
    # adjoint identity <A(X), y> = <X, A*(y)> for X = V S V^T
    lhs = float(gen.primal_image_lowrank(v, s) @ y)
    rhs = float(np.sum(s * gen.adjoint_inner_lowrank(y, v)))
    assert abs(lhs - rhs) <= 1e-10 * (1.0 + abs(lhs))
