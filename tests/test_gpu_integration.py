"""The drop-in boundary exercised the way a reference caller would use it:

* the ``LinOp`` protocol (eigsolve.py:25-36): ``DeviceLinOp.matvec`` on the
  strided column views ``lanczos_top`` passes (``q[:, j]`` of a C-order
  (n, m+1) basis, eigsolve.py:126), ``matmat`` / ``apply_block`` on
  non-contiguous blocks -- and the oracle's own Lanczos (the reference
  algorithm line by line) driving a ``DeviceLinOp``;
* INTEGRATION.md section 3 executed: the oracle's outer loop (the
  reference's solve restated) with ``slack_op`` / ``lanczos`` rebound to the
  device versions, against the unpatched oracle;
* psi_value (subqp.py:546-549) on the device and the reference's
  monotonicity of psi across the alternating half steps
  (test_subqp.py:376-409) on the device alternating maximisation;
* ipm_quad warm-started from a host state with the reference's IpmState
  fields (subqp.py:112-119) behaves like the device state it was read from;
* records handed to a callback own their m-vectors (later iterations do not
  overwrite them).
"""
from __future__ import annotations

from types import SimpleNamespace

import numpy as np
import pytest

from helpers import mixed40, random_graph
from oracle import usbs_cpu as O
from paper_2312_11801_b200 import instances as inst

pytestmark = pytest.mark.gpu


def test_linop_protocol_on_strided_views():
    from paper_2312_11801_b200 import eigen, runtime
    p = inst.baseline_config("C1").problem
    y = np.random.default_rng(5).standard_normal(p.m) * 1e-3
    dp = runtime.DeviceProblem(p)
    op = eigen.dual_slack_operator(dp, y)
    z = O.slack_op(p, y)
    rng = np.random.default_rng(6)
    q = rng.standard_normal((p.n, 33))            # C order: q[:, j] is strided by 33 doubles
    for j in (0, 7, 32):
        v = q[:, j]
        assert not v.flags["C_CONTIGUOUS"]
        np.testing.assert_allclose(op.matvec(v), z.matvec(v), rtol=1e-13, atol=1e-13)
    blk = q[:, 3:14:2]                              # non-contiguous n x 6 block
    np.testing.assert_allclose(op.matmat(blk), z.block(blk), rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(op.apply_block(blk), z.block(blk), rtol=1e-13, atol=1e-13)
    rev = q[::-1, :4][::-1]                         # negative strides
    np.testing.assert_allclose(op.matmat(rev), z.block(rev), rtol=1e-13, atol=1e-13)
    assert op.dim == p.n


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_reference_lanczos_drives_device_linop(name):
    """The oracle's lanczos_top (eigsolve.py:83-181 restated) calls only
    dim/matvec of its operator: with a DeviceLinOp it runs the same Krylov
    recurrence with device SpMVs (restarts and matvecs identical)."""
    from paper_2312_11801_b200 import eigen, runtime
    p = inst.baseline_config(name).problem
    y = np.random.default_rng(8).standard_normal(p.m) * 1e-3
    dp = runtime.DeviceProblem(p)
    ref = O.lanczos(O.slack_op(p, y), 10, seed=0)
    mix = O.lanczos(eigen.dual_slack_operator(dp, y), 10, seed=0)
    assert mix.restarts == ref.restarts and mix.matvecs == ref.matvecs
    np.testing.assert_allclose(mix.eigenvalues, ref.eigenvalues, rtol=1e-12)


def test_integration_section3_rebinding(monkeypatch):
    """rebind the module-level dual_slack_operator
    and lanczos_top of the (restated) reference loop to the device and run
    it; the trajectory matches the unpatched loop to rounding in its first
    iterations and keeps the same step decisions."""
    from paper_2312_11801_b200 import eigen, runtime
    p = inst.maxcut_problem(random_graph(120, 0.1, 4))
    cfg = O.Config(k_c=6, k_p=1, sketch_rank=4, max_iters=8, seed=0)
    ref = []
    O.solve(p, cfg, callback=ref.append)

    dps = {}
    host_lanczos = O.lanczos

    def device_slack_operator(prob, y):
        dp = dps.get(id(prob)) or dps.setdefault(id(prob), runtime.DeviceProblem(prob))
        return eigen.dual_slack_operator(dp, y)

    def device_lanczos_top(op, k_c, inner_iters=32, max_restarts=10, tol=None, seed=0):
        if not isinstance(op, eigen.DeviceLinOp):  # cold start's host LinOp over prob.cost
            return host_lanczos(op, k_c, inner_iters, max_restarts, tol, seed)
        r = eigen.lanczos_top(op, k_c, inner_iters, max_restarts, tol, seed)
        return O.Eig(r.eigenvalues, r.eigenvectors, r.residuals, r.converged, r.restarts, r.ritz_history,
                     r.matvecs)

    monkeypatch.setattr(O, "slack_op", device_slack_operator)
    monkeypatch.setattr(O, "lanczos", device_lanczos_top)
    got = []
    O.solve(p, cfg, callback=got.append)
    assert len(got) == len(ref)
    for a, b in zip(got[:4], ref[:4]):
        assert a.step == b.step
        assert abs(a.f_cand - b.f_cand) <= 1e-8 * max(1.0, abs(b.f_cand))
        assert abs(a.lam_cand - b.lam_cand) <= 1e-8 * max(1.0, abs(b.lam_cand))
        assert a.lanczos_matvecs == b.lanczos_matvecs


def test_psi_value_matches_reference_formula():
    from paper_2312_11801_b200 import subproblem as Q
    from paper_2312_11801_b200.runtime import DeviceProblem
    p = mixed40()
    rng = np.random.default_rng(2)
    y, a_x, nu = rng.standard_normal(p.m), rng.standard_normal(p.m), -np.abs(rng.standard_normal(p.m))
    c_x, rho = 0.37, 0.05
    w = p.b + nu - a_x
    want = c_x + w @ y - (w @ w) / (2 * rho)   # subqp.py:546-549
    got = Q.psi_value(DeviceProblem(p), y, rho, c_x, a_x, nu)
    assert abs(got - want) <= 1e-12 * (1 + abs(want))
    assert abs(Q.psi_value(p, y, rho, c_x, a_x, nu) - want) <= 1e-12 * (1 + abs(want))


def test_psi_monotone_across_half_steps_device():
    """test_subqp.py:376-409 on the device alternating maximisation: with a
    nonzero aggregate (one model update with random directions), psi never
    decreases across the IPM and the nu half steps."""
    from paper_2312_11801_b200 import solver as S
    p = mixed40()
    cfg = S.SolverConfig(k_c=4, k_p=0, rho=0.1, max_iters=1)
    ds = S.DeviceSolver(p, cfg)
    st = ds.cold_start()
    rng = np.random.default_rng(11)
    y = ds.rt.upload(np.abs(rng.standard_normal(p.m)) * 0.05)
    model = st.model
    ds.alternating_max(model, y, ds.rt.zeros(p.m))
    vecs, _ = np.linalg.qr(rng.standard_normal((p.n, model.k)))
    k = model.k
    ds.eng.vec(S.N.VOP_AXPBY, k * k, x=ds.st_q[:k * k], s0=p.alpha, out=ds.s_act.view(-1))
    tr0 = model.stats.trace
    has_eta = tr0 > 0
    eta_act = (p.alpha * float(ds.res_q[3].item()) / tr0) if has_eta else 0.0
    model, pending = ds.model_update(model, eta_act, ds.rt.upload(vecs[:, :model.k_c]), tag=1)
    ds.residuals(y, 0.0, 0.0, S.AggregateStats(0.0, 0.0, ds.ax), pending=pending, model=model)
    assert model.stats.trace > 0
    vals = []
    ds.alternating_max(model, y, ds.rt.zeros(p.m), max_passes=8, tol=-1.0, psi_trace=vals)
    assert len(vals) == 16
    tol = 1e-8 * (1.0 + max(abs(v) for v in vals))
    assert all(b >= a - tol for a, b in zip(vals, vals[1:])), vals


def _quad(rng, k):
    d = k * (k + 1) // 2
    a = rng.standard_normal((d + 2, d))
    z = rng.standard_normal(d + 2)
    return SimpleNamespace(quad_ss=a.T @ a / (d + 2), quad_s_eta=a.T @ z / (d + 2), quad_eta=float(z @ z / (d + 2)),
                           lin_s=rng.standard_normal(d), lin_eta=float(rng.standard_normal()), has_eta=True, k=k)


def test_ipm_warm_state_from_host_fields():
    """A warm state given with the reference's IpmState fields (host arrays)
    warm-starts exactly like the device state it was read from."""
    from paper_2312_11801_b200 import subproblem as Q
    rng = np.random.default_rng(17)
    for _ in range(5):
        c = _quad(rng, int(rng.integers(2, 6)))
        first = Q.ipm_quad(c)
        c.lin_s = c.lin_s + 0.02 * rng.standard_normal(c.lin_s.shape)
        dev_warm = Q.ipm_quad(c, warm=first.state)
        st = first.state
        host = SimpleNamespace(s_mat=st.s_mat.copy(), t_mat=st.t_mat.copy(), eta=st.eta, zeta=st.zeta,
                               omega=st.omega, mu=st.mu, has_eta=True)
        host_warm = Q.ipm_quad(c, warm=host)
        assert host_warm.newton_iters == dev_warm.newton_iters
        np.testing.assert_array_equal(host_warm.s_opt, dev_warm.s_opt)
    with pytest.raises(TypeError):
        Q.ipm_quad(c, warm=SimpleNamespace(s_mat=np.eye(2)))


def test_callback_records_own_their_vectors():
    """IterationInfo / model records keep their values after later
    iterations (buffers were reused)."""
    from paper_2312_11801_b200 import solver as S
    p = mixed40()
    cfg = S.SolverConfig(k_c=4, k_p=1, sketch_rank=4, max_iters=6, seed=0)
    recs, snap = [], []

    def cb(info):
        recs.append(info)
        snap.append((info.y.copy(), info.y_cand.copy(), info.nu_cand.copy(), info.primal.constr_image.copy(),
                     info.model.stats.constr_image.copy()))

    S.solve(p, cfg, callback=cb)
    for info, (y, yc, nu, img, mimg) in zip(recs, snap):
        np.testing.assert_array_equal(info.y, y)
        np.testing.assert_array_equal(info.y_cand, yc)
        np.testing.assert_array_equal(info.nu_cand, nu)
        np.testing.assert_array_equal(info.primal.constr_image, img)
        np.testing.assert_array_equal(info.model.stats.constr_image, mimg)
