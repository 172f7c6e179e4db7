"""CPU oracle for the USBS per-iteration hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) may import it.  The product path
(``paper_2312_11801_b200``) never imports anything under ``oracle/``.

It restates, in plain numpy/scipy, the algorithm of the reference package
``specbundle`` 0.1.0 (``/root/reference/pkg/src/specbundle``) for the path
named by BASELINE.json's north star: penalised dual -> dual-slack operator ->
thick-restart Lanczos, the low-rank primal bookkeeping, the k x k
interior-point subproblem and the Nystrom sketch.  Each function cites the
reference ``file:line`` it follows.  Floating-point operations are issued in
the reference's order so the restatement reproduces the reference bit for bit
on the same numpy/scipy build; that is pinned by ``tests/test_oracle_golden.py``
against fixtures that ``oracle/make_golden.py`` records by running the
reference itself (parity pinned).

Third-party arithmetic at this boundary (not under /root/reference; the
reference leaves the versions unpinned, pkg/pyproject.toml:10-13): numpy 2.3.5
/ scipy 1.18.1 / OpenBLAS 0.3.30 in this image -- scipy.sparse ``_sparsetools``
CSR SpMV, LAPACK syevd/potrf/getrf, PCG64 and legacy MT19937 streams.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np
import scipy.linalg
import scipy.sparse as sp

SQRT2 = math.sqrt(2.0)


class NumericError(RuntimeError):
    pass


class ConditioningError(RuntimeError):
    pass


class EmptyBasisError(ValueError):
    pass


class StepFailureError(RuntimeError):
    pass


# ---------------------------------------------------------------------------
# symmetric vectorisation helpers (symlin.py:45-212)

_TRI: dict = {}


def tri_idx(k: int):
    """(row, col, weight) of svec order: lower triangle column-major,
    sqrt(2) off the diagonal (symlin.py:57-69)."""
    if k not in _TRI:
        r, c = np.triu_indices(k)
        _TRI[k] = (c.copy(), r.copy(), np.where(c == r, 1.0, SQRT2))
    return _TRI[k]


def svec(a):
    a = np.asarray(a, dtype=float)
    i, j, w = tri_idx(a.shape[0])
    return a[i, j] * w


def smat(v):
    v = np.asarray(v, dtype=float)
    k = int((math.isqrt(8 * v.shape[0] + 1) - 1) // 2)
    i, j, w = tri_idx(k)
    out = np.zeros((k, k))
    x = v / w
    out[i, j] = x
    out[j, i] = x
    return out


def svec_eye(k: int):
    return svec(np.eye(k))


_UMAT: dict = {}


def _umat(k: int):
    """vec -> svec compression matrix (symlin.py:109-130)."""
    if k not in _UMAT:
        i, j, _ = tri_idx(k)
        u = np.zeros((i.size, k * k))
        for p, (a, b) in enumerate(zip(i.tolist(), j.tolist())):
            if a == b:
                u[p, b * k + a] = 1.0
            else:
                u[p, b * k + a] = 1.0 / SQRT2
                u[p, a * k + b] = 1.0 / SQRT2
        _UMAT[k] = u
    return _UMAT[k]


def symm_kron(g, h):
    """0.5 U (g (x) h + h (x) g) U^T (symlin.py:133-145)."""
    u = _umat(g.shape[0])
    return 0.5 * u @ (np.kron(g, h) + np.kron(h, g)) @ u.T


def eigh_desc(s):
    """small_eigh (symlin.py:193-198): symmetrise, LAPACK eigh, descending."""
    s = np.asarray(s, dtype=float)
    s = 0.5 * (s + s.T)
    lam, vec = np.linalg.eigh(s)
    return lam[::-1].copy(), vec[:, ::-1].copy()


def chol_solve(m, rhs):
    """solve_spd (symlin.py:201-212)."""
    try:
        f = scipy.linalg.cho_factor(np.asarray(m, dtype=float), lower=True, check_finite=False)
    except (scipy.linalg.LinAlgError, np.linalg.LinAlgError) as exc:
        raise ConditioningError(str(exc)) from exc
    return scipy.linalg.cho_solve(f, np.asarray(rhs, dtype=float), check_finite=False)


def is_pd(m) -> bool:
    try:
        scipy.linalg.cho_factor(m, lower=True, check_finite=False)
        return True
    except (scipy.linalg.LinAlgError, np.linalg.LinAlgError):
        return False


def gs_pivoted(cols, drop_tol: float = 1e-12):
    """orthonormalize (symlin.py:148-190): column-pivoted Gram-Schmidt, two
    projections per pick, drop below drop_tol * max column norm."""
    a = np.array(cols, dtype=float)
    if a.ndim == 1:
        a = a[:, None]
    if a.size == 0:
        raise EmptyBasisError("no input columns")
    top = float(np.max(np.linalg.norm(a, axis=0)))
    if top == 0.0:
        raise EmptyBasisError("all input columns are zero")
    cut = drop_tol * top
    work = a.copy()
    live = list(range(a.shape[1]))
    out = []
    while live:
        nr = np.linalg.norm(work[:, live], axis=0)
        p = int(np.argmax(nr))
        if nr[p] <= cut:
            break
        col = live.pop(p)
        q = work[:, col]
        if out:
            b = np.column_stack(out)
            q = q - b @ (b.T @ q)
        nq = np.linalg.norm(q)
        if nq <= cut:
            continue
        q = q / nq
        out.append(q)
        if live:
            rest = work[:, live]
            work[:, live] = rest - np.outer(q, q @ rest)
    if not out:
        raise EmptyBasisError("all input columns are numerically dependent")
    return np.column_stack(out)


# ---------------------------------------------------------------------------
# constraint operators (problem.py:144-243) dispatched on the data layout


def _is_entries(cons) -> bool:
    return hasattr(cons, "idx") and hasattr(cons, "rows")


def _eff(cons):
    return np.where(cons.rows == cons.cols, 1.0, 2.0) * cons.vals


def image_lowrank(cons, v, s):
    """A(V S V^T) (problem.py:151-152, 200-203)."""
    if not _is_entries(cons):
        return np.einsum("ij,jk,ik->i", v, s, v)
    mid = v[cons.rows] @ s
    val = np.einsum("ej,ej->e", mid, v[cons.cols])
    return np.bincount(cons.idx, weights=val * _eff(cons), minlength=cons.m)


def image_factor(cons, u, lams):
    """A(U diag(lams) U^T) (problem.py:154-155, 205-208)."""
    if not _is_entries(cons):
        return (u * u) @ lams
    mid = u[cons.rows] * lams[None, :]
    val = np.einsum("ej,ej->e", mid, u[cons.cols])
    return np.bincount(cons.idx, weights=val * _eff(cons), minlength=cons.m)


def adjoint_csr(cons, y, n):
    """A*(y) as CSR (problem.py:160-161, 214-220)."""
    if not _is_entries(cons):
        return sp.diags(y)
    data = y[cons.idx] * cons.vals
    off = cons.rows != cons.cols
    r = np.concatenate([cons.rows, cons.cols[off]])
    c = np.concatenate([cons.cols, cons.rows[off]])
    d = np.concatenate([data, data[off]])
    return sp.coo_matrix((d, (r, c)), shape=(n, n)).tocsr()


def adjoint_gram(cons, y, v, n):
    """V^T A*(y) V (problem.py:166-167, 225-227)."""
    if not _is_entries(cons):
        return v.T @ (v * y[:, None])
    g = v.T @ (adjoint_csr(cons, y, n) @ v)
    return 0.5 * (g + g.T)


def compressed(cons, v):
    """Rows svec(V^T A_i V) (problem.py:169-173, 229-239)."""
    k = v.shape[1]
    i, j, w = tri_idx(k)
    if not _is_entries(cons):
        return v[:, i] * v[:, j] * w[None, :]
    g = v[cons.rows][:, :, None] * v[cons.cols][:, None, :]
    g = g + g.transpose(0, 2, 1)
    g[cons.rows == cons.cols] *= 0.5
    g *= cons.vals[:, None, None]
    part = g[:, i, j] * w[None, :]
    out = np.zeros((cons.m, i.size))
    np.add.at(out, cons.idx, part)
    return out


def cost_gram(prob, v):
    """cost_quad (problem.py:284-286)."""
    g = v.T @ (prob.cost @ v)
    return 0.5 * (g + g.T)


def cost_ip(prob, u, lams) -> float:
    """cost_factor_ip (problem.py:288-289)."""
    return float(np.einsum("ij,ij->j", prob.cost @ u, u) @ lams)


def _ineq(prob):
    return np.flatnonzero(np.asarray(prob.ineq_mask, dtype=bool))


def proj_k(z, prob):
    """problem.py:292-298."""
    out = np.asarray(prob.b, dtype=float).copy()
    ii = _ineq(prob)
    if ii.size:
        out[ii] = np.minimum(z[ii], prob.b[ii])
    return out


def proj_n(z, prob):
    """problem.py:301-308."""
    out = np.zeros_like(np.asarray(prob.b, dtype=float))
    ii = _ineq(prob)
    if ii.size:
        out[ii] = np.minimum(z[ii], 0.0)
    return out


# ---------------------------------------------------------------------------
# Lanczos (eigsolve.py:25-181)


@dataclass(frozen=True)
class Op:
    dim: int
    matvec: Callable
    matmat: Optional[Callable] = None

    def block(self, b):
        if self.matmat is not None:
            return self.matmat(b)
        return np.column_stack([self.matvec(b[:, j]) for j in range(b.shape[1])])


@dataclass
class Eig:
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray
    residuals: np.ndarray
    converged: bool
    restarts: int
    ritz_history: list = field(default_factory=list)
    matvecs: int = 0


def slack_op(prob, y) -> Op:
    """dual_slack_operator (problem.py:311-314): Z = C - A*(y) as CSR."""
    z = (prob.cost - adjoint_csr(prob.constraints, y, prob.n)).tocsr()
    return Op(prob.n, lambda v: z @ v, lambda b: z @ b)


def start_vector(n, seed, counter):
    """_seeded_unit (eigsolve.py:49-52): PCG64 default_rng([seed, counter])."""
    g = np.random.default_rng([int(seed) & 0xFFFFFFFF, counter])
    v = g.standard_normal(n)
    return v / np.linalg.norm(v)


def _reseed(q, used, seed, counter):
    """_fresh_direction (eigsolve.py:55-63)."""
    for a in range(8):
        v = start_vector(q.shape[0], seed, counter + a + 1)
        v -= q[:, :used] @ (q[:, :used].T @ v)
        nv = np.linalg.norm(v)
        if nv > 1e-8:
            return v / nv
    return None


def lanczos(op: Op, k_c, inner_iters=32, max_restarts=10, tol=None, seed=0) -> Eig:
    """lanczos_top (eigsolve.py:83-181)."""
    n = op.dim
    if k_c < 1:
        raise ValueError("k_c must be at least 1")
    m = max(int(inner_iters), k_c + 1, 2)
    if k_c >= n or inner_iters >= n or m >= n:
        z = op.block(np.eye(n))  # eigsolve.py:66-80
        if not np.all(np.isfinite(z)):
            raise NumericError("matvec returned non-finite values")
        lam, vec = eigh_desc(0.5 * (z + z.T))
        k = min(k_c, n)
        return Eig(lam[:k], vec[:, :k], np.zeros(k), True, 0, [float(lam[0])], n)
    tol = 1e-9 if tol is None else tol
    q = np.zeros((n, m + 1))
    h = np.zeros((m + 1, m + 1))
    q[:, 0] = start_vector(n, seed, 0)
    ell, ctr, hist, conv, restarts, mv = 0, 0, [], False, 0, 0
    theta, ymat, res = np.zeros(m), np.eye(m), np.full(m, np.inf)
    for cyc in range(max_restarts + 1):
        for j in range(ell, m):
            w = np.asarray(op.matvec(q[:, j]), dtype=float)
            mv += 1
            if not np.all(np.isfinite(w)):
                raise NumericError("matvec returned non-finite values")
            c = q[:, : j + 1].T @ w
            w = w - q[:, : j + 1] @ c
            c2 = q[:, : j + 1].T @ w
            w = w - q[:, : j + 1] @ c2
            c += c2
            h[: j + 1, j] = c
            h[j, : j + 1] = c
            beta = float(np.linalg.norm(w))
            scale = max(1.0, float(np.max(np.abs(c))) if c.size else 0.0)
            if beta <= 1e-13 * scale:
                ctr += 16
                f = _reseed(q, j + 1, seed, ctr)
                q[:, j + 1] = 0.0 if f is None else f
                h[j + 1, j] = h[j, j + 1] = 0.0
            else:
                q[:, j + 1] = w / beta
                h[j + 1, j] = h[j, j + 1] = beta
        theta, ymat = eigh_desc(h[:m, :m])
        res = np.abs(h[m, m - 1] * ymat[m - 1, :])
        hist.append(float(theta[0]))
        if np.all(res[:k_c] <= tol * (1.0 + abs(float(theta[0])))):
            conv = True
            break
        if cyc == max_restarts:
            break
        ell = max(1, min(k_c + 3, m - 2))
        kept = q[:, :m] @ ymat[:, :ell]
        nxt = q[:, m].copy()
        q[:, :ell] = kept
        q[:, ell] = nxt
        h[:, :] = 0.0
        h[:ell, :ell] = np.diag(theta[:ell])
        restarts += 1
    return Eig(theta[:k_c].copy(), q[:, :m] @ ymat[:, :k_c], res[:k_c].copy(), conv,
               restarts, hist, mv)


# ---------------------------------------------------------------------------
# Nystrom sketch (sketch.py:25-111)


def psi_matrix(n, r, seed):
    """make_test_matrix (sketch.py:25-27): legacy MT19937 standard normals."""
    return np.random.RandomState(int(seed) & 0x7FFFFFFF).standard_normal((n, r))


@dataclass
class Sketch:
    n: int
    r: int
    seed: int
    p: np.ndarray
    psi: np.ndarray


def sketch_new(n, r, seed) -> Sketch:
    if not 1 <= r <= n:
        raise ValueError(f"sketch rank {r} must lie in [1, {n}]")
    return Sketch(n, r, int(seed), np.zeros((n, r)), psi_matrix(n, r, seed))


def sketch_apply(s: Sketch, eta, f, lams) -> Sketch:
    """sketch_update with Q = I (sketch.py:58-74, bundle.py:124-126)."""
    if eta < 0:
        raise ValueError("eta must be nonnegative")
    lams = np.asarray(lams, dtype=float)
    if np.any(lams < -1e-12 * max(1.0, float(np.max(np.abs(lams), initial=0.0)))):
        raise ValueError("update eigenvalues must be nonnegative")
    fac = f @ np.eye(f.shape[1])
    p = eta * s.p + (fac * lams[None, :]) @ (fac.T @ s.psi)
    return Sketch(s.n, s.r, s.seed, p, s.psi)


def sketch_factor(s: Sketch):
    """reconstruct (sketch.py:77-111)."""
    p = s.p
    npn = float(np.linalg.norm(p))
    if npn == 0.0:
        u = np.zeros((s.n, s.r))
        u[: s.r, : s.r] = np.eye(s.r)
        return u, np.zeros(s.r)
    shift = np.sqrt(s.n) * np.finfo(float).eps * npn
    ps = p + shift * s.psi
    core = s.psi.T @ ps
    core = 0.5 * (core + core.T)
    try:
        ch = np.linalg.cholesky(core)
        half = scipy.linalg.solve_triangular(ch, ps.T, lower=True).T
    except np.linalg.LinAlgError:
        lam, qm = np.linalg.eigh(core)
        keep = lam > max(lam.max(initial=0.0), 0.0) * 1e-14
        if not np.any(keep):
            u = np.zeros((s.n, s.r))
            u[: s.r, : s.r] = np.eye(s.r)
            return u, np.zeros(s.r)
        half = ps @ (qm[:, keep] / np.sqrt(lam[keep])[None, :])
    u, sv, _ = np.linalg.svd(half, full_matrices=False)
    return u, np.maximum(sv ** 2 - shift, 0.0)


# ---------------------------------------------------------------------------
# interior-point subproblem (subqp.py:60-448)


@dataclass
class IpmOpts:
    mu_tol: float = 1e-11
    kkt_tol: float = 1e-6
    max_newton: int = 100
    step_frac: float = 0.99
    backtrack: float = 0.8
    min_step: float = 1e-12
    max_step_failures: int = 6
    warm_blend: float = 0.2


@dataclass
class Coeffs:
    """QuadCoeffs / EvalCoeffs (subqp.py:60-108); Q = 0 for the eval problem."""
    quad_ss: np.ndarray
    quad_s_eta: np.ndarray
    quad_eta: float
    lin_s: np.ndarray
    lin_eta: float
    has_eta: bool
    k: int
    cost_quad: Optional[np.ndarray] = None
    compressed: Optional[np.ndarray] = None


def linear_coeffs(lin_s, lin_eta, has_eta, k) -> Coeffs:
    d = k * (k + 1) // 2
    return Coeffs(np.zeros((d, d)), np.zeros(d), 0.0, lin_s, lin_eta, has_eta, k)


@dataclass
class IpState:
    s_mat: np.ndarray
    eta: float
    t_mat: np.ndarray
    zeta: float
    omega: float
    mu: float
    has_eta: bool

    @property
    def k(self):
        return self.s_mat.shape[0]

    def slack(self):
        return 1.0 - float(np.trace(self.s_mat)) - self.eta

    def compl(self):
        c = float(np.sum(self.s_mat * self.t_mat)) + self.omega * self.slack()
        if self.has_eta:
            c += self.eta * self.zeta
        return c

    def pairs(self):
        return self.k + (2 if self.has_eta else 1)

    def interior(self):
        if self.omega <= 0 or self.slack() <= 0:
            return False
        if self.has_eta and (self.eta <= 0 or self.zeta <= 0):
            return False
        return is_pd(self.s_mat) and is_pd(self.t_mat)


@dataclass
class IpResult:
    s_opt: np.ndarray
    eta_opt: float
    value: float
    state: IpState
    newton_iters: int
    exact: bool


def _centre(k, has_eta) -> IpState:
    """_cold_state (subqp.py:184-197)."""
    c = 1.0 / (2.0 * (k + (2 if has_eta else 1)))
    st = IpState(c * np.eye(k), c if has_eta else 0.0, np.eye(k), 1.0 if has_eta else 0.0,
                 1.0, 0.0, has_eta)
    st.mu = st.compl() / (2.0 * st.pairs())
    return st


def _value(q: Coeffs, s, eta):
    """_objective (subqp.py:200-207)."""
    v = float(0.5 * s @ (q.quad_ss @ s) + q.lin_s @ s)
    if q.has_eta:
        v += float(eta * (q.quad_s_eta @ s) + 0.5 * eta ** 2 * q.quad_eta + eta * q.lin_eta)
    return v


def _grad(q: Coeffs, st: IpState):
    """_stationarity (subqp.py:210-219)."""
    s, t, vi = svec(st.s_mat), svec(st.t_mat), svec_eye(q.k)
    f1 = q.quad_ss @ s + q.lin_s - t + st.omega * vi
    f2 = 0.0
    if q.has_eta:
        f1 = f1 + st.eta * q.quad_s_eta
        f2 = float(q.quad_s_eta @ s + st.eta * q.quad_eta + q.lin_eta - st.zeta + st.omega)
    return f1, f2


@dataclass
class Dir:
    ds: np.ndarray
    deta: float
    dt: np.ndarray
    dzeta: float
    domega: float


def newton_step(q: Coeffs, st: IpState, mu) -> Dir:
    """newton_direction (subqp.py:222-265)."""
    vi = svec_eye(q.k)
    t = svec(st.t_mat)
    si = np.linalg.inv(st.s_mat)
    si = 0.5 * (si + si.T)
    e = symm_kron(st.t_mat, si)
    f1, f2 = _grad(q, st)
    sig = st.slack()
    rc = mu / st.omega - sig
    rd = mu * svec(si) - t
    k1 = sig / st.omega
    if not q.has_eta:
        ds = chol_solve(q.quad_ss + e + np.outer(vi, vi) / k1, -f1 + rd - (rc / k1) * vi)
        return Dir(ds, 0.0, rd - e @ ds, 0.0, (rc + vi @ ds) / k1)
    re = mu / st.eta - st.zeta
    k2 = st.zeta / st.eta + q.quad_eta
    c = k1 * k2 + 1.0
    g = q.quad_s_eta
    mat = q.quad_ss + e - (np.outer(g, k1 * g + vi) + np.outer(vi, g - k2 * vi)) / c
    rhs = g * ((rc + k1 * (f2 - re)) / c) + vi * ((f2 - re - k2 * rc) / c) - f1 + rd
    ds = chol_solve(mat, rhs)
    deta = -(rc + k1 * (f2 - re) + (k1 * g + vi) @ ds) / c
    return Dir(ds, deta, rd - e @ ds, re - (st.zeta / st.eta) * deta,
               -f2 + re - g @ ds - k2 * deta)


def step_length(st: IpState, d: Dir, o: IpmOpts) -> float:
    """line_search_feasible (subqp.py:294-343)."""
    if not (np.all(np.isfinite(d.ds)) and np.all(np.isfinite(d.dt)) and np.isfinite(d.deta)
            and np.isfinite(d.dzeta) and np.isfinite(d.domega)):
        raise StepFailureError("non-finite direction")
    lim = []
    sc = [(st.omega, d.domega)]
    if st.has_eta:
        sc += [(st.eta, d.deta), (st.zeta, d.dzeta)]
    for x, dx in sc:
        if dx < 0:
            lim.append(-x / dx)
    sig = st.slack()
    dsig = -(svec_eye(st.k) @ d.ds + d.deta)
    if dsig < 0:
        lim.append(-sig / dsig)
    delta = min(1.0, o.step_frac * min(lim)) if lim else 1.0
    dsm, dtm = smat(d.ds), smat(d.dt)
    while delta >= o.min_step:
        ok = is_pd(st.s_mat + delta * dsm) and is_pd(st.t_mat + delta * dtm)
        if ok:
            if st.omega + delta * d.domega <= 0 or sig + delta * dsig <= 0:
                ok = False
            if st.has_eta and (st.eta + delta * d.deta <= 0 or st.zeta + delta * d.dzeta <= 0):
                ok = False
        if ok:
            return delta
        delta *= o.backtrack
    raise StepFailureError("no strictly feasible step above minimum")


def ipm(q: Coeffs, warm: Optional[IpState] = None, o: Optional[IpmOpts] = None) -> IpResult:
    """_ipm_solve (subqp.py:353-435)."""
    o = o or IpmOpts()
    st = None
    if warm is not None and warm.k == q.k and warm.has_eta == q.has_eta and warm.interior():
        lam = o.warm_blend
        c0 = _centre(q.k, q.has_eta)
        st = IpState((1 - lam) * warm.s_mat + lam * c0.s_mat, (1 - lam) * warm.eta + lam * c0.eta,
                     (1 - lam) * warm.t_mat + lam * c0.t_mat, (1 - lam) * warm.zeta + lam * c0.zeta,
                     (1 - lam) * warm.omega + lam * c0.omega, 0.0, q.has_eta)
        st.mu = st.compl() / (2.0 * st.pairs())
    if st is None:
        st = _centre(q.k, q.has_eta)
    mu = st.mu
    scale = 1.0 + max(float(np.max(np.abs(q.lin_s))) if q.lin_s.size else 0.0, abs(q.lin_eta),
                      float(np.max(np.abs(q.quad_ss))) if q.quad_ss.size else 0.0,
                      float(np.max(np.abs(q.quad_s_eta))) if q.quad_s_eta.size else 0.0,
                      abs(q.quad_eta))
    exact, fails, it = False, 0, 0
    for it in range(1, o.max_newton + 1):
        f1, f2 = _grad(q, st)
        sres = max(float(np.max(np.abs(f1))), abs(f2))
        ach = st.compl() / (2.0 * st.pairs())
        if mu < o.mu_tol and ach < o.mu_tol and sres <= o.kkt_tol * scale:
            exact = True
            it -= 1
            break
        try:
            d = newton_step(q, st, mu)
            delta = step_length(st, d, o)
        except (ConditioningError, StepFailureError):
            fails += 1
            if fails > o.max_step_failures:
                break
            mu = max(mu * 10.0, 10.0 * o.mu_tol)
            st.mu = mu
            continue
        fails = 0
        st.s_mat = st.s_mat + delta * smat(d.ds)
        st.t_mat = st.t_mat + delta * smat(d.dt)
        st.omega += delta * d.domega
        if q.has_eta:
            st.eta += delta * d.deta
            st.zeta += delta * d.dzeta
        gam = 1.0 if delta <= 0.2 else 0.5 - 0.4 * delta ** 2  # barrier_update 346-350
        mu = min(st.mu, gam * (st.compl() / (2.0 * st.pairs())))
        st.mu = mu
    return IpResult(st.s_mat.copy(), st.eta if q.has_eta else 0.0, _value(q, svec(st.s_mat), st.eta),
                    st, it, exact)


def eval_coeffs(prob, basis, stats, y) -> Coeffs:
    """assemble_eval_coeffs (subqp.py:455-468)."""
    a = prob.alpha
    sq = adjoint_gram(prob.constraints, y, basis, prob.n) - cost_gram(prob, basis)
    lin_s = a * svec(sq)
    tr = stats.trace
    if tr > 0.0:
        return linear_coeffs(lin_s, a / tr * float(y @ stats.constr_image - stats.cost_ip), True,
                             basis.shape[1])
    return linear_coeffs(lin_s, 0.0, False, basis.shape[1])


def quad_coeffs(prob, basis, stats, y, nu, rho, base: Optional[Coeffs] = None) -> Coeffs:
    """assemble_quad_coeffs (subqp.py:471-527)."""
    a = prob.alpha
    tr = stats.trace
    has_eta = tr > 0.0
    if base is None:
        cm = compressed(prob.constraints, basis)
        qss = (a ** 2 / rho) * (cm.T @ cm)
        d = basis.shape[1] * (basis.shape[1] + 1) // 2
        if has_eta:
            ai = stats.constr_image
            qse = (a ** 2 / (rho * tr)) * (cm.T @ ai)
            qe = (a ** 2 / (rho * tr ** 2)) * float(ai @ ai)
        else:
            qse, qe = np.zeros(d), 0.0
        cq = cost_gram(prob, basis)
    else:
        cm, qss, qse, qe, cq = base.compressed, base.quad_ss, base.quad_s_eta, base.quad_eta, base.cost_quad
    w = y - (prob.b + nu) / rho
    lin_s = a * (cm.T @ w - svec(cq))
    lin_eta = a / tr * float(stats.constr_image @ w - stats.cost_ip) if has_eta else 0.0
    return Coeffs(qss, qse, qe, lin_s, lin_eta, has_eta, basis.shape[1], cq, cm)


@dataclass
class AltResult:
    eta: float
    s_mat: np.ndarray
    nu: np.ndarray
    a_x: np.ndarray
    c_x: float
    tr_x: float
    passes: int
    exact: bool
    newton: list = field(default_factory=list)


def alternate(prob, basis, stats, y, rho, o=None, max_passes=50, tol=1e-8, nu0=None) -> AltResult:
    """alternating_max (subqp.py:552-614)."""
    o = o or IpmOpts()
    a = prob.alpha
    tr = stats.trace
    has_eta = tr > 0.0
    nu = proj_n(nu0, prob) if nu0 is not None else np.zeros(prob.m)
    warm, base, exact = None, None, True
    bn = float(np.linalg.norm(prob.b))
    has_ineq = _ineq(prob).size > 0
    eta_act, s_act, a_x, newton = 0.0, np.zeros((basis.shape[1],) * 2), np.zeros(prob.m), []
    passes = 0
    for passes in range(1, max_passes + 1):
        base = quad_coeffs(prob, basis, stats, y, nu, rho, base)
        r = ipm(base, warm, o)
        warm = r.state
        newton.append(r.newton_iters)
        exact = exact and r.exact
        s_act = a * r.s_opt
        eta_act = (a * r.eta_opt / tr) if has_eta else 0.0
        a_x = eta_act * stats.constr_image + image_lowrank(prob.constraints, basis, s_act)
        nxt = proj_n(a_x + rho * y - prob.b, prob)
        done = (not has_ineq) or (np.linalg.norm(nxt - nu) <= tol * (1.0 + bn))
        nu = nxt
        if done:
            break
    c_x = eta_act * stats.cost_ip + float(np.sum(base.cost_quad * s_act))
    tr_x = eta_act * tr + float(np.trace(s_act))
    return AltResult(eta_act, s_act, nu, a_x, c_x, tr_x, passes, exact, newton)


# ---------------------------------------------------------------------------
# outer loop (bundle.py:64-529)


@dataclass
class Config:
    """SolverConfig (bundle.py:64-91)."""
    rho: float = 0.01
    beta: float = 0.25
    k_c: int = 10
    k_p: int = 1
    eps: float = 1e-3
    sketch_rank: int = 0
    max_iters: int = 1000
    max_time: Optional[float] = None
    seed: int = 0
    inner_iters: int = 32
    max_restarts: int = 10
    lanczos_tol: Optional[float] = None
    linf_check: bool = False
    ipm: IpmOpts = field(default_factory=IpmOpts)


@dataclass
class Stats:
    trace: float
    cost_ip: float
    constr_image: np.ndarray

    def copy(self):
        return Stats(self.trace, self.cost_ip, self.constr_image.copy())


@dataclass
class Dense:
    """ExplicitStore (bundle.py:104-117)."""
    xbar: np.ndarray

    def update(self, eta, f, lams):
        self.xbar = eta * self.xbar + (f * lams[None, :]) @ f.T

    def factorize(self):
        lam, vec = eigh_desc(self.xbar)
        keep = lam > max(lam.max(initial=0.0), 0.0) * 1e-12
        if not np.any(keep):
            return np.eye(self.xbar.shape[0], 1), np.zeros(1)
        return vec[:, keep], lam[keep]


@dataclass
class Sketched:
    """SketchStore (bundle.py:120-129)."""
    sk: Sketch

    def update(self, eta, f, lams):
        self.sk = sketch_apply(self.sk, eta, f, lams)

    def factorize(self):
        return sketch_factor(self.sk)


@dataclass
class Model:
    basis: np.ndarray
    stats: Stats
    k_c: int
    k_p: int
    store: object


@dataclass
class Resid:
    rel_subopt: float
    rel_infeas: float
    linf_infeas: float
    dual_gap: float
    dual_feas: float

    def converged(self, eps, linf=False):
        ok = self.rel_subopt <= eps and self.rel_infeas <= eps and self.dual_feas <= eps
        return ok and (self.linf_infeas <= eps if linf else True)


@dataclass
class State:
    y: np.ndarray
    nu: np.ndarray
    f_y: Optional[float]
    lam_y: Optional[float]
    model: Model
    descent_steps: int = 0
    null_steps: int = 0
    iterations: int = 0
    last_primal: Optional[Stats] = None
    residuals: Optional[Resid] = None
    status: Optional[str] = None


@dataclass
class IterRecord:
    t: int
    elapsed: float
    step: str
    f_y: float
    f_cand: float
    model_val: float
    y_cand: np.ndarray
    nu_cand: np.ndarray
    residuals: Resid
    primal: Stats
    eta: float
    lam_cand: float
    alt_passes: int
    newton: list
    lanczos_matvecs: int
    lanczos_restarts: int


def penalised(prob, y, cfg: Config, k_c):
    """penalized_obj (bundle.py:212-236)."""
    ii = _ineq(prob)
    if ii.size and np.min(y[ii]) < 0:
        return np.inf, None
    eig = lanczos(slack_op(prob, y), k_c, cfg.inner_iters, cfg.max_restarts, cfg.lanczos_tol, cfg.seed)
    return prob.alpha * max(float(eig.eigenvalues[0]), 0.0) + float(prob.b @ y), eig


def candidate(y, nu, a_x, b, rho, ineq_idx):
    """candidate_iterate (bundle.py:239-255)."""
    out = y - (b - a_x) / rho
    if ineq_idx.size:
        sub = out[ineq_idx]
        out[ineq_idx] = np.where(nu[ineq_idx] < 0.0, 0.0, np.maximum(sub, 0.0))
    return out


def complete(basis, k, seed, tag):
    """_completion_columns (bundle.py:264-282)."""
    n = basis.shape[0]
    cols = [basis]
    have, att = basis.shape[1], 0
    while have < k:
        v = np.random.default_rng([int(seed) & 0xFFFFFFFF, 0x5EED, tag, att]).standard_normal(n)
        cur = np.column_stack(cols) if len(cols) > 1 else cols[0]
        v -= cur @ (cur.T @ v)
        nv = np.linalg.norm(v)
        att += 1
        if nv < 1e-10:
            continue
        cols.append((v / nv)[:, None])
        have += 1
    out = np.column_stack(cols) if len(cols) > 1 else cols[0]
    return out[:, :k]


def fold(model: Model, eta, s_next, new_vecs, prob, seed=0, tag=0) -> Model:
    """model_update (bundle.py:285-341)."""
    kp = model.k_p
    lam, q = eigh_desc(s_next)
    lc = np.maximum(lam[kp:], 0.0)
    f = model.basis @ q[:, kp:]
    st = model.stats
    ns = Stats(eta * st.trace + float(lc.sum()), eta * st.cost_ip + cost_ip(prob, f, lc),
               eta * st.constr_image + image_factor(prob.constraints, f, lc))
    if model.store is not None:
        model.store.update(eta, f, lc)
    if kp == 0:
        nb = np.asarray(new_vecs, dtype=float)
    else:
        try:
            nb = gs_pivoted(np.column_stack([model.basis @ q[:, :kp], new_vecs]))
        except EmptyBasisError:
            nb = np.zeros((model.basis.shape[0], 0))
    k = model.basis.shape[1]
    if nb.shape[1] < k:
        nb = complete(np.zeros((model.basis.shape[0], 0)) if nb.shape[1] == 0 else nb, k, seed, tag)
    return Model(nb, ns, model.k_c, kp, model.store)


def residuals(prob, y, f_y, lam_y, primal: Stats) -> Resid:
    """compute_residuals (bundle.py:344-372)."""
    ax = primal.constr_image
    diff = ax - proj_k(ax, prob)
    bn = float(np.linalg.norm(prob.b))
    cx = primal.cost_ip
    return Resid((cx - f_y) / (1.0 + abs(cx)), float(np.linalg.norm(diff)) / (1.0 + bn),
                 float(np.max(np.abs(diff))) if diff.size else 0.0,
                 abs(float(prob.b @ y) - cx), lam_y)


def dims(prob, cfg):
    kc = min(cfg.k_c, prob.n)
    return kc, min(cfg.k_p, prob.n - kc)


def sketch_seed(seed) -> int:
    """_derived_seeds (bundle.py:385-387)."""
    return int(np.random.SeedSequence(int(seed)).generate_state(2)[0])


def cold(prob, cfg: Config) -> State:
    """cold_start (bundle.py:390-423)."""
    kc, kp = dims(prob, cfg)
    eig = lanczos(Op(prob.n, lambda v: prob.cost @ v, lambda b: prob.cost @ b), kc,
                  cfg.inner_iters, cfg.max_restarts, cfg.lanczos_tol, cfg.seed)
    basis = complete(eig.eigenvectors, kc + kp, cfg.seed, 0)
    st = Stats(0.0, 0.0, np.zeros(prob.m))
    if cfg.sketch_rank > 0:
        store = Sketched(sketch_new(prob.n, min(cfg.sketch_rank, prob.n), sketch_seed(cfg.seed)))
    else:
        store = Dense(np.zeros((prob.n, prob.n)))
    return State(np.zeros(prob.m), np.zeros(prob.m), None, None, Model(basis, st, kc, kp, store),
                 last_primal=st.copy())


def solve(prob, cfg: Config, init: Optional[State] = None, callback=None):
    """solve (bundle.py:426-529); returns (state, (factor, lams))."""
    state = init if init is not None else cold(prob, cfg)
    model = state.model
    t0 = time.monotonic()
    y = state.y
    if state.f_y is None or state.lam_y is None:
        f_y, eig = penalised(prob, y, cfg, model.k_c)
        if not np.isfinite(f_y):
            raise ValueError("initial dual point violates the sign constraints")
        lam_y = float(eig.eigenvalues[0])
    else:
        f_y, lam_y = state.f_y, state.lam_y
    primal = state.last_primal if state.last_primal is not None else model.stats.copy()
    res = residuals(prob, y, f_y, lam_y, primal)
    state.f_y, state.lam_y, state.residuals = f_y, lam_y, res
    status = "converged" if res.converged(cfg.eps, cfg.linf_check) else None
    ii = _ineq(prob)
    t = 0
    inner_nu = state.nu.copy()
    while status is None:
        if t >= cfg.max_iters or (cfg.max_time is not None and time.monotonic() - t0 > cfg.max_time):
            status = "budget"
            break
        alt = alternate(prob, model.basis, model.stats, y, cfg.rho, cfg.ipm, nu0=inner_nu)
        inner_nu = alt.nu
        yc = candidate(y, alt.nu, alt.a_x, prob.b, cfg.rho, ii)
        f_c, eig_c = penalised(prob, yc, cfg, model.k_c)
        ev = ipm(eval_coeffs(prob, model.basis, model.stats, yc), None, cfg.ipm)
        mval = float(prob.b @ yc) - ev.value
        accept = cfg.beta * (f_y - mval) <= f_y - f_c  # descent_test bundle.py:258-261
        if accept:
            y, f_y, lam_y = yc, f_c, float(eig_c.eigenvalues[0])
            state.nu = alt.nu
            state.descent_steps += 1
        else:
            state.null_steps += 1
        model = fold(model, alt.eta, alt.s_mat, eig_c.eigenvectors, prob, cfg.seed, t + 1)
        primal = Stats(alt.tr_x, alt.c_x, alt.a_x)
        res = residuals(prob, y, f_y, lam_y, primal)
        state.y, state.f_y, state.lam_y, state.model = y, f_y, lam_y, model
        state.last_primal, state.residuals, state.iterations = primal, res, t + 1
        if callback is not None:
            callback(IterRecord(t, time.monotonic() - t0, "descent" if accept else "null", f_y, f_c,
                                mval, yc, alt.nu, res, primal, alt.eta,
                                float(eig_c.eigenvalues[0]), alt.passes, alt.newton,
                                eig_c.matvecs, eig_c.restarts))
        t += 1
        if res.converged(cfg.eps, cfg.linf_check):
            status = "converged"
    state.status = status
    return state, (model.store.factorize() if model.store is not None else None)
