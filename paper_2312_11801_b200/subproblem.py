"""Host-facing mirrors of subqp.ipm_quad / ipm_eval (subqp.py:438-448) that
run the single-CTA device IPM (csrc/usbs_ipm.cu).  Coefficient objects are
duck-typed (reference QuadCoeffs / EvalCoeffs or anything with the same
fields); numpy in, numpy out."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from ._native import check, ptr
from .runtime import runtime

__all__ = ["IpmState", "IpmResult", "ipm_quad", "ipm_eval"]


@dataclass
class IpmState:
    """IpmState (subqp.py:111-147) backed by the device state vector."""

    dev: object
    k: int

    def _h(self):
        return self.dev.cpu().numpy()

    @property
    def s_mat(self):
        return self._h()[: self.k * self.k].reshape(self.k, self.k)

    @property
    def t_mat(self):
        k = self.k
        return self._h()[k * k: 2 * k * k].reshape(k, k)

    @property
    def eta(self):
        return float(self._h()[2 * self.k * self.k])

    @property
    def zeta(self):
        return float(self._h()[2 * self.k * self.k + 1])

    @property
    def omega(self):
        return float(self._h()[2 * self.k * self.k + 2])

    @property
    def mu(self):
        return float(self._h()[2 * self.k * self.k + 3])


@dataclass
class IpmResult:
    s_opt: np.ndarray
    eta_opt: float
    value: float
    state: IpmState
    newton_iters: int
    exact: bool


def _opts(o):
    if o is None:
        return None
    return (C.c_double * 8)(o.mu_tol, o.kkt_tol, o.max_newton, o.step_frac, o.backtrack, o.min_step,
                            o.max_step_failures, o.warm_blend)


def _pack_warm(warm, k, sl):
    """A host warm state with the reference's fields (subqp.py:112-119:
    s_mat, t_mat, eta, zeta, omega, mu, has_eta) in the device state layout
    [S (k*k), T (k*k), eta, zeta, omega, mu, has_eta, k, valid]; the kernel
    applies the reference's feasibility check and 0.2 blend to it."""
    for f in ("s_mat", "t_mat", "eta", "zeta", "omega", "mu", "has_eta"):
        if not hasattr(warm, f):
            raise TypeError(f"warm state lacks {f!r} (expected a device IpmState or the reference's IpmState)")
    s_mat = np.asarray(warm.s_mat, dtype=float)
    t_mat = np.asarray(warm.t_mat, dtype=float)
    if s_mat.shape != (k, k) or t_mat.shape != (k, k):
        raise ValueError("warm state size does not match the coefficients")
    v = np.zeros(sl)
    kk = k * k
    v[:kk] = s_mat.reshape(-1)
    v[kk:2 * kk] = t_mat.reshape(-1)
    v[2 * kk:2 * kk + 7] = [float(warm.eta), float(warm.zeta), float(warm.omega), float(warm.mu),
                            1.0 if warm.has_eta else 0.0, float(k), 1.0]
    return v


def _solve(k, has_eta, quad_ss, quad_s_eta, quad_eta, lin_s, lin_eta, warm: Optional[IpmState], opts):
    rt = runtime()
    lib = rt.lib
    Q = rt.upload(quad_ss) if quad_ss is not None else None
    g = rt.upload(quad_s_eta) if (quad_s_eta is not None and has_eta) else None
    h = rt.upload(lin_s)
    scal = rt.upload(np.array([float(quad_eta), float(lin_eta)]))
    sl = int(lib.usbs_ipm_state_len(k))
    st = rt.zeros(sl)
    res = rt.zeros(8)
    wp = None
    if warm is not None:
        if getattr(warm, "dev", None) is not None:
            wp = C.c_void_p(ptr(warm.dev))
        else:
            warm_dev = rt.upload(_pack_warm(warm, k, sl))
            wp = C.c_void_p(ptr(warm_dev))
    check(lib.usbs_ipm_solve(rt.h, k, 1 if has_eta else 0, C.c_void_p(ptr(Q)) if Q is not None else None,
                             C.c_void_p(ptr(g)) if g is not None else None, C.c_void_p(ptr(h)),
                             C.c_void_p(ptr(scal)), wp, C.c_void_p(ptr(st)), C.c_void_p(ptr(res)), _opts(opts)),
          "ipm_solve")
    r = res.cpu().numpy()
    s = st.cpu().numpy()[: k * k].reshape(k, k).copy()
    return IpmResult(s, float(r[3]), float(r[0]), IpmState(st, k), int(r[1]), bool(r[2]))


def ipm_quad(coeffs, warm: Optional[IpmState] = None, opts=None) -> IpmResult:
    """Minimise the quadratic proximal objective over the budget set."""
    return _solve(int(coeffs.k), bool(coeffs.has_eta), np.asarray(coeffs.quad_ss, dtype=float),
                  np.asarray(coeffs.quad_s_eta, dtype=float), float(coeffs.quad_eta),
                  np.asarray(coeffs.lin_s, dtype=float), float(coeffs.lin_eta), warm, opts)


def ipm_eval(coeffs, opts=None) -> IpmResult:
    """Minimise the linear model objective over the budget set."""
    return _solve(int(coeffs.k), bool(coeffs.has_eta), None, None, 0.0, np.asarray(coeffs.lin_s, dtype=float),
                  float(coeffs.lin_eta), None, opts)


def psi_value(prob, y, rho: float, c_x: float, a_x, nu, engine=None) -> float:
    """psi_value (subqp.py:546-549): the proximal coupling objective of an
    (X, nu) pair at anchor y, c_x + <w, y> - ||w||^2 / (2 rho) with
    w = b + nu - a_x.  The two m-sized reductions run on the device
    (usbs_vec ops 10/11); y, a_x, nu may be device tensors or host arrays.
    ``prob`` is a DeviceProblem or any object with a ``b`` vector."""
    from . import _native as N
    from .engine import Engine
    from .runtime import DeviceProblem
    rt = runtime()
    dp = prob if isinstance(prob, DeviceProblem) else None
    eng = engine or (Engine(dp) if dp is not None else None)
    as_dev = (lambda v: v if hasattr(v, "data_ptr") else rt.upload(np.asarray(v, dtype=float)))
    b = dp.b if dp is not None else as_dev(prob.b)
    yd, ad, nd = as_dev(y), as_dev(a_x), as_dev(nu)
    red = rt.zeros(4)
    m = int(b.numel())
    lib = rt.lib
    h = eng.h if eng is not None else rt.h
    check(lib.usbs_vec(h, N.VOP_PSIWY, m, C.c_void_p(ptr(ad)), C.c_void_p(ptr(yd)), C.c_void_p(ptr(nd)),
                       C.c_void_p(ptr(b)), None, 0.0, 0.0, None, C.c_void_p(ptr(red[0:2]))), "vec")
    check(lib.usbs_vec(h, N.VOP_PSIWW, m, C.c_void_p(ptr(ad)), None, C.c_void_p(ptr(nd)), C.c_void_p(ptr(b)),
                       None, 0.0, 0.0, None, C.c_void_p(ptr(red[2:4]))), "vec")
    wy, ww = (float(v) for v in red.cpu().numpy()[[0, 2]])
    return float(c_x + wy - ww / (2.0 * float(rho)))
