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
    if warm is not None and getattr(warm, "dev", None) is not None:
        wp = C.c_void_p(ptr(warm.dev))
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
