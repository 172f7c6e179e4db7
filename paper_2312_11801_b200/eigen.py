"""Device eigensolver surface, mirroring specbundle.eigsolve
(eigsolve.py:25-181) and symlin.small_eigh (symlin.py:193-198).

``DeviceLinOp`` satisfies the reference ``LinOp`` protocol (dim, matvec,
matmat, apply_block) for host numpy callers while exposing the device
operator to :func:`lanczos_top`, which runs the whole thick-restart Lanczos
as one persistent sm_100a kernel (csrc/usbs_lanczos.cu).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native
from ._native import check, ptr
from .errors import NumericError
from .runtime import DeviceProblem, Runtime, runtime

__all__ = ["DeviceLinOp", "EigResult", "lanczos_top", "small_eigh", "dual_slack_operator", "cost_operator"]


@dataclass
class EigResult:
    """eigsolve.EigResult (eigsolve.py:39-46) + the device copy of the vectors."""

    eigenvalues: np.ndarray
    eigenvectors_dev: object  # torch (n, k_c), row-major
    residuals: np.ndarray
    converged: bool
    restarts: int
    ritz_history: list = field(default_factory=list)
    matvecs: int = 0

    @property
    def eigenvectors(self) -> np.ndarray:
        return self.eigenvectors_dev.cpu().numpy()


class DeviceLinOp:
    """LinOp-compatible view of M = C (which=0) or Z = C - A*(y) (which=1)."""

    def __init__(self, dprob: DeviceProblem, which: int):
        self.dprob = dprob
        self.which = int(which)
        self.dim = dprob.n

    def _run(self, block: np.ndarray) -> np.ndarray:
        rt = self.dprob.rt
        one = block.ndim == 1
        B = rt.upload(block.reshape(self.dim, -1))
        out = self.dprob.apply(self.which, B)
        res = rt.download(out)
        return res[:, 0].copy() if one else res

    def matvec(self, v):
        return self._run(np.asarray(v, dtype=float))

    def matmat(self, b):
        return self._run(np.asarray(b, dtype=float))

    def apply_block(self, block):
        return self.matmat(block)


def dual_slack_operator(dprob: DeviceProblem, y) -> DeviceLinOp:
    """problem.dual_slack_operator (problem.py:311-314): assembles Z on the
    device (y: numpy or device tensor)."""
    rt = dprob.rt
    y_dev = y if hasattr(y, "data_ptr") else rt.upload(np.asarray(y, dtype=float))
    dprob.assemble(y_dev)
    return DeviceLinOp(dprob, 1)


def cost_operator(dprob: DeviceProblem) -> DeviceLinOp:
    """LinOp of the cost alone (bundle.py:397)."""
    return DeviceLinOp(dprob, 0)


def lanczos_top(op: DeviceLinOp, k_c: int, inner_iters: int = 32, max_restarts: int = 10,
                tol: Optional[float] = None, seed: int = 0, out=None) -> EigResult:
    """Algebraically largest k_c Ritz pairs (eigsolve.py:83-181), on device.

    Same arguments, defaults, budget semantics and error behaviour
    (ValueError for k_c < 1, NumericError for a non-finite matvec).  Fresh
    directions after an invariant subspace use the reference's PCG64 stream
    (generated on the host through a callback)."""
    if not isinstance(op, DeviceLinOp):
        raise TypeError("lanczos_top on the device needs a DeviceLinOp (see dual_slack_operator)")
    if k_c < 1:
        raise ValueError("k_c must be at least 1")
    dp = op.dprob
    rt = dp.rt
    n = dp.n
    k_eff = min(k_c, n)
    vecs = out if out is not None else rt.empty(n, k_eff)
    v0 = rt.start_vector(n, seed)
    seed32 = int(seed) & 0xFFFFFFFF

    def fill(user, counter, dst, nn):
        try:
            g = np.random.default_rng([seed32, int(counter)])
            rt.h2d_ptr(int(dst), g.standard_normal(int(nn)))
            return 0
        except Exception:  # pragma: no cover - reported as USBS_ERR_CALLBACK
            return 1

    cb = _native.RNG_FILL(fill)
    vals = (C.c_double * max(k_c, 1))()
    res = (C.c_double * max(k_c, 1))()
    hist = (C.c_double * (max_restarts + 2))()
    conv, rst, nh, mv = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    st = rt.lib.usbs_lanczos_top(rt.h, dp.h, op.which, int(k_c), int(inner_iters), int(max_restarts),
                                 -1.0 if tol is None else float(tol), C.c_void_p(ptr(v0)), cb, None,
                                 vals, C.c_void_p(ptr(vecs)), vecs.stride(0), res, C.byref(conv), C.byref(rst),
                                 hist, C.byref(nh), C.byref(mv))
    check(st, "lanczos_top")
    return EigResult(np.array(vals[:k_eff]), vecs, np.array(res[:k_eff]), bool(conv.value), int(rst.value),
                     [float(hist[i]) for i in range(nh.value)], int(mv.value))


def small_eigh(s, rt: Optional[Runtime] = None):
    """symlin.small_eigh (symlin.py:193-198) on the device (k <= 64).
    Host numpy in -> host numpy out; use ``small_eigh_dev`` on tensors."""
    rt = rt or runtime()
    a = rt.upload(np.asarray(s, dtype=float))
    vals, vecs = small_eigh_dev(a, rt)
    return rt.download(vals), rt.download(vecs)


def small_eigh_dev(a, rt: Optional[Runtime] = None):
    rt = rt or runtime()
    k = a.shape[0]
    vals = rt.empty(k)
    vecs = rt.empty(k, k)
    check(rt.lib.usbs_small_eigh(rt.h, k, C.c_void_p(ptr(a.contiguous())), C.c_void_p(ptr(vals)),
                                 C.c_void_p(ptr(vecs))), "small_eigh")
    return vals, vecs
