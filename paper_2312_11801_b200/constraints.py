"""Device-backed constraint bundle: the duck type of DiagonalConstraints /
SparseConstraintFamilies (problem.py:144-243) over the C ABI, returning numpy
on demand.  The solver itself keeps everything resident and never calls this
surface; it serves code written against the reference's constraint objects
(tests, the reference's own loop with rebound names).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np
import scipy.sparse as sp

from ._native import check

__all__ = ["DeviceConstraints", "device_constraints"]


def _entries_of(cons, n):
    """(idx, rows, cols, vals, diag_only) of a constraint family object."""
    if hasattr(cons, "idx"):
        return (np.ascontiguousarray(cons.idx, np.int64), np.ascontiguousarray(cons.rows, np.int64),
                np.ascontiguousarray(cons.cols, np.int64), np.ascontiguousarray(cons.vals, np.float64), 0)
    ar = np.arange(n, dtype=np.int64)
    return ar, ar, ar.copy(), np.ones(n), 1


class DeviceConstraints:
    """``n``, ``m`` and the bundle methods, computed on the GPU.  ``cons`` is a
    diagonal family (any object without entry arrays) or an entry family with
    ``idx, rows, cols, vals`` (rows <= cols)."""

    def __init__(self, n: int, m: int, cons, rt=None):
        from .runtime import runtime
        self.rt = rt or runtime()
        self.n, self.m = int(n), int(m)
        self._cons = cons
        idx, rows, cols, vals, diag = _entries_of(cons, self.n)
        if rows.size and np.any(rows > cols):
            raise ValueError("entries must have rows <= cols")
        self._host = (idx, rows, cols, vals)
        self.diag_only = bool(diag)
        ip = np.zeros(self.n + 1, dtype=np.int64)
        ix = np.zeros(1, dtype=np.int32)
        dt = np.zeros(1, dtype=np.float64)
        h = C.c_void_p()
        check(self.rt.lib.usbs_problem_create(
            self.rt.h, self.n, max(self.m, 1), C.c_void_p(ip.ctypes.data), C.c_void_p(ix.ctypes.data),
            C.c_void_p(dt.ctypes.data), int(vals.size), C.c_void_p(idx.ctypes.data), C.c_void_p(rows.ctypes.data),
            C.c_void_p(cols.ctypes.data), C.c_void_p(vals.ctypes.data), diag, C.byref(h)), "problem_create")
        self.h = h
        self._pattern = None

    def __del__(self):
        try:
            if getattr(self, "h", None) is not None:
                self.rt.lib.usbs_problem_destroy(self.h)
                self.h = None
        except Exception:
            pass

    # ------------------------------------------------------------ helpers
    def _dev(self, a):
        a = np.asarray(a, dtype=np.float64)
        return self.rt.upload(a)

    def _block(self, v):
        v = np.asarray(v, dtype=np.float64)
        vec = v.ndim == 1
        return self._dev(v.reshape(self.n, -1)), vec

    # ------------------------------------------------------------ images
    def primal_image_lowrank(self, v, s) -> np.ndarray:
        """A(V S V^T) (problem.py:151-152, 200-203)."""
        V, _ = self._block(v)
        S = self._dev(np.asarray(s, dtype=float).reshape(V.shape[1], V.shape[1]))
        out = self.rt.empty(self.m)
        check(self.rt.lib.usbs_cons_image(self.rt.h, self.h, V.data_ptr(), V.stride(0), V.shape[1], S.data_ptr(),
                                          0, 1.0, None, 0.0, None, out.data_ptr()), "cons_image")
        return self.rt.download(out)

    def primal_image_factor(self, u, lams) -> np.ndarray:
        """A(U diag(lams) U^T) (problem.py:154-155, 205-208)."""
        U, _ = self._block(u)
        L = self._dev(np.asarray(lams, dtype=float).reshape(-1))
        out = self.rt.empty(self.m)
        check(self.rt.lib.usbs_cons_image(self.rt.h, self.h, U.data_ptr(), U.stride(0), U.shape[1], L.data_ptr(),
                                          1, 1.0, None, 0.0, None, out.data_ptr()), "cons_image")
        return self.rt.download(out)

    def primal_image_dense(self, x) -> np.ndarray:
        """A(X) for a dense symmetric n x n X (problem.py:157-158, 210-212)."""
        X = self._dev(np.asarray(x, dtype=float).reshape(self.n, self.n))
        out = self.rt.empty(self.m)
        check(self.rt.lib.usbs_cons_image_dense(self.rt.h, self.h, X.data_ptr(), X.stride(0), out.data_ptr()),
              "cons_image_dense")
        return self.rt.download(out)

    # ------------------------------------------------------------ adjoint
    def adjoint_matrix(self, y):
        """A*(y) as a scipy CSR (problem.py:160-161, 214-220)."""
        if self._pattern is None:
            nnz = int(self._nnz())
            rp = np.zeros(self.n + 1, dtype=np.int64)
            col = np.zeros(max(nnz, 1), dtype=np.int32)
            nent = np.zeros(max(nnz, 1), dtype=np.int32)
            check(self.rt.lib.usbs_problem_pattern(self.h, C.c_void_p(rp.ctypes.data), C.c_void_p(col.ctypes.data),
                                                   C.c_void_p(nent.ctypes.data)), "problem_pattern")
            self._pattern = (rp, col[:nnz], nent[:nnz] > 0, nnz)
        rp, col, keep, nnz = self._pattern
        Y = self._dev(np.asarray(y, dtype=float).reshape(-1))
        vals = self.rt.empty(max(nnz, 1))
        check(self.rt.lib.usbs_cons_adjoint_values(self.rt.h, self.h, Y.data_ptr(), vals.data_ptr()),
              "cons_adjoint_values")
        v = self.rt.download(vals)[:nnz]
        rows = np.repeat(np.arange(self.n), np.diff(rp))
        return sp.csr_matrix((v[keep], (rows[keep], col[keep])), shape=(self.n, self.n))

    def _nnz(self):
        a, b = C.c_int64(), C.c_int64()
        c_, d = C.c_int(), C.c_int()
        check(self.rt.lib.usbs_problem_info(self.h, C.byref(a), C.byref(b), C.byref(c_), C.byref(d)), "info")
        return a.value

    def _adjoint_apply(self, y, v, gram: bool):
        V, vec = self._block(v)
        k = V.shape[1]
        Y = self._dev(np.asarray(y, dtype=float).reshape(-1))
        out = self.rt.empty(self.n, k)
        g = self.rt.empty(k, k) if gram else None
        check(self.rt.lib.usbs_cons_adjoint_apply(self.rt.h, self.h, Y.data_ptr(), V.data_ptr(), V.stride(0), k,
                                                  out.data_ptr(), out.stride(0), g.data_ptr() if gram else None),
              "cons_adjoint_apply")
        if gram:
            return self.rt.download(g)
        r = self.rt.download(out)
        return r.reshape(-1) if vec else r

    def adjoint_matvec(self, y, v) -> np.ndarray:
        """A*(y) v (problem.py:163-164, 222-223)."""
        return self._adjoint_apply(y, v, False)

    def adjoint_inner_lowrank(self, y, v) -> np.ndarray:
        """sym(V^T A*(y) V) (problem.py:166-167, 225-227)."""
        return self._adjoint_apply(y, v, True)

    # ------------------------------------------------------------ rows / norms
    def compressed_rows(self, v) -> np.ndarray:
        """Rows svec(V^T A_i V) (problem.py:169-173, 229-239), m x k(k+1)/2."""
        V, _ = self._block(v)
        k = V.shape[1]
        d = k * (k + 1) // 2
        out = self.rt.empty(self.m, d)
        check(self.rt.lib.usbs_cons_compressed_rows(self.rt.h, self.h, V.data_ptr(), V.stride(0), k,
                                                    out.data_ptr(), out.stride(0)), "cons_compressed_rows")
        return self.rt.download(out)

    def frob_norms(self) -> np.ndarray:
        """||A_i||_F (problem.py:175-176, 241-243): static data, computed once
        on the host like the reference."""
        if self.diag_only:
            return np.ones(self.m)
        idx, rows, cols, vals = self._host
        sq = vals ** 2 * np.where(rows == cols, 1.0, 2.0)
        return np.sqrt(np.bincount(idx, weights=sq, minlength=self.m))

    def scaled(self, factors) -> "DeviceConstraints":
        """Entry family with vals * factors[idx] (problem.py:195-198)."""
        if self.diag_only:
            raise AttributeError("the diagonal family has no scaled()")
        idx, rows, cols, vals = self._host

        class _E:
            pass
        e = _E()
        e.idx, e.rows, e.cols, e.vals = idx, rows, cols, vals * np.asarray(factors, dtype=float)[idx]
        return DeviceConstraints(self.n, self.m, e, self.rt)


def device_constraints(prob, rt=None) -> DeviceConstraints:
    """The device bundle of an SdpProblem's constraints."""
    return DeviceConstraints(prob.n, prob.m, prob.constraints, rt)
