"""Standalone device versions of the reference's dense helpers that its
package re-exports (symlin.orthonormalize, sketch.sketch_init /
sketch_update / reconstruct), numpy in and out.  The solver uses the same
device code on resident tensors (solver.orthonormalize_dev,
solver.DeviceSketchStore); these wrappers serve callers of the reference API.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = ["orthonormalize", "NystromSketch", "make_test_matrix", "sketch_init", "sketch_update", "reconstruct"]


class _Ctx:
    """Problem-free engine context (the dense kernels need no operator)."""

    def __init__(self, rt, n):
        self.rt, self.h, self.n, self.m = rt, None, int(n), 0


def _engine(n):
    from .engine import Engine
    from .runtime import runtime
    rt = runtime()
    return Engine(_Ctx(rt, n)), rt


def orthonormalize(cols, drop_tol: float = 1e-12) -> np.ndarray:
    """Orthonormal basis for the span of the columns (symlin.py:148-190):
    pivot order and drop rule of the reference's column-pivoted Gram-Schmidt
    (drop below drop_tol x the largest column norm), computed on the GPU."""
    from .errors import EmptyBasisError
    from .solver import orthonormalize_dev
    if isinstance(cols, np.ndarray):
        a = np.array(cols, dtype=float)
        if a.ndim == 1:
            a = a[:, None]
    else:
        a = np.column_stack([np.asarray(c, dtype=float) for c in cols])
    if a.size == 0:
        raise EmptyBasisError("no input columns")
    if a.shape[1] > 40:
        raise ValueError("orthonormalize supports at most 40 columns")
    eng, rt = _engine(a.shape[0])
    return rt.download(orthonormalize_dev(eng, rt.upload(a), drop_tol))


def make_test_matrix(n: int, r: int, seed: int) -> np.ndarray:
    """The Nystrom test matrix (sketch.py:25-27): legacy MT19937 normals."""
    return np.random.RandomState(int(seed) & 0x7FFFFFFF).standard_normal((n, r))


@dataclass
class NystromSketch:
    """sketch.NystromSketch (sketch.py:30-44): same fields."""

    n: int
    r: int
    psi_seed: int
    sketch_mat: np.ndarray
    psi_cache: Optional[np.ndarray] = field(default=None, repr=False)

    def psi(self) -> np.ndarray:
        return self.psi_cache if self.psi_cache is not None else make_test_matrix(self.n, self.r, self.psi_seed)


def sketch_init(n: int, r: int, seed: int, store_psi: bool = True) -> NystromSketch:
    """Zero sketch with a reproducible test matrix (sketch.py:47-55)."""
    if not 1 <= r <= n:
        raise ValueError(f"sketch rank {r} must lie in [1, {n}]")
    psi = make_test_matrix(n, r, seed)
    return NystromSketch(n, r, int(seed), np.zeros((n, r)), psi if store_psi else None)


def _store(s: NystromSketch):
    from .solver import DeviceSketchStore
    eng, rt = _engine(s.n)
    st = DeviceSketchStore(eng, s.n, s.r, s.psi_seed, psi_host=s.psi())
    st.P.copy_(rt.upload(np.asarray(s.sketch_mat, dtype=float)))
    return st, eng, rt


def sketch_update(s: NystromSketch, eta: float, v, q, lams) -> NystromSketch:
    """eta * old + (V Q) diag(lams) (V Q)^T applied to the sketch
    (sketch.py:58-74): P <- eta P + (F L)(F^T Psi), F = V Q, on the GPU."""
    if eta < 0:
        raise ValueError("eta must be nonnegative")
    lams = np.asarray(lams, dtype=float)
    if np.any(lams < -1e-12 * max(1.0, float(np.max(np.abs(lams), initial=0.0)))):
        raise ValueError("update eigenvalues must be nonnegative")
    v = np.asarray(v, dtype=float)
    q = np.asarray(q, dtype=float)
    if v.shape[0] != s.n or v.shape[1] != q.shape[0]:
        raise ValueError("dimension mismatch in sketch update")
    st, eng, rt = _store(s)
    F = eng.rowgemm(rt.upload(v), rt.upload(q), rt.empty(s.n, q.shape[1]))
    st.update(float(eta), F, rt.upload(lams))
    return NystromSketch(s.n, s.r, s.psi_seed, rt.download(st.P), s.psi_cache)


def reconstruct(s: NystromSketch):
    """Shift-stabilised Nystrom reconstruction (sketch.py:77-111): (U, lams)
    with the core Gram, its Cholesky and the triangular solve on the GPU and
    the final thin SVD on the host."""
    st, _, _ = _store(s)
    return st.factorize()
