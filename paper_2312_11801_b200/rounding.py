"""Combinatorial rounding of reconstructed primal factors (rounding.py).

``maxcut_round`` runs on the device (``usbs_maxcut_round``: one pass over
the edges per factor column, exact for integer weights, so the cut value and
the assignment equal the reference's bit for bit).  ``qap_round`` keeps the
Hungarian step on the host as the reference does (scipy's
``linear_sum_assignment``); it is exit-time work, not part of the iteration.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np
from scipy.optimize import linear_sum_assignment

from ._native import check

__all__ = ["CutResult", "PermResult", "maxcut_round", "hungarian", "qap_round", "assignment_objective",
           "GapTracker"]


@dataclass
class CutResult:
    assignment: np.ndarray  # entries in {-1, +1}
    value: float
    values: Optional[np.ndarray] = None  # cut value of every column


@dataclass
class PermResult:
    perm: np.ndarray
    objective: float
    relative_gap: Optional[float] = None


def _edges(g):
    eu = getattr(g, "eu", None)
    if eu is None:  # reference GraphInstance
        return g.n, g.edges_u, g.edges_v, g.edges_w
    return g.n, g.eu, g.ev, g.ew


def maxcut_round(u, g, rt=None) -> CutResult:
    """maxcut_round (rounding.py:34-51): the sign cut of every factor column,
    the largest kept (first one on ties); zero entries sign to +1.
    ``u``: n x r host array or device tensor; ``g``: a graph with edge arrays
    (instances.Graph or the reference GraphInstance)."""
    from .runtime import runtime
    rt = rt or runtime()
    torch = rt.torch
    n, eu, ev, ew = _edges(g)
    if isinstance(u, np.ndarray) or not hasattr(u, "data_ptr"):
        u = np.atleast_2d(np.asarray(u, dtype=float))
        if u.ndim != 2 or u.shape[0] != n or u.shape[1] == 0:
            raise ValueError("factor must be a nonempty n x r matrix")
        U = rt.upload(u)
    else:
        U = u if u.dim() == 2 else u.view(-1, 1)
        if U.shape[0] != n or U.shape[1] == 0:
            raise ValueError("factor must be a nonempty n x r matrix")
        U = U.contiguous()
    r = U.shape[1]
    dev = rt.device
    deu = torch.as_tensor(np.asarray(eu, dtype=np.int32), device=dev)
    dev_v = torch.as_tensor(np.asarray(ev, dtype=np.int32), device=dev)
    dew = torch.as_tensor(np.asarray(ew, dtype=np.float64), device=dev)
    x = torch.empty(n, dtype=torch.int32, device=dev)
    vals = (C.c_double * r)()
    best = C.c_int()
    check(rt.lib.usbs_maxcut_round(rt.h, int(n), int(deu.numel()), deu.data_ptr(), dev_v.data_ptr(),
                                   dew.data_ptr(), U.data_ptr(), U.stride(0), int(r), vals, C.byref(best),
                                   x.data_ptr()), "maxcut_round")
    return CutResult(assignment=x.cpu().numpy().astype(int), value=float(vals[best.value]),
                     values=np.array(vals[:], dtype=float))


def hungarian(cost: np.ndarray) -> np.ndarray:
    """Row -> column map of a minimum-cost assignment (rounding.py:54-64),
    scipy's solver as in the reference, so ties resolve identically."""
    c = np.asarray(cost, dtype=float)
    if c.ndim != 2 or c.shape[0] != c.shape[1] or not np.isfinite(c).all():
        raise ValueError("hungarian needs a finite square cost matrix")
    r_idx, c_idx = linear_sum_assignment(c)
    out = np.zeros(c.shape[0], dtype=np.int64)
    out[r_idx] = c_idx
    return out


def assignment_objective(q, perm: np.ndarray) -> float:
    """<W, P D P^T> for the permutation perm (rounding.py:67-69)."""
    p = np.asarray(perm)
    return float(np.sum(q.weights * q.distances[p][:, p]))


def qap_round(u, q, known_optimum: Optional[float] = None) -> PermResult:
    """qap_round (rounding.py:72-93).  Column j of the (l^2 + 1) x r factor,
    minus its affine first entry, is the l x l block X_j with X_j[a, b] =
    u[1 + a + l b, j]; its permutation maximises <X_j, P>, and the column
    with the smallest objective wins (the first on ties)."""
    l = q.weights.shape[0]
    f = u.cpu().numpy() if hasattr(u, "cpu") else u
    f = np.atleast_2d(np.asarray(f, dtype=float))
    if f.shape[0] != l * l + 1:
        raise ValueError(f"factor must have {l * l + 1} rows")
    # blocks[j][a, b] = f[1 + a + l b, j]
    blocks = f[1:].T.reshape(f.shape[1], l, l).transpose(0, 2, 1)
    cands = [hungarian(-blk) for blk in blocks]
    objs = [assignment_objective(q, pm) for pm in cands]
    j = int(np.argmin(objs))  # argmin keeps the first minimum
    res = PermResult(perm=cands[j], objective=objs[j])
    opt = known_optimum if known_optimum is not None else getattr(q, "known_optimum", None)
    if opt:
        res.relative_gap = (res.objective - opt) / opt
    return res


class GapTracker:
    """Best (smallest) relative gap seen so far (rounding.py:96-109)."""

    def __init__(self):
        self.best: Optional[float] = None

    def update(self, gap) -> float:
        g = gap.relative_gap if isinstance(gap, PermResult) else float(gap)
        if g is None:
            raise ValueError("result carries no relative gap")
        self.best = g if self.best is None else min(self.best, g)
        return self.best
