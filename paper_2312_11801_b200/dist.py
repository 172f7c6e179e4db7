"""Row sharding of the USBS hot path over several GPUs.

GPU p owns a contiguous row block [r_p, r_{p+1}) of Z = C - A*(y) (balanced
on nnz + rows, for power-law degree sequences), of the basis V, of the
Lanczos basis Q, of F, Psi and P, and -- for diagonal constraints (MaxCut,
the sharded configs C4) -- of the m = n constraint vectors (y, nu, A Xbar,
a_x, b).  Everything k x k / d x d (Grams, IPM, Rayleigh-Ritz) is computed
redundantly on every rank from allreduced inputs, so all ranks take the same
branches.  Collectives (torch.distributed: NCCL on GPUs, gloo in the CPU
tests):
  * per SpMV (each Lanczos step, each SpMM): allgather of the input block;
  * per Lanczos step: allreduce of Q^T w twice (<= 33 doubles) and ||w||^2;
  * per outer iteration: allreduce of the k x k / d x d Grams, d-vectors and
    residual scalars.
Reductions run in a fixed order for a fixed communicator, so runs are
reproducible; parity with the single-GPU path is to rounding, not bitwise.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np
import scipy.sparse as sp

from .errors import NumericError


@dataclass
class Shard:
    rank: int
    world: int
    n: int
    bounds: np.ndarray  # world + 1 row boundaries

    @property
    def r0(self) -> int:
        return int(self.bounds[self.rank])

    @property
    def r1(self) -> int:
        return int(self.bounds[self.rank + 1])

    @property
    def rows(self) -> int:
        return self.r1 - self.r0

    @property
    def counts(self):
        return np.diff(self.bounds).astype(np.int64)

    @staticmethod
    def balanced(indptr: np.ndarray, world: int, rank: int, row_cost: float = 4.0) -> "Shard":
        """Row blocks with equal nnz + row_cost * rows (every rank gets >= 1 row)."""
        indptr = np.asarray(indptr, dtype=np.int64)
        n = indptr.size - 1
        cost = indptr[1:] - indptr[:-1] + row_cost
        cum = np.concatenate([[0.0], np.cumsum(cost)])
        targets = cum[-1] * np.arange(1, world) / world
        cuts = np.searchsorted(cum, targets, side="left")
        bounds = np.concatenate([[0], cuts, [n]]).astype(np.int64)
        for p in range(1, world + 1):  # enforce strictly increasing
            bounds[p] = max(bounds[p], bounds[p - 1] + 1)
        for p in range(world - 1, -1, -1):
            bounds[p] = min(bounds[p], bounds[p + 1] - 1)
        if bounds[0] != 0 or bounds[-1] != n:
            raise ValueError("cannot shard fewer rows than ranks")
        return Shard(rank, world, n, bounds)


class Comm:
    """torch.distributed collectives on flat tensors (no-ops for world 1)."""

    def __init__(self, world: int, group=None):
        self.world = world
        self.group = group

    def _dist(self):
        import torch.distributed as dist
        return dist

    def allreduce_sum(self, t):
        if self.world > 1:
            self._dist().all_reduce(t, group=self.group)
        return t

    def allreduce_max(self, t):
        if self.world > 1:
            d = self._dist()
            d.all_reduce(t, op=d.ReduceOp.MAX, group=self.group)
        return t

    def allgather_rows(self, local, out, shard: Shard):
        """out (n x k) = concatenation of every rank's local (rows_p x k)."""
        if self.world == 1:
            out.copy_(local)
            return out
        import torch
        d = self._dist()
        counts = shard.counts
        mx = int(counts.max())
        k = local.shape[1]
        buf = torch.zeros((mx, k), dtype=local.dtype, device=local.device)
        buf[: local.shape[0]].copy_(local)
        parts = [torch.empty_like(buf) for _ in range(self.world)]
        d.all_gather(parts, buf, group=self.group)
        for p in range(self.world):
            out[shard.bounds[p]: shard.bounds[p + 1]].copy_(parts[p][: counts[p]])
        return out


def shard_maxcut(prob, shard: Shard):
    """Local arrays of a diagonal-constraint problem (MaxCut) for one rank:
    CSR rows [r0, r1) of C with global columns, the directed diagonal
    entries (i, i, r0 + i, 1.0), b and the inequality mask slices."""
    cons = prob.constraints
    if hasattr(cons, "idx"):
        raise NotImplementedError("row sharding currently covers diagonal constraints (MaxCut, C4); "
                                  "entry-family sharding (C5) is listed in DESIGN.md as next")
    c = prob.cost.tocsr()
    r0, r1 = shard.r0, shard.r1
    loc = c[r0:r1]
    nl = r1 - r0
    ar = np.arange(nl, dtype=np.int64)
    return dict(indptr=np.ascontiguousarray(loc.indptr, dtype=np.int64),
                indices=np.ascontiguousarray(loc.indices, dtype=np.int32),
                data=np.ascontiguousarray(loc.data, dtype=np.float64),
                e_idx=ar, e_rows=ar.copy(), e_cols=ar + r0, e_vals=np.ones(nl),
                b=np.asarray(prob.b, dtype=float)[r0:r1],
                ineq=np.asarray(prob.ineq_mask, dtype=bool)[r0:r1])


class ShardedDeviceProblem:
    """The rank's row block of an SdpProblem on its GPU (C-ABI shard problem:
    local rows, global columns).  Same methods as runtime.DeviceProblem; the
    operator apply gathers the input block from all ranks first."""

    def __init__(self, prob, shard: Shard, comm: Comm, rt=None):
        import ctypes as C

        from ._native import check
        from .runtime import runtime

        self.rt = rt or runtime()
        self.prob, self.shard, self.comm = prob, shard, comm
        a = shard_maxcut(prob, shard)
        self.n = shard.rows
        self.m = shard.rows
        self.n_global = shard.n
        h = C.c_void_p()
        check(self.rt.lib.usbs_problem_create_shard(
            self.rt.h, self.n, shard.n, self.m, C.c_void_p(a["indptr"].ctypes.data),
            C.c_void_p(a["indices"].ctypes.data), C.c_void_p(a["data"].ctypes.data), self.n,
            C.c_void_p(a["e_idx"].ctypes.data), C.c_void_p(a["e_rows"].ctypes.data),
            C.c_void_p(a["e_cols"].ctypes.data), C.c_void_p(a["e_vals"].ctypes.data), 1, C.byref(h)),
            "problem_create_shard")
        self.h = h
        self.diag_only = True
        self.b = self.rt.upload(a["b"])
        self.ineq_mask = a["ineq"]
        self.has_ineq = bool(np.asarray(prob.ineq_mask, dtype=bool).any())
        self.ineq = self.rt.upload(a["ineq"].astype(np.float64))
        self.alpha = float(prob.alpha)
        self._xfull = {}

    def __del__(self):
        try:
            if getattr(self, "h", None) is not None:
                self.rt.lib.usbs_problem_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def assemble(self, y_dev):
        import ctypes as C

        from ._native import check, ptr
        check(self.rt.lib.usbs_slack_assemble(self.rt.h, self.h, C.c_void_p(ptr(y_dev))), "slack_assemble")

    def apply(self, which, V, out=None, gram=None, xfull=None):
        import ctypes as C

        from ._native import check, ptr
        if V.dim() == 1:
            V = V.view(-1, 1)
        k = V.shape[1]
        if xfull is None:
            xfull = self._xfull.get(k)
            if xfull is None:
                xfull = self.rt.empty(self.n_global, k)
                self._xfull[k] = xfull
        self.comm.allgather_rows(V.contiguous() if V.stride(1) != 1 else V, xfull, self.shard)
        if out is None:
            out = self.rt.empty(self.n, k)
        check(self.rt.lib.usbs_op_apply(self.rt.h, self.h, int(which), C.c_void_p(ptr(xfull)), xfull.stride(0), k,
                                        C.c_void_p(ptr(out)), out.stride(0), None), "op_apply")
        if gram is not None:
            check(self.rt.lib.usbs_gram(self.rt.h, self.n, C.c_void_p(ptr(V)), V.stride(0), k, C.c_void_p(ptr(out)),
                                        out.stride(0), k, C.c_void_p(ptr(gram)), 1), "gram")
            self.comm.allreduce_sum(gram)
        return out


def lanczos_sharded(eng, dp, which: int, k_c: int, inner_iters: int = 32, max_restarts: int = 10,
                    tol: Optional[float] = None, seed: int = 0, out=None):
    """lanczos_top (eigsolve.py:83-181) on a row-sharded operator, host-driven
    step by step on the engine's primitives (SpMV with allgather, allreduced
    Grams, local row GEMMs).  Same m, ell, tolerance, breakdown and restart
    rules as the single-GPU kernel; H and the Ritz data are replicated."""
    from .eigen import EigResult

    rt = eng.rt
    shard = dp.shard
    n = shard.n
    nl = dp.n
    if k_c < 1:
        raise ValueError("k_c must be at least 1")
    m = max(int(inner_iters), k_c + 1, 2)
    if k_c >= n or inner_iters >= n or m >= n:
        raise NotImplementedError("dense fallback (n <= inner_iters) is not sharded")
    tol = 1e-9 if tol is None else tol
    seed32 = int(seed) & 0xFFFFFFFF

    def seeded(counter):
        g = np.random.default_rng([seed32, counter])
        v = g.standard_normal(n)
        return v / np.linalg.norm(v)

    Q = rt.zeros(nl, m + 1)
    h = np.zeros((m + 1, m + 1))
    Q[:, 0:1].copy_(rt.upload(seeded(0)[shard.r0: shard.r1].reshape(-1, 1)))
    xfull = rt.empty(n, 1)
    w = rt.empty(nl, 1)
    cvec = rt.empty(m + 1, 1)
    red = rt.zeros(2)
    ell, ctr, hist, conv, restarts, mv = 0, 0, [], False, 0, 0
    theta, ymat, res = np.zeros(m), np.eye(m), np.full(m, np.inf)

    def proj_out(v, used):
        """v -= Q[:, :used] (Q[:, :used]^T v), allreduced coefficients."""
        cv = cvec[:used]
        eng.gram(Q[:, :used], v, cv)
        eng.rowgemm(Q[:, :used], cv, v, alpha=-1.0, beta=1.0, Y0=v)
        return cv

    def norm(v):
        eng.dot_into(v.view(-1), v.view(-1), red[0:1])
        return math.sqrt(max(float(red[0].item()), 0.0))

    for cyc in range(max_restarts + 1):
        for j in range(ell, m):
            dp.apply(which, Q[:, j: j + 1], out=w, xfull=xfull)
            mv += 1
            eng.dot_into(w.view(-1), w.view(-1), red[0:1])
            if not math.isfinite(float(red[0].item())):
                raise NumericError("matvec returned non-finite values")
            c1 = proj_out(w, j + 1).cpu().numpy().ravel().copy()
            c2 = proj_out(w, j + 1).cpu().numpy().ravel().copy()
            c = c1 + c2
            h[: j + 1, j] = c
            h[j, : j + 1] = c
            beta = norm(w)
            scale = max(1.0, float(np.max(np.abs(c))) if c.size else 0.0)
            if beta <= 1e-13 * scale:
                ctr += 16
                got = False
                for att in range(8):
                    v = rt.upload(seeded(ctr + att + 1)[shard.r0: shard.r1].reshape(-1, 1))
                    proj_out(v, j + 1)
                    nv = norm(v)
                    if nv > 1e-8:
                        eng.rowgemm(v, rt.upload(np.ones((1, 1))), Q[:, j + 1: j + 2], alpha=1.0 / nv)
                        got = True
                        break
                if not got:
                    Q[:, j + 1: j + 2].zero_()
                h[j + 1, j] = h[j, j + 1] = 0.0
            else:
                eng.rowgemm(w, rt.upload(np.ones((1, 1))), Q[:, j + 1: j + 2], alpha=1.0 / beta)
                h[j + 1, j] = h[j, j + 1] = beta
        hm = rt.upload(h[:m, :m])
        vals, vecs = rt.empty(m), rt.empty(m, m)
        eng.small_eigh(hm, vals, vecs)
        theta, ymat = vals.cpu().numpy(), vecs.cpu().numpy()
        res = np.abs(h[m, m - 1] * ymat[m - 1, :])
        hist.append(float(theta[0]))
        if np.all(res[:k_c] <= tol * (1.0 + abs(float(theta[0])))):
            conv = True
            break
        if cyc == max_restarts:
            break
        ell = max(1, min(k_c + 3, m - 2))
        kept = rt.empty(nl, ell)
        eng.rowgemm(Q[:, :m], rt.upload(ymat[:, :ell]), kept)
        Q[:, ell: ell + 1].copy_(Q[:, m: m + 1])
        Q[:, :ell].copy_(kept)
        h[:, :] = 0.0
        h[:ell, :ell] = np.diag(theta[:ell])
        restarts += 1
    k = min(k_c, n)
    vecs_out = out if out is not None else rt.empty(nl, k)
    eng.rowgemm(Q[:, :m], rt.upload(ymat[:, :k_c]), vecs_out)
    return EigResult(theta[:k_c].copy(), vecs_out, res[:k_c].copy(), conv, restarts, hist, mv)
