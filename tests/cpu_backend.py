"""CPU (numpy/torch-CPU) stand-in for the device engine -- TEST INFRASTRUCTURE.

Implements the Engine / DeviceProblem method surface used by
paper_2312_11801_b200.solver.DeviceSolver and dist.lanczos_sharded with host
arithmetic, so the row-sharded host logic (partitioning, which reductions are
allreduced, gathers, replicated k x k work) can be exercised under a
world_size-2 gloo process group on a machine without GPUs.  The k x k IPM
and small eigensolves delegate to the CPU oracle.  Never used by the product.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp
import torch

from oracle import usbs_cpu as O
from paper_2312_11801_b200 import _native as N
from paper_2312_11801_b200 import instances as inst
from paper_2312_11801_b200.dist import Comm, EntryShardPlan, Shard, _allgather_var, shard_maxcut


class CpuRuntime:
    def __init__(self):
        self.torch = torch
        self.device = torch.device("cpu")
        self.stream = None

    def empty(self, *shape):
        return torch.empty(*shape, dtype=torch.float64)

    def zeros(self, *shape):
        return torch.zeros(*shape, dtype=torch.float64)

    def upload(self, a):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).clone()

    def download(self, t):
        return t.numpy()

    def sync(self):
        pass

    def launches(self):
        return 0


class CpuShardProblem:
    def __init__(self, prob, shard: Shard, comm: Comm, rt: CpuRuntime):
        self.rt, self.prob, self.shard, self.comm = rt, prob, shard, comm
        self.n = shard.rows
        self.n_global = shard.n
        self.entries = hasattr(prob.constraints, "idx")
        c = prob.cost.tocsr()[shard.r0:shard.r1]
        self.C = sp.csr_matrix((c.data, c.indices, c.indptr), shape=(self.n, shard.n))
        self.Z = self.C.copy()
        if self.entries:
            self.plan = pl = EntryShardPlan(prob, shard)
            self.m = pl.m_own
            b, ineq = pl.b, pl.ineq
            self.owned_family = inst.EntryFamilies(shard.n, max(pl.m_own, 1), pl.o_idx, pl.o_rows, pl.o_cols,
                                                   pl.o_vals)
        else:
            a = shard_maxcut(prob, shard)
            self.m = shard.rows
            b, ineq = a["b"], a["ineq"]
        self.b = rt.upload(b)
        self.ineq_mask = ineq
        self.has_ineq = bool(np.asarray(prob.ineq_mask).any())
        self.ineq = rt.upload(ineq.astype(float))
        self.alpha = float(prob.alpha)
        self.diag_only = not self.entries

    def assemble(self, y):
        if not self.entries:
            d = sp.csr_matrix((y.numpy().copy(), (np.arange(self.n), self.shard.r0 + np.arange(self.n))),
                              shape=(self.n, self.shard.n))
        else:
            pl = self.plan
            cat = torch.zeros(pl.m_total, dtype=torch.float64)
            _allgather_var(self.comm, y, pl.counts, cat)
            y_ext = np.concatenate([y.numpy(), cat.numpy()[pl.ghost_pos]])
            d = sp.coo_matrix((y_ext[pl.d_idx] * pl.d_vals, (pl.d_rows, pl.d_cols)),
                              shape=(self.n, self.shard.n)).tocsr()
        self.Z = (self.C - d).tocsr()

    def full_rows(self, V):
        full = torch.empty(self.shard.n, V.shape[1], dtype=torch.float64)
        self.comm.allgather_rows(V, full, self.shard)
        return full

    def apply(self, which, V, out=None, gram=None, xfull=None):
        if V.dim() == 1:
            V = V.view(-1, 1)
        k = V.shape[1]
        full = torch.empty(self.shard.n, k, dtype=torch.float64)
        self.comm.allgather_rows(V, full, self.shard)
        M = self.Z if which else self.C
        res = torch.from_numpy(M @ full.numpy())
        if out is None:
            out = torch.empty(self.n, k, dtype=torch.float64)
        out.copy_(res)
        if gram is not None:
            g = V.numpy().T @ out.numpy()
            gram.copy_(torch.from_numpy(0.5 * (g + g.T)))
            self.comm.allreduce_sum(gram)
        return out


class CpuEngine:
    def __init__(self, dp: CpuShardProblem, comm: Comm):
        self.dp, self.rt = dp, dp.rt
        self.n, self.m = dp.n, dp.m
        self.comm = comm if comm.world > 1 else None

    def _ar(self, t, op="sum"):
        if self.comm is not None:
            (self.comm.allreduce_sum if op == "sum" else self.comm.allreduce_max)(t)

    # ---- vectors
    def vec(self, op, m, x=None, y=None, z=None, b=None, ineq=None, s0=0.0, s1=0.0, out=None, red=None):
        X = x.reshape(-1).numpy()[:m] if x is not None else None
        Y = y.reshape(-1).numpy()[:m] if y is not None else None
        Zv = z.reshape(-1).numpy()[:m] if z is not None else None
        B = b.numpy()[:m] if b is not None else None
        iq = (ineq.numpy()[:m] != 0.0) if ineq is not None else np.zeros(m, bool)
        r0, r1, res = 0.0, 0.0, None
        if op == N.VOP_W:
            res = X - (B + Y) / s0
        elif op == N.VOP_PROJN:
            res = np.where(iq, np.minimum(X, 0.0), 0.0)
        elif op == N.VOP_AXPBY:
            res = s0 * X + (s1 * Y if Y is not None else 0.0)
        elif op == N.VOP_NUNEXT:
            t = X + s0 * Y - B
            res = np.where(iq, np.minimum(t, 0.0), 0.0)
            r0 = float(np.sum((res - Zv) ** 2))
        elif op == N.VOP_CAND:
            v = Y - (B - X) / s0
            res = np.where(iq, np.where(Zv < 0.0, 0.0, np.maximum(v, 0.0)), v)
        elif op == N.VOP_RESID:
            pk = np.where(iq, np.minimum(X, B), B)
            dlt = X - pk
            r0, r1 = float(dlt @ dlt), float(np.max(np.abs(dlt))) if m else 0.0
        elif op in (N.VOP_DOT, N.VOP_DOTAFF):
            r0 = float(X @ Y)
        elif op == N.VOP_MINI:
            r1 = float(np.max(-X[iq])) if iq.any() else -np.inf
        elif op == N.VOP_RELU:
            res = np.maximum(X, 0.0)
        if res is not None and out is not None:
            out.reshape(-1)[:m].copy_(torch.from_numpy(np.asarray(res, dtype=float)))
        if red is not None:
            t = torch.tensor([r0, r1], dtype=torch.float64)
            self._ar(t[0:1])
            self._ar(t[1:2], "max")
            if op == N.VOP_DOTAFF:
                red[0] = s0 * t[0] + s1
            else:
                red[0:2].copy_(t)

    def dot_into(self, x, y, red, scale=1.0, shift=0.0):
        self.vec(N.VOP_DOTAFF, x.numel(), x=x, y=y, s0=scale, s1=shift, red=red)

    # ---- dense
    def rowgemm(self, X, B, Y, alpha=1.0, beta=0.0, Y0=None, xs=None, n=None):
        Xn = X.numpy()
        if xs is not None:
            Xn = Xn * xs.numpy()[None, : Xn.shape[1]]
        v = alpha * (Xn @ B.numpy())
        if Y0 is not None:
            v = v + beta * Y0.numpy()
        Y.copy_(torch.from_numpy(np.ascontiguousarray(v)))
        return Y

    def gram(self, A, B, out, sym=False):
        g = A.numpy().T @ B.numpy()
        if sym:
            g = 0.5 * (g + g.T)
        out.copy_(torch.from_numpy(np.ascontiguousarray(g)).reshape(out.shape))
        self._ar(out)
        return out

    def wcoldot(self, F, G, w, out):
        out[0] = float(np.sum(F.numpy() * G.numpy() * w.numpy()[None, : F.shape[1]]))
        self._ar(out[0:1])

    def lz_step_finish(self, j, m1, c1, c2, nrm2, H, flags, w, q):
        c = (c1.reshape(-1) + c2.reshape(-1)).numpy()
        beta = math.sqrt(max(float(nrm2.reshape(-1)[0]), 0.0))
        bad = (not np.all(np.isfinite(c))) or not math.isfinite(beta)
        mx = float(np.max(np.abs(c))) if c.size else 0.0
        brk = not (beta > 1e-13 * max(1.0, mx))
        H[: j + 1, j] = torch.from_numpy(c)
        H[j, : j + 1] = torch.from_numpy(c)
        H[j + 1, j] = H[j, j + 1] = 0.0 if brk else beta
        if brk and int(flags[0]) < 0:
            flags[0] = j
        if bad:
            flags[1] = 1
        q.copy_(w * (0.0 if brk else 1.0 / beta))

    def lz_restart_h(self, m1, ell, theta, H):
        H.zero_()
        for u in range(ell):
            H[u, u] = theta[u]

    def small_eigh(self, a, vals, vecs):
        lam, q = O.eigh_desc(a.numpy())
        vals.copy_(torch.from_numpy(lam))
        vecs.copy_(torch.from_numpy(q))

    def svec(self, A, out, scale=1.0):
        out.copy_(torch.from_numpy(scale * O.svec(A.numpy())))
        return out

    def pivchol(self, G, drop_tol, perm, rinv, info):
        g = G.numpy().copy()
        c = g.shape[0]
        mx = float(np.sqrt(np.maximum(np.diag(g), 0.0)).max())
        thresh = 0.0 if drop_tol < 0 else drop_tol * mx
        alive = list(range(c))
        order, minratio = [], 1.0
        A = g.copy()
        while alive:
            if drop_tol < 0:
                best = alive[0]
            else:
                best = max(alive, key=lambda j: A[j, j])
            nb = math.sqrt(max(A[best, best], 0.0))
            if nb <= thresh or nb == 0.0:
                break
            alive.remove(best)
            order.append(best)
            minratio = min(minratio, nb / mx if mx else 0.0)
            for j in alive:
                for i in alive:
                    A[i, j] -= A[best, i] * A[best, j] / (nb * nb)
        r = len(order)
        R = np.linalg.cholesky(g[np.ix_(order, order)]).T if r else np.zeros((0, 0))
        Ri = np.linalg.inv(R) if r else R
        full = np.zeros((c, c))
        full[:r, :r] = Ri
        rinv.copy_(torch.from_numpy(full).reshape(rinv.shape) if rinv.numel() == c * c
                   else torch.from_numpy(full[: rinv.shape[0], : rinv.shape[1]]))
        p = np.zeros(perm.numel(), dtype=np.int32)
        p[:r] = order[: perm.numel()]
        perm.copy_(torch.from_numpy(p))
        info.copy_(torch.tensor([float(r), minratio, mx], dtype=torch.float64))

    def perm_rows(self, perm, rinv, info, out):
        c = out.shape[0]
        r = int(info[0])
        b = np.zeros((c, c))
        p = perm.numpy().astype(np.int64)
        b[p[:r], :r] = rinv.numpy().reshape(-1)[: c * c].reshape(c, c)[:r, :r]
        out.copy_(torch.from_numpy(b))
        return out

    def dense_update(self, X, eta, F, lams):
        raise NotImplementedError

    # ---- operator / constraints
    def apply(self, which, V, out, gram=None):
        return self.dp.apply(which, V, out=out, gram=gram)

    def image(self, V, S, out, s_is_diag=False, s_scale=1.0, beta=0.0, beta_dev=None, base=None):
        if self.dp.entries:  # owned constraints on the allgathered basis
            v, fam = self.dp.full_rows(V).numpy(), self.dp.owned_family
            k = v.shape[1]
            if s_is_diag:
                img = O.image_factor(fam, v, s_scale * S.numpy().reshape(-1)[:k])
            else:
                img = O.image_lowrank(fam, v, s_scale * S.numpy())
            img = img[: self.m]
        elif s_is_diag:
            v = V.numpy()
            img = (v * v) @ (s_scale * S.numpy().reshape(-1)[: v.shape[1]])
        else:
            v = V.numpy()
            img = np.einsum("ij,jk,ik->i", v, s_scale * S.numpy(), v)
        bt = beta * (float(beta_dev[0]) if beta_dev is not None else 1.0)
        res = img + (bt * base.numpy() if base is not None else 0.0)
        out.copy_(torch.from_numpy(np.asarray(res, dtype=float)))
        return out

    def compressed(self, V, scale_gram=0.0, gram_out=None, a=None, scale_a=0.0, a_out=None, w=None, scale_w=0.0,
                   w_out=None):
        if self.dp.entries:  # rows of the owned constraints, allgathered basis
            cm = O.compressed(self.dp.owned_family, self.dp.full_rows(V).numpy())[: self.m]
        else:
            cm = O.compressed(object(), V.numpy())  # diagonal family: rows svec(v_i v_i^T)
        if gram_out is not None:
            gram_out.copy_(torch.from_numpy(scale_gram * cm.T @ cm))
            self._ar(gram_out)
        if a is not None:
            a_out.copy_(torch.from_numpy(scale_a * cm.T @ a.numpy()))
            self._ar(a_out)
        if w is not None:
            w_out.copy_(torch.from_numpy(scale_w * cm.T @ w.numpy()))
            self._ar(w_out)

    # ---- ipm (oracle)
    def state_len(self, k):
        return 2 * k * k + 7

    def ipm(self, k, has_eta, Q11, q12, lin_s, scal, warm, state_out, result, opts=None):
        d = k * (k + 1) // 2
        q22, le = (float(x) for x in scal.numpy()[:2])
        q = O.Coeffs(Q11.numpy().copy() if Q11 is not None else np.zeros((d, d)),
                     q12.numpy().copy() if q12 is not None else np.zeros(d), q22 if has_eta else 0.0,
                     lin_s.numpy().copy(), le if has_eta else 0.0, bool(has_eta), k)
        ws = None
        if warm is not None:
            w = warm.numpy()
            if w[2 * k * k + 6] != 0.0 and int(w[2 * k * k + 5]) == k and int(w[2 * k * k + 4]) == int(has_eta):
                ws = O.IpState(w[:k * k].reshape(k, k).copy(), float(w[2 * k * k]), w[k * k:2 * k * k].reshape(k, k).copy(),
                               float(w[2 * k * k + 1]), float(w[2 * k * k + 2]), float(w[2 * k * k + 3]), bool(has_eta))
        o = O.IpmOpts(*opts) if opts is not None else O.IpmOpts()
        o.max_newton, o.max_step_failures = int(o.max_newton), int(o.max_step_failures)
        r = O.ipm(q, ws, o)
        st = r.state
        vec = np.concatenate([st.s_mat.ravel(), st.t_mat.ravel(),
                              [st.eta, st.zeta, st.omega, st.mu, float(has_eta), float(k), 1.0]])
        state_out.copy_(torch.from_numpy(vec))
        result[:5].copy_(torch.tensor([r.value, float(r.newton_iters), float(r.exact), r.eta_opt, 0.0]))
