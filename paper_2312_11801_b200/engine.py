"""Thin typed wrappers over the C-ABI for device tensors (torch float64 CUDA
tensors as buffers).  Every method is one or two library calls; nothing
here computes on the host or with eager PyTorch ops."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from ._native import check, ptr
from .runtime import DeviceProblem, Runtime


def _p(t):
    # device tensors only: the raw address goes straight into ctypes (the
    # c_void_p argtype converts ints in C; no per-argument wrapper objects)
    return None if t is None else t.data_ptr()


class Engine:
    """comm (dist.Comm or None): when the problem is row-sharded, every
    reduction over the n/m dimension is completed with an allreduce, so the
    callers (solver.py) are identical for 1 and N GPUs."""

    def __init__(self, dp: DeviceProblem, comm=None, h=None):
        self.dp = dp
        self.rt: Runtime = dp.rt
        self.lib = self.rt.lib
        self.h = h or self.rt.h  # context (and therefore stream) the kernels go to
        self.n, self.m = dp.n, dp.m
        self.comm = comm if (comm is not None and comm.world > 1) else None
        self._red2 = None

    # ---------------------------------------------------------------- vectors
    def vec(self, op, m, x=None, y=None, z=None, b=None, ineq=None, s0=0.0, s1=0.0, out=None, red=None):
        if self.comm is not None and red is not None and op == N.VOP_DOTAFF:
            if self._red2 is None:
                self._red2 = self.rt.zeros(2)
            check(self.lib.usbs_vec(self.h, N.VOP_DOT, int(m), _p(x), _p(y), None, None, None, 0.0, 0.0, None,
                                    _p(self._red2)), "vec")
            self.comm.allreduce_sum(self._red2[0:1])
            red[0:1].copy_(self._red2[0:1] * s0 + s1)
            return
        check(self.lib.usbs_vec(self.h, op, int(m), _p(x), _p(y), _p(z), _p(b), _p(ineq), float(s0), float(s1),
                                _p(out), _p(red)), "vec")
        if self.comm is not None and red is not None:
            self.comm.allreduce_sum(red[0:1])
            self.comm.allreduce_max(red[1:2])

    def dot_into(self, x, y, red, scale=1.0, shift=0.0):
        """red[0] = scale * <x, y> + shift (device scalar)."""
        self.vec(N.VOP_DOTAFF, x.numel(), x=x, y=y, s0=scale, s1=shift, red=red)

    # ---------------------------------------------------------------- dense
    def rowgemm(self, X, B, Y, alpha=1.0, beta=0.0, Y0=None, xs=None, n=None):
        n = X.shape[0] if n is None else n
        ka = X.shape[1]
        kb = B.shape[1]
        check(self.lib.usbs_rowgemm(self.h, int(n), _p(X), X.stride(0), ka, _p(B), B.stride(0), kb, _p(xs),
                                    float(alpha), float(beta), _p(Y0), Y0.stride(0) if Y0 is not None else 0,
                                    _p(Y), Y.stride(0)), "rowgemm")
        return Y

    def gram(self, A, B, out, sym=False):
        check(self.lib.usbs_gram(self.h, A.shape[0], _p(A), A.stride(0), A.shape[1], _p(B), B.stride(0),
                                 B.shape[1], _p(out), 1 if sym else 0), "gram")
        if self.comm is not None:  # sym(sum of partials) == sum of sym(partials)
            self.comm.allreduce_sum(out)
        return out

    def wcoldot(self, F, G, w, out):
        check(self.lib.usbs_wcoldot(self.h, F.shape[0], _p(F), F.stride(0), _p(G), G.stride(0), F.shape[1],
                                    _p(w), _p(out)), "wcoldot")
        if self.comm is not None:
            self.comm.allreduce_sum(out[0:1])

    # ---------------------------------------------------------------- sharded Lanczos
    def lz_step_finish(self, j, m1, c1, c2, nrm2, H, flags, w, q):
        """Step epilogue of the row-sharded Lanczos (usbs_lz_step_finish):
        H column j, beta, q_{j+1} = w / beta on the local rows, flags."""
        check(self.lib.usbs_lz_step_finish(self.h, int(j), int(m1), _p(c1), _p(c2), _p(nrm2), _p(H), _p(flags),
                                           _p(w), w.shape[0], w.stride(0), _p(q), q.stride(0)), "lz_step_finish")

    def lz_restart_h(self, m1, ell, theta, H):
        check(self.lib.usbs_lz_restart_h(self.h, int(m1), int(ell), _p(theta), _p(H)), "lz_restart_h")

    def small_eigh(self, a, vals, vecs):
        check(self.lib.usbs_small_eigh(self.h, a.shape[0], _p(a), _p(vals), _p(vecs)), "small_eigh")

    def pivchol(self, G, drop_tol, perm, rinv, info):
        check(self.lib.usbs_pivchol(self.h, G.shape[0], _p(G), float(drop_tol), _p(perm), _p(rinv), _p(info)),
              "pivchol")

    def perm_rows(self, perm, rinv, info, out):
        check(self.lib.usbs_perm_rows(self.h, out.shape[0], _p(perm), _p(rinv), _p(info), _p(out)), "perm_rows")
        return out

    def gather_rows(self, idx, src, out):
        """out[i] = src[idx[i]] row-wise, zero rows where idx[i] < 0."""
        k = out.shape[1]
        check(self.lib.usbs_gather_rows(self.h, out.shape[0], k, _p(idx), _p(src), src.stride(0), _p(out),
                                        out.stride(0)), "gather_rows")
        return out

    def svec(self, A, out, scale=1.0):
        check(self.lib.usbs_svec(self.h, A.shape[0], _p(A), float(scale), _p(out)), "svec")
        return out

    def dense_update(self, X, eta, F, lams):
        if self.comm is not None:
            raise NotImplementedError("the explicit n x n store is not sharded; use sketch_rank > 0")
        check(self.lib.usbs_dense_update(self.h, X.shape[0], _p(X), float(eta), _p(F), F.stride(0), F.shape[1],
                                         _p(lams)), "dense_update")

    # ---------------------------------------------------------------- operator / constraints
    def apply(self, which, V, out, gram=None):
        if self.h is not self.rt.h:
            return self.dp.apply(which, V, out=out, gram=gram, h=self.h)
        return self.dp.apply(which, V, out=out, gram=gram)

    def _cons_operands(self, V):
        f = getattr(self.dp, "image_operands", None)
        return f(V) if f is not None else (self.dp.h, V)

    def image(self, V, S, out, s_is_diag=False, s_scale=1.0, beta=0.0, beta_dev=None, base=None):
        hp, V = self._cons_operands(V)
        check(self.lib.usbs_cons_image(self.h, hp, _p(V), V.stride(0), V.shape[1], _p(S),
                                       1 if s_is_diag else 0, float(s_scale), _p(beta_dev), float(beta), _p(base),
                                       _p(out)), "cons_image")
        return out

    def compressed(self, V, scale_gram=0.0, gram_out=None, a=None, scale_a=0.0, a_out=None, w=None, scale_w=0.0,
                   w_out=None):
        hp, V = self._cons_operands(V)
        check(self.lib.usbs_cons_compressed(self.h, hp, _p(V), V.stride(0), V.shape[1], float(scale_gram),
                                            _p(gram_out), _p(a), float(scale_a), _p(a_out), _p(w), float(scale_w),
                                            _p(w_out)), "cons_compressed")
        if self.comm is not None:
            for t in (gram_out, a_out if a is not None else None, w_out if w is not None else None):
                if t is not None:
                    self.comm.allreduce_sum(t)

    # ---------------------------------------------------------------- ipm
    def ipm(self, k, has_eta, Q11, q12, lin_s, scal, warm, state_out, result, opts=None):
        o = None
        if opts is not None:
            arr = (C.c_double * 8)(*opts)
            o = arr
        check(self.lib.usbs_ipm_solve(self.h, int(k), 1 if has_eta else 0, _p(Q11), _p(q12), _p(lin_s),
                                      _p(scal), _p(warm), _p(state_out), _p(result), o), "ipm_solve")

    def state_len(self, k):
        return int(self.lib.usbs_ipm_state_len(int(k)))
