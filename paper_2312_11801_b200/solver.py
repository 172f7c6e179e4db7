"""Device-resident USBS outer loop: the drop-in for specbundle.solve.

Mirrors bundle.py:426-529 (solve), 390-423 (cold_start), 285-341
(model_update), 344-372 (compute_residuals), 212-261 (penalized_obj,
candidate_iterate, descent_test) and subqp.py:455-614 (coefficient
assembly, alternating_max) with every n- and m-sized array and every k x k
solve on the GPU.  The host keeps only control flow and the scalars the
reference branches on (lambda_max, f(y), model value, residuals, the
alternating-pass stop test), fetched in a few small D2H copies per
iteration.

Configuration objects are duck-typed: a reference ``SolverConfig`` (with
``lanczos`` and ``ipm`` members) or this module's ``SolverConfig`` work.
"""
from __future__ import annotations

import dataclasses
import math
import os
import time
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _native as N
from ._native import check
from .eigen import DeviceLinOp, lanczos_top
from .engine import Engine
from .errors import EmptyBasisError
from .runtime import DeviceProblem, runtime


def _device_loop_enabled() -> bool:
    """USBS_DEVICE_LOOP=0 keeps the host-driven alternating loop (A/B, debugging)."""
    return os.environ.get("USBS_DEVICE_LOOP", "1") != "0"

__all__ = ["LanczosSettings", "IpmOptions", "SolverConfig", "AggregateStats", "Residuals", "SolverState",
           "IterationInfo", "PrimalOutput", "DeviceSolver", "solve"]


# ---------------------------------------------------------------------------
# configuration (bundle.py:64-91, subqp.py:150-162)


@dataclass
class LanczosSettings:
    inner_iters: int = 32
    max_restarts: int = 10
    tol: Optional[float] = None


@dataclass
class IpmOptions:
    mu_tol: float = 1e-11
    kkt_tol: float = 1e-6
    max_newton: int = 100
    step_frac: float = 0.99
    backtrack: float = 0.8
    min_step: float = 1e-12
    max_step_failures: int = 6
    warm_blend: float = 0.2


@dataclass
class SolverConfig:
    rho: float = 0.01
    beta: float = 0.25
    k_c: int = 10
    k_p: int = 1
    eps: float = 1e-3
    sketch_rank: int = 0
    max_iters: int = 1000
    max_time: Optional[float] = None
    seed: int = 0
    lanczos: LanczosSettings = field(default_factory=LanczosSettings)
    linf_check: bool = False
    store_psi: bool = True
    ipm: IpmOptions = field(default_factory=IpmOptions)

    def __post_init__(self):
        if not (self.rho > 0 and 0 < self.beta < 1 and self.k_c >= 1 and self.k_p >= 0):
            raise ValueError("invalid solver configuration")
        if self.eps <= 0 or self.sketch_rank < 0:
            raise ValueError("invalid solver configuration")


def _ipm_opts(cfg):
    o = getattr(cfg, "ipm", None) or IpmOptions()
    return [o.mu_tol, o.kkt_tol, o.max_newton, o.step_frac, o.backtrack, o.min_step, o.max_step_failures,
            o.warm_blend]


# ---------------------------------------------------------------------------
# state records (bundle.py:94-205); arrays live on the device, numpy on demand


@dataclass
class AggregateStats:
    trace: float
    cost_ip: float
    constr_image_dev: object

    @property
    def constr_image(self) -> np.ndarray:
        return self.constr_image_dev.cpu().numpy()


@dataclass
class Residuals:
    rel_subopt: float
    rel_infeas: float
    linf_infeas: float
    dual_gap: float
    dual_feas: float

    def converged(self, eps: float, linf_check: bool = False) -> bool:
        ok = self.rel_subopt <= eps and self.rel_infeas <= eps and self.dual_feas <= eps
        if linf_check:
            ok = ok and self.linf_infeas <= eps
        return ok


_PSI_POOL = None


def make_test_matrix_rows(n, r, seed, r0, r1) -> np.ndarray:
    """Rows [r0, r1) of make_test_matrix(n, r, seed) (sketch.py:25-27),
    filled by the library's native restatement of numpy's legacy generator
    (usbs_make_test_matrix, bit-identical; the ctypes call releases the GIL,
    so the fill overlaps the Python-side setup instead of contending with
    it)."""
    from ._native import check, load
    out = np.empty((r1 - r0, r), dtype=np.float64)
    check(load().usbs_make_test_matrix(int(seed), int(n), int(r), int(r0), int(r1), out.ctypes.data),
          "make_test_matrix")
    return out


def _psi_async(n, r, seed, r0, r1):
    global _PSI_POOL
    if _PSI_POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _PSI_POOL = ThreadPoolExecutor(max_workers=1, thread_name_prefix="usbs-psi")
    return _PSI_POOL.submit(make_test_matrix_rows, n, r, seed, r0, r1)


# tall factors from this many rows on take the device thin SVD at exit
DEVICE_SVD_MIN_ROWS = 65536


def thin_svd_device(eng, B):
    """Thin SVD of a tall device matrix B (n x c) as U (host) and the singular
    values: CholQR2 on the device (two Gram + row-GEMM rounds, B = Q R with
    R = R2 R1, both Cholesky factors from the c x c Grams on the host), then
    LAPACK's SVD of the c x c R on the host and U = Q U_R on the device --
    the O(n c^2) work on the GPU, O(c^3) on the host (the reference's
    np.linalg.svd of the whole n x c factor costs ~0.2 s at n = 10^6).
    Column signs follow LAPACK's SVD of R, not of B (singular vectors are
    defined up to sign; the sign-insensitive MaxCut rounding is the large-n
    use).  Returns None when a Gram is not numerically positive definite
    (condition number beyond CholQR2's ~1e8), and the caller falls back to
    the host SVD."""
    import scipy.linalg as sla

    rt = eng.rt
    n, c = B.shape
    G = rt.empty(c, c)
    eng.gram(B, B, G, sym=True)
    try:
        r1 = np.linalg.cholesky(G.cpu().numpy()).T  # G = R1^T R1
    except np.linalg.LinAlgError:
        return None
    eye = np.eye(c)
    Q1 = eng.rowgemm(B, rt.upload(sla.solve_triangular(r1, eye)), rt.empty(n, c))
    eng.gram(Q1, Q1, G, sym=True)
    try:
        r2 = np.linalg.cholesky(G.cpu().numpy()).T
    except np.linalg.LinAlgError:
        return None
    ur, sv, _ = np.linalg.svd(r2 @ r1)
    U = eng.rowgemm(Q1, rt.upload(sla.solve_triangular(r2, eye) @ ur), rt.empty(n, c))
    return U.cpu().numpy(), sv


class DeviceSketchStore:
    """SketchStore + sketch.py on the device: P (n x r), Psi (n x r)."""

    def __init__(self, eng: Engine, n: int, r: int, seed: int, psi_host: Optional[np.ndarray] = None,
                 rows: Optional[tuple] = None, shard=None, comm=None, psi_job=None):
        """n is the global dimension; rows = (r0, r1) selects this rank's
        block of Psi and P when the problem is row-sharded."""
        if not 1 <= r <= n:
            raise ValueError(f"sketch rank {r} must lie in [1, {n}]")
        self.eng, self.n, self.r, self.psi_seed = eng, n, r, int(seed)
        self.shard, self.comm = shard, comm
        r0, r1 = rows if rows is not None else (0, n)
        rt = eng.rt
        self._psi = None
        self._psi_job = None
        if psi_job is not None:
            self._psi_job = psi_job
        elif psi_host is None:
            # make_test_matrix (sketch.py:25-27): legacy MT19937 normals on the
            # host (bit-exact with the reference), generated on a worker thread
            # (numpy releases the GIL while filling) so it overlaps the cold
            # start; joined at the first use
            self._psi_job = _psi_async(n, r, seed, r0, r1)
        else:
            self._psi = rt.upload(psi_host)
        self.P = rt.zeros(r1 - r0, r)
        self.G = rt.empty(64, max(r, 1))

    @property
    def psi(self):
        if self._psi is None:
            self._psi = self.eng.rt.upload(self._psi_job.result())
            self._psi_job = None
        return self._psi

    def update(self, eta: float, F, lams) -> None:
        """sketch_update with Q = I (sketch.py:58-74): P <- eta P + (F L)(F^T Psi)."""
        if eta < 0:
            raise ValueError("eta must be nonnegative")
        kc = F.shape[1]
        G = self.G[:kc]
        self.eng.gram(F, self.psi, G)
        self.eng.rowgemm(F, G, self.P, alpha=1.0, beta=float(eta), Y0=self.P, xs=lams)

    @property
    def sketch_mat(self) -> np.ndarray:
        return self.P.cpu().numpy()

    def factorize(self):
        """reconstruct (sketch.py:77-111): shift, core Gram, Cholesky and the
        triangular solve on the device; the final thin SVD of the n x r
        factor runs on the host at exit (LAPACK sign conventions)."""
        eng, rt, n, r = self.eng, self.eng.rt, self.n, self.r
        sc = rt.zeros(4)
        eng.dot_into(self.P.view(-1), self.P.view(-1), sc[0:1])
        norm_p = math.sqrt(float(sc[0].item()))
        if norm_p == 0.0:
            u = np.zeros((n, r))
            u[:r, :r] = np.eye(r)
            return u, np.zeros(r)
        shift = math.sqrt(n) * np.finfo(float).eps * norm_p
        nl = self.P.shape[0]  # local rows (== n unless sharded)
        ps = rt.empty(nl, r)
        eng.vec(N.VOP_AXPBY, nl * r, x=self.P.view(-1), y=self.psi.view(-1), s0=1.0, s1=shift, out=ps.view(-1))
        core = rt.empty(r, r)
        eng.gram(self.psi, ps, core, sym=True)
        perm = rt.torch.zeros(r, dtype=rt.torch.int32, device=rt.device)
        rinv = rt.zeros(r, r)
        info = rt.zeros(3)
        eng.pivchol(core, -1.0, perm, rinv, info)
        if int(info[0].item()) == r and float(info[1].item()) > 0.0:
            half = eng.rowgemm(ps, rinv, rt.empty(nl, r))
        else:  # rank-deficient core: eigenvalue pseudo-inverse (sketch.py:100-108)
            vals, vecs = rt.empty(r), rt.empty(r, r)
            eng.small_eigh(core, vals, vecs)
            w = vals.cpu().numpy()[::-1].copy()
            qm = vecs.cpu().numpy()[:, ::-1].copy()
            keep = w > max(w.max(initial=0.0), 0.0) * 1e-14
            if not np.any(keep):
                u = np.zeros((n, r))
                u[:r, :r] = np.eye(r)
                return u, np.zeros(r)
            B = rt.upload(qm[:, keep] / np.sqrt(w[keep])[None, :])
            half = eng.rowgemm(ps, B, rt.empty(nl, int(keep.sum())))
        if self.shard is not None and self.comm is not None and self.comm.world > 1:
            full = rt.empty(n, half.shape[1])
            self.comm.allgather_rows(half, full, self.shard)
            half = full
        elif half.shape[0] >= DEVICE_SVD_MIN_ROWS and not os.environ.get("USBS_HOST_SVD"):
            res = thin_svd_device(eng, half)
            if res is not None:
                u, sv = res
                return u, np.maximum(sv ** 2 - shift, 0.0)
        u, sv, _ = np.linalg.svd(half.cpu().numpy(), full_matrices=False)
        return u, np.maximum(sv ** 2 - shift, 0.0)


class DeviceExplicitStore:
    """ExplicitStore (bundle.py:104-117) with Xbar on the device."""

    def __init__(self, eng: Engine, n: int):
        self.eng = eng
        self.X = eng.rt.zeros(n, n)

    def update(self, eta: float, F, lams) -> None:
        self.eng.dense_update(self.X, eta, F, lams)

    @property
    def xbar(self) -> np.ndarray:
        return self.X.cpu().numpy()

    def factorize(self):
        x = self.xbar
        vals, vecs = np.linalg.eigh(0.5 * (x + x.T))
        vals, vecs = vals[::-1].copy(), vecs[:, ::-1].copy()
        keep = vals > max(vals.max(initial=0.0), 0.0) * 1e-12
        if not np.any(keep):
            return np.eye(x.shape[0], 1), np.zeros(1)
        return vecs[:, keep], vals[keep]


@dataclass
class BundleModel:
    basis_dev: object
    stats: AggregateStats
    k_c: int
    k_p: int
    store: object

    @property
    def basis(self) -> np.ndarray:
        return self.basis_dev.cpu().numpy()

    @property
    def k(self) -> int:
        return self.basis_dev.shape[1]


@dataclass
class SolverState:
    y_dev: object
    nu_dev: object
    f_y: Optional[float]
    lam_y: Optional[float]
    model: BundleModel
    descent_steps: int = 0
    null_steps: int = 0
    iterations: int = 0
    last_primal: Optional[AggregateStats] = None
    residuals: Optional[Residuals] = None
    status: Optional[str] = None
    scale_x: float = 1.0
    scale_c: float = 1.0
    best_rel_infeas: float = np.inf
    best_rel_subopt: float = np.inf
    device_problem: Optional[object] = field(default=None, repr=False, compare=False)

    @property
    def y(self) -> np.ndarray:
        return self.y_dev.cpu().numpy()

    @property
    def nu(self) -> np.ndarray:
        return self.nu_dev.cpu().numpy()


@dataclass
class IterationInfo:
    """bundle.IterationInfo (bundle.py:180-198); m-vectors download lazily."""

    t: int
    elapsed: float
    step: str
    f_y: float
    f_cand: float
    model_val: float
    y_dev: object
    y_cand_dev: object
    nu_cand_dev: object
    residuals: Residuals
    primal: AggregateStats
    eta: float
    lam_cand: float
    state: SolverState
    model: BundleModel
    alt_passes: int = 0
    lanczos_matvecs: int = 0
    lanczos_restarts: int = 0

    @property
    def y(self):
        return self.y_dev.cpu().numpy()

    @property
    def y_cand(self):
        return self.y_cand_dev.cpu().numpy()

    @property
    def nu_cand(self):
        return self.nu_cand_dev.cpu().numpy()


@dataclass
class PrimalOutput:
    factor: np.ndarray
    lams: np.ndarray
    dense: Optional[np.ndarray] = None


# scalar slots of the device scratch vector
S_Q22, S_LINETA, S_EQ22, S_ELINETA, S_DNU, S_CQS, S_BYC, S_RES, S_BY, S_MINI, S_CFIP, S_PSI = (0, 1, 2, 3, 4, 6, 8, 10, 12,
                                                                           14, 16, 20)


def orthonormalize_dev(eng: Engine, A, drop_tol: float = 1e-12):
    """symlin.orthonormalize (symlin.py:148-190) on device tensors: pivot order
    and drop rule from a pivoted Cholesky of the Gram, then CholQR2 (the
    second pass speculatively issued for full rank, so the common case costs
    one round trip).  Falls back to the exact column-pivoted Gram-Schmidt when
    a selected residual is below 1e-6 of the largest column or a column is
    dropped: there a Gram cannot resolve the drop rule."""
    rt = eng.rt
    n, c = A.shape
    # scratch reused across calls (usbs_pivchol writes every entry of its
    # outputs); the result is a fresh tensor (callers keep bases around)
    cache = eng.__dict__.setdefault("_orth_scratch", {})
    key = (n, c)
    if key not in cache:
        i32 = rt.torch.int32
        cache[key] = {"G": rt.empty(c, c), "perm": rt.torch.zeros(c, dtype=i32, device=rt.device),
                      "rinv": rt.zeros(c, c), "info": rt.zeros(3), "B": rt.empty(c, c), "Y": rt.empty(n, c),
                      "G2": rt.empty(c, c), "perm2": rt.torch.zeros(c, dtype=i32, device=rt.device),
                      "rinv2": rt.zeros(c, c), "info2": rt.zeros(3)}
    sc = cache[key]
    G, perm, rinv, info = sc["G"], sc["perm"], sc["rinv"], sc["info"]
    eng.gram(A, A, G)
    eng.pivchol(G, drop_tol, perm, rinv, info)
    B = eng.perm_rows(perm, rinv, info, sc["B"])
    Y = eng.rowgemm(A, B, sc["Y"])
    G2 = sc["G2"]
    eng.gram(Y, Y, G2)
    eng.pivchol(G2, -1.0, sc["perm2"], sc["rinv2"], sc["info2"])
    Q = eng.rowgemm(Y, sc["rinv2"], rt.empty(n, c))
    info_h = info.cpu().numpy()
    r = int(info_h[0])
    if info_h[2] == 0.0:
        raise EmptyBasisError("all input columns are zero")
    if r == 0:
        raise EmptyBasisError("all input columns are numerically dependent")
    if info_h[1] < 1e-6 or r < c:
        # a selected residual below what a Gram resolves, or dropped columns
        # (whose true residual the Gram cannot tell from the 1e-12 rule)
        return _gs_exact_dev(eng, A, drop_tol)
    return Q


def _gs_exact_dev(eng: Engine, A, drop_tol: float = 1e-12):
    """Column-pivoted two-pass Gram-Schmidt on device primitives."""
    rt = eng.rt
    n, c = A.shape
    ident = rt.upload(np.eye(c))
    work = rt.empty(n, c)
    eng.rowgemm(A, ident, work)
    G = rt.empty(c, c)
    eng.gram(work, work, G)
    norms = np.sqrt(np.maximum(np.diag(G.cpu().numpy()), 0.0))
    thresh = drop_tol * float(norms.max())
    alive = list(range(c))
    basis = rt.empty(n, c)
    nb = 0
    coef = rt.empty(c, c)
    red = rt.zeros(2)
    while alive:
        eng.gram(work, work, G)
        g = G.cpu().numpy()
        nr = np.sqrt(np.maximum(np.array([g[j, j] for j in alive]), 0.0))
        pick = int(np.argmax(nr))
        if nr[pick] <= thresh:
            break
        piv = alive.pop(pick)
        q = rt.empty(n, 1)
        eng.rowgemm(work[:, piv:piv + 1], ident[:1, :1], q)
        if nb:
            Bm = basis[:, :nb]
            cv = coef.view(-1)[:nb].view(nb, 1)  # gram writes a contiguous block
            eng.gram(Bm, q, cv)
            eng.rowgemm(Bm, cv, q, alpha=-1.0, beta=1.0, Y0=q)
        eng.dot_into(q.view(-1), q.view(-1), red)
        nq = math.sqrt(float(red[0].item()))
        if nq <= thresh:
            continue
        eng.rowgemm(q, ident[:1, :1], basis[:, nb:nb + 1], alpha=1.0 / nq)
        qb = basis[:, nb:nb + 1]
        nb += 1
        for j in alive:
            col = work[:, j:j + 1]
            eng.gram(qb, col, coef[:1, :1])
            eng.rowgemm(qb, coef[:1, :1], col, alpha=-1.0, beta=1.0, Y0=col)
    if nb == 0:
        raise EmptyBasisError("all input columns are numerically dependent")
    out = rt.empty(n, nb)
    eng.rowgemm(basis[:, :nb], ident[:nb, :nb], out)
    return out


class DeviceSolver:
    """Holds the uploaded problem and scratch buffers for one solve."""

    def __init__(self, prob, cfg, dprob: Optional[DeviceProblem] = None, comm=None, engine=None):
        self.prob = prob
        self.cfg = cfg
        # the sketch test matrix (host, legacy MT19937) is generated while the
        # problem is uploaded and planned and the cold-start Lanczos runs
        self._psi_job = None
        if getattr(cfg, "sketch_rank", 0) > 0 and (dprob is None or getattr(dprob, "shard", None) is None):
            n0 = int(prob.n)
            self._psi_job = _psi_async(n0, min(int(cfg.sketch_rank), n0),
                                       int(np.random.SeedSequence(int(cfg.seed)).generate_state(2)[0]), 0, n0)
        self.dp = dprob or DeviceProblem(prob)
        self.comm = comm
        self.eng = engine or Engine(self.dp, comm)
        self.rt = self.dp.rt
        self.n, self.m = self.dp.n, self.dp.m
        # row sharding (dist.py): local rows [r0, r1) of the global n
        self.shard = getattr(self.dp, "shard", None)
        self.n_global = int(prob.n)
        self.r0 = self.shard.r0 if self.shard is not None else 0
        self.r1 = self.shard.r1 if self.shard is not None else self.n
        self.alpha = float(prob.alpha)
        self.b = self.dp.b
        self.ineq = self.dp.ineq
        self.has_ineq = self.dp.has_ineq
        self.b_norm = float(np.linalg.norm(np.asarray(prob.b, dtype=float)))
        # the scalars the host reads each iteration live in one buffer, so a
        # single D2H fetches them (sc 0:64, res_q 64:72, res_e 72:80, a k-vector
        # slot 80:144, lamc 144:208)
        self._scratch = self.rt.zeros(208)
        on_gpu = self._scratch.is_cuda
        self._scratch_h = self.rt.torch.empty(208, dtype=self.rt.torch.float64, pin_memory=on_gpu)
        self.sc = self._scratch[:64]
        self.opts = _ipm_opts(cfg)
        lz = getattr(cfg, "lanczos", None) or LanczosSettings()
        self.lz = (int(lz.inner_iters), int(lz.max_restarts), lz.tol)
        self.seed = int(cfg.seed)
        self.k_c = min(cfg.k_c, self.n_global)
        self.k_p = min(cfg.k_p, self.n_global - self.k_c)
        k = self.k_c + self.k_p
        self.k = k
        # device limits, checked up front (not at the first subproblem):
        # the k x k master problem (k_ipm) and the Lanczos basis (m <= 64)
        if k > 32:
            raise ValueError(f"k_c + k_p = {k} exceeds the device IPM limit of 32")
        m_lz = max(int(lz.inner_iters), self.k_c + 1, 2)
        if m_lz > 64 and m_lz < self.n_global:
            raise ValueError(f"Lanczos basis size {m_lz} exceeds the device limit of 64")
        rt = self.rt
        n, m = self.n, self.m
        self.tmp_nk = rt.empty(n, max(k, 1))
        self.tmp_nk2 = rt.empty(n, max(k, 1))
        self.vecs = rt.empty(n, max(self.k_c, 1))
        self.wv = rt.empty(m)
        self.nu_a = rt.empty(m)
        self.nu_b = rt.empty(m)
        self.loop_cnt = None  # device int32: passes run by the device loop (lazy)
        self.device_loop = _device_loop_enabled() and getattr(rt, "lib", None) is not None
        self.ax = rt.empty(m)
        self.ycand = rt.empty(m)
        d = k * (k + 1) // 2
        self.d = d
        self.Q11 = rt.empty(d, d)
        self.q12 = rt.empty(d)
        self.lin_s = rt.empty(d)
        self.csv = rt.empty(d)
        self.cq = rt.empty(k, k)
        self.zq = rt.empty(k, k)
        sl = self.eng.state_len(k)
        self.st_q = rt.zeros(sl)
        self.st_e = rt.zeros(sl)
        self.res_q = self._scratch[64:72]
        self.res_e = self._scratch[72:80]
        self.s_act = rt.empty(k, k)
        self.evals = rt.empty(k)
        self.evecs = rt.empty(k, k)
        self.lamc = self._scratch[144:144 + max(self.k_c, 1)] if self.k_c <= 64 else rt.empty(self.k_c)
        self.ident = rt.upload(np.eye(max(k, 1)))
        self.lz_probe = None  # list -> (start, end, restarts, matvecs) per Lanczos call
        # overlap the model-evaluation IPM with the Lanczos kernel (single GPU,
        # CUDA runtime only; USBS_NO_OVERLAP=1 disables it)
        import os
        self.overlap = (self.shard is None and engine is None and hasattr(self.rt, "aux")
                        and not os.environ.get("USBS_NO_OVERLAP"))
        self.eng_aux = Engine(self.dp, None, h=self.rt.aux()[1]) if self.overlap else None

    # ------------------------------------------------------------ helpers
    def _fetch(self, *tensors):
        """One synchronising D2H of several small device arrays."""
        return [t.cpu().numpy() for t in tensors]

    def _fetch_scratch(self, upto: int) -> np.ndarray:
        """The first `upto` entries of the scalar buffer in one synchronising
        D2H (pinned)."""
        h = self._scratch_h[:upto]
        if self._scratch.is_cuda:
            h.copy_(self._scratch[:upto], non_blocking=True)
            self.rt.stream.synchronize()
        else:  # the CPU stand-in of the multi-process tests
            h.copy_(self._scratch[:upto])
        return h.numpy().copy()

    def penalized_lanczos(self, y_dev, which=1, assembled=False):
        """penalized_obj (bundle.py:212-236) minus the <b,y> term (device dot)."""
        if which == 1 and not assembled:
            self.dp.assemble(y_dev)
        op = DeviceLinOp(self.dp, which)
        inner, rst, tol = self.lz
        probe = self.lz_probe
        if probe is not None:  # bench: CUDA events on the launching stream around the kernel
            ev0 = self.rt.torch.cuda.Event(enable_timing=True)
            ev1 = self.rt.torch.cuda.Event(enable_timing=True)
            ev0.record(self.rt.stream)
        if self.shard is not None:
            from .dist import lanczos_sharded
            return lanczos_sharded(self.eng, self.dp, which, self.k_c, inner, rst, tol, self.seed, out=self.vecs)
        res = lanczos_top(op, self.k_c, inner, rst, tol, self.seed, out=self.vecs)
        if probe is not None:
            ev1.record(self.rt.stream)
            probe.append((ev0, ev1, res.restarts, res.matvecs))
        return res

    def completion(self, basis, k, tag):
        """_completion_columns (bundle.py:264-282) with host PCG64 vectors."""
        rt, eng, n = self.rt, self.eng, self.n
        have = 0 if basis is None else basis.shape[1]
        out = rt.empty(n, k)
        if have:
            eng.rowgemm(basis, self.ident[:have, :have], out[:, :have])
        attempt = 0
        coef = rt.empty(k, 1)
        red = rt.zeros(2)
        while have < k:
            g = np.random.default_rng([self.seed & 0xFFFFFFFF, 0x5EED, tag, attempt])
            v = rt.upload(g.standard_normal(self.n_global)[self.r0:self.r1].reshape(n, 1))
            if have:
                cur = out[:, :have]
                eng.gram(cur, v, coef[:have])
                eng.rowgemm(cur, coef[:have], v, alpha=-1.0, beta=1.0, Y0=v)
            eng.dot_into(v.view(-1), v.view(-1), red)
            nv = math.sqrt(float(red[0].item()))
            attempt += 1
            if nv < 1e-10:
                continue
            eng.rowgemm(v, self.ident[:1, :1], out[:, have:have + 1], alpha=1.0 / nv)
            have += 1
        return out

    def orthonormalize(self, A):
        """symlin.orthonormalize (symlin.py:148-190) on the device."""
        return orthonormalize_dev(self.eng, A)

    # ------------------------------------------------------------ cold start
    def cold_start(self) -> SolverState:
        """bundle.cold_start (bundle.py:390-423)."""
        rt = self.rt
        sketch_seed = int(np.random.SeedSequence(self.seed).generate_state(2)[0])
        eig = self.penalized_lanczos(None, which=0)
        basis = self.completion(eig.eigenvectors_dev, self.k, tag=0)
        stats = AggregateStats(0.0, 0.0, rt.zeros(self.m))
        if self.cfg.sketch_rank > 0:
            job, self._psi_job = self._psi_job, None
            store = DeviceSketchStore(self.eng, self.n_global, min(self.cfg.sketch_rank, self.n_global), sketch_seed,
                                      rows=(self.r0, self.r1), shard=self.shard, comm=self.comm, psi_job=job)
        else:
            store = DeviceExplicitStore(self.eng, self.n)
        model = BundleModel(basis, stats, self.k_c, self.k_p, store)
        return SolverState(rt.zeros(self.m), rt.zeros(self.m), None, None, model,
                           last_primal=AggregateStats(0.0, 0.0, stats.constr_image_dev),
                           scale_x=float(self.prob.scale_x), scale_c=float(self.prob.scale_c))

    def state_from_arrays(self, y, nu, f_y, lam_y, basis, trace, cost_ip, image, xbar=None, sketch=None,
                          descent=0, null=0, last_primal=None, psi_seed=None) -> SolverState:
        """Device state from host arrays (a reference SolverState's fields or
        a loaded USBS state record), e.g. for warm starts and lock-step replay."""
        rt = self.rt
        if sketch is not None:
            sketch_seed = (int(np.random.SeedSequence(self.seed).generate_state(2)[0]) if psi_seed is None
                           else int(psi_seed))
            store = DeviceSketchStore(self.eng, self.n, sketch.shape[1], sketch_seed)
            store.P.copy_(rt.upload(sketch))
        elif xbar is not None:
            store = DeviceExplicitStore(self.eng, self.n)
            store.X.copy_(rt.upload(xbar))
        else:
            store = None
        stats = AggregateStats(float(trace), float(cost_ip), rt.upload(image))
        model = BundleModel(rt.upload(basis), stats, self.k_c, self.k_p, store)
        lp = stats if last_primal is None else AggregateStats(last_primal[0], last_primal[1],
                                                              rt.upload(last_primal[2]))
        return SolverState(rt.upload(y), rt.upload(nu), f_y, lam_y, model, descent_steps=int(descent),
                           null_steps=int(null), last_primal=lp, scale_x=float(self.prob.scale_x),
                           scale_c=float(self.prob.scale_c))

    # ------------------------------------------------------------ subproblem
    def alternating_max(self, model: BundleModel, y, nu0, max_passes=50, tol=1e-8, psi_trace=None):
        """subqp.alternating_max (subqp.py:552-614) + assemble_quad_coeffs
        (471-527): compressed Gram, C^T w, IPM and A(V S V^T) on device.
        psi_trace (a list) receives psi_value (subqp.py:546-549) before and
        after every nu update -- the reference's monotonicity check
        (test_subqp.py:376-409); it costs host syncs, so only tests pass it."""
        eng, rt, sc = self.eng, self.rt, self.sc
        a, rho = self.alpha, float(self.cfg.rho)
        V = model.basis_dev
        k = V.shape[1]
        tr = model.stats.trace
        has_eta = tr > 0.0
        img = model.stats.constr_image_dev
        nu = self.nu_a
        eng.vec(N.VOP_PROJN, self.m, x=nu0, ineq=self.ineq, out=nu)
        a2 = a * a
        eng.compressed(V, scale_gram=a2 / rho, gram_out=self.Q11, a=img if has_eta else None,
                       scale_a=(a2 / (rho * tr)) if has_eta else 0.0, a_out=self.q12 if has_eta else None)
        if has_eta:
            eng.dot_into(img, img, sc[S_Q22:S_Q22 + 1], scale=a2 / (rho * tr * tr))
        else:
            eng.dot_into(img[:1], img[:1], sc[S_Q22:S_Q22 + 1], scale=0.0)
        eng.apply(0, V, self.tmp_nk[:, :k], gram=self.cq)  # cost_quad = sym(V^T C V)
        eng.svec(self.cq, self.csv, scale=a)
        def enqueue_pass(nu, nxt, warm):
            """One pass of subqp.py:575-611 enqueued on the device."""
            eng.vec(N.VOP_W, self.m, x=y, y=nu, b=self.b, s0=rho, out=self.wv)
            eng.compressed(V, w=self.wv, scale_w=a, w_out=self.lin_s)
            eng.vec(N.VOP_AXPBY, self.d, x=self.lin_s, y=self.csv, s0=1.0, s1=-1.0, out=self.lin_s)
            if has_eta:
                eng.dot_into(img, self.wv, sc[S_LINETA:S_LINETA + 1], scale=a / tr,
                             shift=-(a / tr) * model.stats.cost_ip)
            else:
                eng.dot_into(img[:1], img[:1], sc[S_LINETA:S_LINETA + 1], scale=0.0)
            eng.ipm(k, has_eta, self.Q11, self.q12 if has_eta else None, self.lin_s, sc[S_Q22:S_Q22 + 2], warm,
                    self.st_q, self.res_q, self.opts)
            S = self.st_q[:k * k].view(k, k)
            eng.image(V, S, self.ax, s_scale=a, beta_dev=self.res_q[3:4] if has_eta else None,
                      beta=(a / tr) if has_eta else 0.0, base=img if has_eta else None)

        def finish_pass(nu, nxt):
            eng.vec(N.VOP_NUNEXT, self.m, x=self.ax, y=y, z=nu, b=self.b, ineq=self.ineq, s0=rho, out=nxt,
                    red=sc[S_DNU:S_DNU + 2])

        warm = None
        passes = 0
        thresh = tol * (1.0 + self.b_norm)
        # after the first pass the remaining ones run as a device-controlled
        # loop (CUDA-graph WHILE node, usbs_loop_*): no host read between
        # passes; the host-driven loop stays for sharded solves (collectives
        # between the kernels) and when psi is traced
        device_loop = (self.device_loop and eng.comm is None and psi_trace is None and self.has_ineq
                       and max_passes > 1)
        for passes in range(1, max_passes + 1):
            enqueue_pass(nu, None, warm)
            warm = self.st_q
            nxt = self.nu_b if nu is self.nu_a else self.nu_a
            if psi_trace is not None:
                from .subproblem import psi_value
                eng.dot_into(self.cq.view(-1), self.st_q[:k * k], sc[S_PSI:S_PSI + 1], scale=a)
                eta_act = a * float(self.res_q[3].item()) / tr if has_eta else 0.0
                c_x = eta_act * model.stats.cost_ip + float(sc[S_PSI].item())
                psi_trace.append(psi_value(self.dp, y, rho, c_x, self.ax, nu, engine=eng))
            finish_pass(nu, nxt)
            if psi_trace is not None:
                psi_trace.append(psi_value(self.dp, y, rho, c_x, self.ax, nxt, engine=eng))
            nu = nxt
            if not self.has_ineq:
                break
            dnu = math.sqrt(max(float(sc[S_DNU].item()), 0.0))
            if dnu <= thresh:
                break
            if device_loop:
                # passes 2.. : nu -> other -> copied back, so the body's
                # operands are the same buffers every time round
                other = self.nu_b if nu is self.nu_a else self.nu_a
                if self.loop_cnt is None:
                    import torch
                    self.loop_cnt = torch.zeros(1, dtype=torch.int32, device=rt.device)
                self.loop_cnt.zero_()
                l0 = rt.launches()
                if rt.lib.usbs_loop_begin(eng.h) != 0:
                    # no conditional graph nodes on this driver: keep the host-driven loop
                    self.device_loop = device_loop = False
                    continue
                try:
                    enqueue_pass(nu, None, self.st_q)
                    finish_pass(nu, other)
                    eng.vec(N.VOP_AXPBY, self.m, x=other, s0=1.0, s1=0.0, out=nu)
                except Exception:
                    rt.lib.usbs_loop_abort(eng.h)
                    raise
                check(rt.lib.usbs_loop_end(eng.h, sc[S_DNU:S_DNU + 1].data_ptr(), float(thresh), max_passes - 1,
                                           self.loop_cnt.data_ptr()), "loop_end")
                body = rt.launches() - l0 - 1  # captured kernels (usbs_loop_end counted the graph launch)
                done = int(self.loop_cnt.item())
                rt.note_replays(body * done - body)  # the capture counted the body once
                passes = 1 + done
                break
        eng.dot_into(self.cq.view(-1), self.st_q[:k * k], sc[S_CQS:S_CQS + 1], scale=a)
        return nu, passes, has_eta

    # ------------------------------------------------------------ model update
    def model_update(self, model: BundleModel, eta, new_vecs, tag):
        """bundle.model_update (bundle.py:285-341) on device; returns the new
        model with trace/cost statistics still pending (finalised at the
        residual sync)."""
        eng, rt = self.eng, self.rt
        kp, kc = model.k_p, model.k_c
        V = model.basis_dev
        k = V.shape[1]
        eng.small_eigh(self.s_act, self.evals, self.evecs)
        eng.vec(N.VOP_RELU, kc, x=self.evals[kp:], out=self.lamc[:kc])
        lamc = self.lamc[:kc]
        F = self.tmp_nk[:, :kc]
        eng.rowgemm(V, self.evecs[:, kp:], F)
        CF = self.tmp_nk2[:, :kc]
        eng.apply(0, F, CF)
        eng.wcoldot(F, CF, lamc, self.sc[S_CFIP:S_CFIP + 1])
        # every model owns its image (the reference's BundleModel owns its
        # arrays): a fresh tensor, never the previous model's or the caller's
        img_new = rt.empty(self.m)
        eng.image(F, lamc, img_new, s_is_diag=True, beta=eta, base=model.stats.constr_image_dev)
        if model.store is not None:
            model.store.update(eta, F, lamc)
        if kp == 0:
            new_basis = rt.empty(self.n, kc)
            eng.rowgemm(new_vecs, self.ident[:kc, :kc], new_basis)
        else:
            cand = rt.empty(self.n, kp + kc)
            eng.rowgemm(V, self.evecs[:, :kp], cand[:, :kp])
            eng.rowgemm(new_vecs, self.ident[:kc, :kc], cand[:, kp:])
            try:
                new_basis = self.orthonormalize(cand)
            except EmptyBasisError:
                new_basis = None
        if new_basis is None or new_basis.shape[1] < k:
            new_basis = self.completion(new_basis, k, tag)
        pending = (eta, model.stats.trace, model.stats.cost_ip)
        stats = AggregateStats(float("nan"), float("nan"), img_new)
        return BundleModel(new_basis, stats, kc, kp, model.store), pending

    # ------------------------------------------------------------ outer loop
    def solve(self, init: Optional[SolverState] = None, callback: Optional[Callable] = None):
        """bundle.solve (bundle.py:426-529)."""
        cfg, rt, eng, sc = self.cfg, self.rt, self.eng, self.sc
        state = init if init is not None else self.cold_start()
        model = state.model
        if model.basis_dev.shape[0] != self.n or state.y_dev.shape[0] != self.m:
            raise ValueError("initial state does not match the problem dimensions")
        t_start = time.monotonic()
        y = state.y_dev.clone()  # never overwrite the caller's buffers
        if state.f_y is None or state.lam_y is None:
            if self.has_ineq:
                eng.vec(N.VOP_MINI, self.m, x=y, ineq=self.ineq, red=sc[S_MINI:S_MINI + 2])
                if float(sc[S_MINI + 1].item()) > 0.0:
                    raise ValueError("initial dual point violates the sign constraints")
            eig = self.penalized_lanczos(y)
            eng.dot_into(self.b, y, sc[S_BY:S_BY + 1])
            lam_y = float(eig.eigenvalues[0])
            f_y = self.alpha * max(lam_y, 0.0) + float(sc[S_BY].item())
        else:
            f_y, lam_y = state.f_y, state.lam_y
        primal = state.last_primal if state.last_primal is not None else model.stats
        residuals = self.residuals(y, f_y, lam_y, primal)
        state.f_y, state.lam_y, state.residuals = f_y, lam_y, residuals
        status = "converged" if residuals.converged(cfg.eps, cfg.linf_check) else None
        t = 0
        inner_nu = rt.empty(self.m)
        inner_nu.copy_(state.nu_dev)
        y_buf = rt.empty(self.m)
        a = self.alpha
        while status is None:
            if t >= cfg.max_iters or (cfg.max_time is not None and time.monotonic() - t_start > cfg.max_time):
                status = "budget"
                break
            nu, passes, has_eta = self.alternating_max(model, y, inner_nu)
            inner_nu, nu_keep = nu, nu
            k = model.k
            eng.vec(N.VOP_CAND, self.m, x=self.ax, y=y, z=nu, b=self.b, ineq=self.ineq, s0=float(cfg.rho),
                    out=self.ycand)
            if self.has_ineq:
                eng.vec(N.VOP_MINI, self.m, x=self.ycand, ineq=self.ineq, red=sc[S_MINI:S_MINI + 2])
            tr = model.stats.trace
            if self.overlap:
                # the model evaluation at y_cand (assemble_eval_coeffs + ipm_eval,
                # subqp.py:455-468) depends only on the assembled Z, so it runs on a
                # second stream concurrently with the Lanczos kernel (which leaves
                # a few SMs free for it)
                torch = self.rt.torch
                self.dp.assemble(self.ycand)
                aux_stream, _ = self.rt.aux()
                ev0 = torch.cuda.Event()
                ev0.record(self.rt.stream)
                aux_stream.wait_event(ev0)
                self._eval_at_candidate(self.eng_aux, model, k, tr)
                ev1 = torch.cuda.Event()
                ev1.record(aux_stream)
                eig = self.penalized_lanczos(self.ycand, assembled=True)
                self.rt.stream.wait_event(ev1)
            else:
                eig = self.penalized_lanczos(self.ycand)
                self._eval_at_candidate(eng, model, k, tr)
            lam_c = float(eig.eigenvalues[0])
            # s_act = alpha S (original units) for model_update
            S = self.st_q[:k * k].view(k, k)
            eng.vec(N.VOP_AXPBY, k * k, x=S.reshape(-1), s0=a, out=self.s_act.view(-1))
            self._scratch[80:80 + k].copy_(S.diagonal())
            buf = self._fetch_scratch(80 + k)
            sc_h, rq, re_, sdiag = buf[:18], buf[64:72], buf[72:80], buf[80:80 + k]
            if self.has_ineq and sc_h[S_MINI + 1] > 0.0:
                raise ValueError("candidate dual point violates the sign constraints")
            eta_act = (a * float(rq[3]) / tr) if has_eta else 0.0
            c_x = eta_act * model.stats.cost_ip + float(sc_h[S_CQS])
            tr_x = eta_act * tr + float(np.sum(a * sdiag))
            b_yc = float(sc_h[S_BYC])
            f_cand = a * max(lam_c, 0.0) + b_yc
            model_val = b_yc - float(re_[0])
            accept = cfg.beta * (f_y - model_val) <= f_y - f_cand
            if accept:
                y_buf.copy_(self.ycand)
                y, y_buf = y_buf, y
                f_y, lam_y = f_cand, lam_c
                state.nu_dev = nu_keep.clone()
                state.descent_steps += 1
            else:
                state.null_steps += 1
            step = "descent" if accept else "null"
            model, pending = self.model_update(model, eta_act, eig.eigenvectors_dev, tag=t + 1)
            # records handed to a callback own their m-vectors (the solver's
            # scratch and the y ping-pong buffers are reused by later iterations)
            own = (lambda v: v.clone()) if callback is not None else (lambda v: v)
            primal = AggregateStats(tr_x, c_x, own(self.ax))
            residuals = self.residuals(y, f_y, lam_y, primal, pending=pending, model=model)
            state.y_dev, state.f_y, state.lam_y, state.model = y, f_y, lam_y, model
            state.last_primal, state.residuals, state.iterations = primal, residuals, t + 1
            state.best_rel_infeas = min(state.best_rel_infeas, residuals.rel_infeas)
            state.best_rel_subopt = min(state.best_rel_subopt, residuals.rel_subopt)
            if callback is not None:
                callback(IterationInfo(t, time.monotonic() - t_start, step, f_y, f_cand, model_val, own(y),
                                       own(self.ycand), own(nu_keep), residuals, primal, eta_act, lam_c, state,
                                       model, passes,
                                       eig.matvecs, eig.restarts))
            t += 1
            if residuals.converged(cfg.eps, cfg.linf_check):
                status = "converged"
        state.status = status
        state.last_primal = AggregateStats(state.last_primal.trace, state.last_primal.cost_ip,
                                           state.last_primal.constr_image_dev.clone())
        return state, self.primal_output(model)

    def _eval_at_candidate(self, eng, model, k, tr):
        """ipm_eval(assemble_eval_coeffs(prob, model, y_cand)) (subqp.py:455-468)
        and <b, y_cand>, launched through `eng` (main or auxiliary stream)."""
        sc, a = self.sc, self.alpha
        eng.apply(1, model.basis_dev, self.tmp_nk2[:, :k], gram=self.zq)
        eng.svec(self.zq, self.lin_s, scale=-a)
        eng.dot_into(self.ycand[:1], self.ycand[:1], sc[S_EQ22:S_EQ22 + 1], scale=0.0)
        if tr > 0.0:
            eng.dot_into(self.ycand, model.stats.constr_image_dev, sc[S_ELINETA:S_ELINETA + 1],
                         scale=a / tr, shift=-(a / tr) * model.stats.cost_ip)
        else:
            eng.dot_into(self.ycand[:1], self.ycand[:1], sc[S_ELINETA:S_ELINETA + 1], scale=0.0)
        eng.ipm(k, tr > 0.0, None, None, self.lin_s, sc[S_EQ22:S_EQ22 + 2], None, self.st_e, self.res_e,
                self.opts)
        eng.dot_into(self.b, self.ycand, sc[S_BYC:S_BYC + 1])

    def residuals(self, y, f_y, lam_y, primal, pending=None, model=None) -> Residuals:
        """compute_residuals (bundle.py:344-372); also finalises the pending
        trace / cost statistics of a model update in the same sync."""
        eng, sc = self.eng, self.sc
        eng.vec(N.VOP_RESID, self.m, x=primal.constr_image_dev, b=self.b, ineq=self.ineq,
                red=sc[S_RES:S_RES + 2])
        eng.dot_into(self.b, y, sc[S_BY:S_BY + 1])
        if pending is not None:
            if self.lamc.data_ptr() == self._scratch[144:].data_ptr():
                buf = self._fetch_scratch(144 + model.k_c)
                sc_h, lamc = buf[:18], buf[144:144 + model.k_c]
            else:
                sc_h, lamc = self._fetch(sc[:18], self.lamc[:model.k_c])
            eta, tr_old, cip_old = pending
            model.stats.trace = eta * tr_old + float(lamc.sum())
            model.stats.cost_ip = eta * cip_old + float(sc_h[S_CFIP])
        else:
            sc_h = self._fetch_scratch(18)
        c_x = primal.cost_ip
        rel_infeas = math.sqrt(max(float(sc_h[S_RES]), 0.0)) / (1.0 + self.b_norm)
        linf = float(sc_h[S_RES + 1]) if self.m else 0.0
        return Residuals((c_x - f_y) / (1.0 + abs(c_x)), rel_infeas, linf, abs(float(sc_h[S_BY]) - c_x), lam_y)

    def primal_output(self, model: BundleModel) -> PrimalOutput:
        """bundle.primal_output (bundle.py:532-538)."""
        if model.store is None:
            return PrimalOutput(np.eye(self.n, 1), np.zeros(1))
        factor, lams = model.store.factorize()
        dense = model.store.xbar if isinstance(model.store, DeviceExplicitStore) else None
        return PrimalOutput(factor, lams, dense)


def solve(prob, cfg, init: Optional[SolverState] = None, callback: Optional[Callable] = None):
    """Drop-in for specbundle.solve (bundle.py:426-529): same arguments and
    return value (SolverState, PrimalOutput); arrays of the state live on the
    GPU and convert to numpy on attribute access.  ``init`` may be a device
    state (cold start, ``state.warm_start_pad`` / ``state_from_record``) or a
    host one with the reference's attribute names; as in the reference, the
    state's own k_c / k_p drive the iteration."""
    dprob = None
    if init is not None:
        if not hasattr(init, "y_dev"):
            from .state import state_from_host
            init = state_from_host(init)
        dp = getattr(init, "device_problem", None)
        if dp is not None and dp.prob is prob:
            dprob = dp
        kc, kp = int(init.model.k_c), int(init.model.k_p)
        if (kc, kp) != (min(cfg.k_c, int(prob.n)), min(cfg.k_p, int(prob.n) - min(cfg.k_c, int(prob.n)))):
            cfg = dataclasses.replace(cfg, k_c=kc, k_p=kp)
    return DeviceSolver(prob, cfg, dprob=dprob).solve(init=init, callback=callback)
