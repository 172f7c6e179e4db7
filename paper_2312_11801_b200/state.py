"""Warm-start state files and padding.

* ``save_state`` / ``load_state`` read and write the reference's versioned
  little-endian ``USBS`` v1 container (bundle.py:541-700) byte for byte:
  header ``<4sI QQQQ II B II dd dd QQ dd`` (magic, version, the problem
  fingerprint n, m, #inequalities, b-hash; k_c, k_p; store kind; sketch rank,
  psi seed; scale_x, scale_c; f(y), lambda(y) with NaN for "unknown";
  descent / null step counts; trace, <C, Xbar>), then y, nu, A(Xbar) and
  the n x k basis as float64, then Xbar (n x n, explicit store) or the
  n x r sketch.  A file written here loads in the reference and vice versa.
* ``state_from_record`` / ``record_to_state`` rebuild a device-resident
  ``SolverState`` (bundle.py:703-742), with the same fingerprint check.
* ``warm_start_pad`` (bundle.py:745-817) embeds a solved state into a larger
  problem on the device: the dual vectors, basis and primal factor are
  gathered through the inverse vertex / constraint maps
  (``usbs_gather_rows``), the statistics recomputed against the new problem
  data (K1 cost apply + weighted column dots, K5 image) and the store
  rebuilt (dense update / sketch update with eta = 0).
* ``state_from_host`` turns a host state with the reference's attribute
  names (e.g. a reference ``SolverState``) into a device one, so
  ``solve(prob, cfg, init=...)`` accepts either.
"""
from __future__ import annotations

import hashlib
import struct
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .errors import FingerprintMismatch

__all__ = ["StateRecord", "Mapping", "fingerprint_of", "save_state", "load_state", "state_from_record",
           "record_to_state", "warm_start_pad", "state_from_host", "FingerprintMismatch"]

_MAGIC = b"USBS"
_VERSION = 1
_HEAD = "<4sI QQQQ II B II dd dd QQ dd"
_HEAD_SIZE = struct.calcsize(_HEAD)


def _ineq_count(prob) -> int:
    idx = getattr(prob, "ineq_idx", None)
    if idx is not None:
        return int(np.asarray(idx).size)
    return int(np.count_nonzero(np.asarray(prob.ineq_mask, dtype=bool)))


def fingerprint_of(prob) -> tuple:
    """(n, m, #inequalities, first 8 bytes of sha256(b as <f8), little
    endian) -- bundle.py:546-548."""
    digest = hashlib.sha256(np.ascontiguousarray(prob.b, dtype="<f8").tobytes()).digest()
    return (int(prob.n), int(prob.m), _ineq_count(prob), int.from_bytes(digest[:8], "little"))


@dataclass
class StateRecord:
    """The decoded container (bundle.py:551-575); host arrays."""

    n: int
    m: int
    n_ineq: int
    b_hash: int
    k_c: int
    k_p: int
    store_kind: int  # 0 none, 1 explicit, 2 sketch
    sketch_rank: int
    psi_seed: int
    scale_x: float
    scale_c: float
    f_y: Optional[float]
    lam_y: Optional[float]
    descent_steps: int
    null_steps: int
    y: np.ndarray
    nu: np.ndarray
    a_xbar: np.ndarray
    trace: float
    cost_ip: float
    basis: np.ndarray
    xbar: Optional[np.ndarray]
    sketch_mat: Optional[np.ndarray]


@dataclass
class Mapping:
    """Embedding of a smaller instance into a larger one (bundle.py:745-751):
    position p of each array holds the index in the larger problem."""

    vertex_map: np.ndarray
    constraint_map: np.ndarray


# ---------------------------------------------------------------------------
# host views of device / reference states

def _store_kind(store):
    """(kind, rank, psi_seed, payload getter) of a device or reference store."""
    from .solver import DeviceExplicitStore, DeviceSketchStore
    if store is None:
        return 0, 0, 0, None
    if isinstance(store, DeviceExplicitStore):
        return 1, 0, 0, lambda: store.xbar
    if isinstance(store, DeviceSketchStore):
        return 2, store.r, store.psi_seed, lambda: store.sketch_mat
    sk = getattr(store, "sk", None)
    if sk is not None:  # reference SketchStore
        return 2, int(sk.r), int(sk.psi_seed), lambda: np.asarray(sk.sketch_mat)
    if hasattr(store, "xbar"):  # reference ExplicitStore
        return 1, 0, 0, lambda: np.asarray(store.xbar)
    raise TypeError(f"unknown primal store {type(store).__name__}")


def _f8(a) -> bytes:
    return np.ascontiguousarray(a, dtype="<f8").tobytes()


def save_state(path, state, prob) -> None:
    """save_state (bundle.py:578-622): the USBS v1 container of a device (or
    reference) SolverState.  The arrays come off the device in one pass."""
    n, m, n_ineq, b_hash = fingerprint_of(prob)
    model = state.model
    kind, rank, seed, payload = _store_kind(model.store)
    if kind == 2 and getattr(model.store, "shard", None) is not None and model.store.P.shape[0] != model.store.n:
        raise ValueError("save_state needs the full sketch; gather a row-sharded state first")
    f_y = state.f_y if state.f_y is not None else np.nan
    lam_y = state.lam_y if state.lam_y is not None else np.nan
    header = struct.pack(_HEAD, _MAGIC, _VERSION, n, m, n_ineq, b_hash, int(model.k_c), int(model.k_p), kind,
                         int(rank), int(seed) & 0xFFFFFFFF, float(state.scale_x), float(state.scale_c), float(f_y),
                         float(lam_y), int(state.descent_steps), int(state.null_steps), float(model.stats.trace),
                         float(model.stats.cost_ip))
    with open(path, "wb") as fh:
        fh.write(header)
        for arr in (state.y, state.nu, model.stats.constr_image, model.basis):
            fh.write(_f8(arr))
        if payload is not None:
            fh.write(_f8(payload()))


def load_state(path) -> StateRecord:
    """load_state (bundle.py:625-700): ValueError on a truncated file, a
    foreign magic or another version."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < _HEAD_SIZE:
        raise ValueError("truncated state file")
    (magic, version, n, m, n_ineq, b_hash, k_c, k_p, kind, rank, psi_seed, scale_x, scale_c, f_y, lam_y, descent,
     null, trace, cost_ip) = struct.unpack(_HEAD, raw[:_HEAD_SIZE])
    if magic != _MAGIC:
        raise ValueError("not a solver state file")
    if version != _VERSION:
        raise ValueError(f"unsupported state file version {version}")
    off = [_HEAD_SIZE]

    def take(count):
        out = np.frombuffer(raw, dtype="<f8", count=count, offset=off[0]).astype(float)
        off[0] += count * 8
        return out

    k = k_c + k_p
    y, nu, a_xbar = take(m), take(m), take(m)
    basis = take(n * k).reshape(n, k)
    xbar = take(n * n).reshape(n, n) if kind == 1 else None
    sketch_mat = take(n * rank).reshape(n, rank) if kind == 2 else None
    return StateRecord(n, m, n_ineq, b_hash, k_c, k_p, kind, rank, psi_seed, scale_x, scale_c,
                       None if np.isnan(f_y) else float(f_y), None if np.isnan(lam_y) else float(lam_y),
                       descent, null, y, nu, a_xbar, trace, cost_ip, basis, xbar, sketch_mat)


# ---------------------------------------------------------------------------
# device states

def _engine(n, dp=None):
    if dp is not None:
        from .engine import Engine
        return Engine(dp), dp.rt
    from .linalg import _engine as problem_free
    return problem_free(n)


def _device_state(eng, rt, *, y, nu, f_y, lam_y, basis, k_c, k_p, trace, cost_ip, image, kind, xbar=None,
                  sketch=None, psi_seed=0, descent=0, null=0, last_primal=None, scale_x=1.0, scale_c=1.0):
    from .solver import AggregateStats, BundleModel, DeviceExplicitStore, DeviceSketchStore, SolverState
    dev = lambda a: a if hasattr(a, "data_ptr") else rt.upload(np.ascontiguousarray(a, dtype=float))  # noqa: E731
    n = basis.shape[0]
    if kind == 1:
        store = DeviceExplicitStore(eng, n)
        store.X.copy_(dev(xbar))
    elif kind == 2:
        store = DeviceSketchStore(eng, n, sketch.shape[1], psi_seed)
        store.P.copy_(dev(sketch))
    else:
        store = None
    stats = AggregateStats(float(trace), float(cost_ip), dev(image).clone())
    model = BundleModel(dev(basis).clone(), stats, int(k_c), int(k_p), store)
    if last_primal is None:
        lp = AggregateStats(stats.trace, stats.cost_ip, stats.constr_image_dev.clone())
    else:
        lp = AggregateStats(float(last_primal[0]), float(last_primal[1]), dev(last_primal[2]).clone())
    return SolverState(dev(y).clone(), dev(nu).clone(), f_y, lam_y, model, descent_steps=int(descent),
                       null_steps=int(null), last_primal=lp, scale_x=float(scale_x), scale_c=float(scale_c))


def record_to_state(rec: StateRecord, dprob=None):
    """record_to_state (bundle.py:703-729): no fingerprint check (for
    cross-problem padding)."""
    eng, rt = _engine(rec.n, dprob)
    st = _device_state(eng, rt, y=rec.y, nu=rec.nu, f_y=rec.f_y, lam_y=rec.lam_y, basis=rec.basis, k_c=rec.k_c,
                       k_p=rec.k_p, trace=rec.trace, cost_ip=rec.cost_ip, image=rec.a_xbar, kind=rec.store_kind,
                       xbar=rec.xbar, sketch=rec.sketch_mat, psi_seed=rec.psi_seed, descent=rec.descent_steps,
                       null=rec.null_steps, scale_x=rec.scale_x, scale_c=rec.scale_c)
    st.device_problem = dprob
    return st


def state_from_record(rec: StateRecord, prob, dprob=None):
    """state_from_record (bundle.py:732-739): FingerprintMismatch unless the
    record was saved from this problem; scales taken from the problem."""
    if (rec.n, rec.m, rec.n_ineq, rec.b_hash) != fingerprint_of(prob):
        raise FingerprintMismatch("state fingerprint does not match this problem")
    st = record_to_state(rec, dprob)
    st.scale_x, st.scale_c = float(prob.scale_x), float(prob.scale_c)
    return st


def state_from_host(st, dprob=None):
    """A device SolverState from a host one with the reference's attribute
    names (bundle.SolverState: y, nu, f_y, lam_y, model.{basis, stats, k_c,
    k_p, store}, last_primal, step counts, scales)."""
    model = st.model
    kind, rank, seed, payload = _store_kind(model.store)
    data = payload() if payload is not None else None
    n = np.asarray(model.basis).shape[0]
    eng, rt = _engine(n, dprob)
    lp = st.last_primal
    out = _device_state(eng, rt, y=st.y, nu=st.nu, f_y=st.f_y, lam_y=st.lam_y, basis=model.basis, k_c=model.k_c,
                        k_p=model.k_p, trace=model.stats.trace, cost_ip=model.stats.cost_ip,
                        image=model.stats.constr_image, kind=kind, xbar=data if kind == 1 else None,
                        sketch=data if kind == 2 else None, psi_seed=seed, descent=st.descent_steps,
                        null=st.null_steps,
                        last_primal=None if lp is None else (lp.trace, lp.cost_ip, lp.constr_image),
                        scale_x=getattr(st, "scale_x", 1.0), scale_c=getattr(st, "scale_c", 1.0))
    out.device_problem = dprob
    return out


def _inverse_map(fwd: np.ndarray, size: int) -> np.ndarray:
    inv = np.full(size, -1, dtype=np.int64)
    inv[fwd] = np.arange(fwd.size, dtype=np.int64)  # repeated targets: the last one wins, as in the reference
    return inv


def warm_start_pad(prev, new_prob, mapping: Mapping, sketch_seed: Optional[int] = None, dprob=None):
    """warm_start_pad (bundle.py:754-817) on the device.

    Duals padded with zeros on new constraints; the primal factor padded
    with zero rows on new vertices, its eigenvalues rescaled by
    prev.scale_x / new.scale_x; trace, <C, X> and A(X) recomputed on the new
    problem; the store rebuilt from the padded factor.  ``prev`` may be a
    device state or a host state with the reference's attribute names.  The
    returned state keeps its DeviceProblem, which ``solve(new_prob, ...,
    init=state)`` reuses."""
    from .runtime import DeviceProblem
    from .solver import AggregateStats, BundleModel, DeviceExplicitStore, DeviceSketchStore, SolverState
    vmap = np.asarray(mapping.vertex_map, dtype=np.int64)
    cmap = np.asarray(mapping.constraint_map, dtype=np.int64)
    if vmap.size and (vmap.min() < 0 or vmap.max() >= new_prob.n):
        raise ValueError("vertex mapping out of range")
    if cmap.size and (cmap.min() < 0 or cmap.max() >= new_prob.m):
        raise ValueError("constraint mapping out of range")
    model = prev.model
    basis_prev = model.basis_dev if hasattr(model, "basis_dev") else np.asarray(model.basis, dtype=float)
    y_prev = prev.y_dev if hasattr(prev, "y_dev") else np.asarray(prev.y, dtype=float)
    nu_prev = prev.nu_dev if hasattr(prev, "nu_dev") else np.asarray(prev.nu, dtype=float)
    if vmap.size != basis_prev.shape[0] or cmap.size != y_prev.shape[0]:
        raise ValueError("mapping does not match the previous state dimensions")

    dp = dprob if dprob is not None else DeviceProblem(new_prob)
    from .engine import Engine
    eng = Engine(dp)
    rt = dp.rt
    dev = lambda a: a if hasattr(a, "data_ptr") else rt.upload(np.ascontiguousarray(a, dtype=float))  # noqa: E731
    n, m = int(new_prob.n), int(new_prob.m)
    tau = float(prev.scale_x) / float(new_prob.scale_x)
    kind, rank, seed, _ = _store_kind(model.store)
    if isinstance(model.store, DeviceSketchStore) and model.store.P.shape[0] != model.store.n:
        raise ValueError("warm_start_pad needs an unsharded state")
    if model.store is not None:
        factor_old, lams_old = model.store.factorize()
    else:
        factor_old, lams_old = np.zeros((vmap.size, 1)), np.zeros(1)
    factor_old = np.atleast_2d(np.asarray(factor_old, dtype=float))
    lams = tau * np.asarray(lams_old, dtype=float)

    inv_v = rt.torch.as_tensor(_inverse_map(vmap, n), device=rt.device)
    inv_c = rt.torch.as_tensor(_inverse_map(cmap, m), device=rt.device)
    r = factor_old.shape[1]
    k = basis_prev.shape[1]
    F = eng.gather_rows(inv_v, dev(factor_old), rt.empty(n, r))
    y = eng.gather_rows(inv_c, dev(y_prev).view(-1, 1), rt.empty(m, 1)).view(-1)
    nu = eng.gather_rows(inv_c, dev(nu_prev).view(-1, 1), rt.empty(m, 1)).view(-1)
    basis = eng.gather_rows(inv_v, dev(basis_prev), rt.empty(n, k))

    lam_d = rt.upload(lams)
    trace = float(lams.sum())
    # statistics and store from the padded factor, in column blocks of <= 64
    # (the kernels' width limit; an explicit store's factor can be n wide)
    CF = eng.apply(0, F, rt.empty(n, r)) if r <= 64 else None
    cip = rt.zeros(max(1, (r + 63) // 64))
    image = rt.empty(m)
    if kind == 1:
        store = DeviceExplicitStore(eng, n)
    elif kind == 2:
        sd = int(sketch_seed) if sketch_seed is not None else int(seed)
        store = DeviceSketchStore(eng, n, min(int(rank), n), sd)
    else:
        store = None
    for c, j0 in enumerate(range(0, r, 64)):
        j1 = min(r, j0 + 64)
        Fj, lj = F[:, j0:j1], lam_d[j0:j1]
        CFj = CF[:, j0:j1] if CF is not None else eng.apply(0, Fj.contiguous(), rt.empty(n, j1 - j0))
        eng.wcoldot(Fj, CFj, lj, cip[c:c + 1])
        eng.image(Fj, lj, image, s_is_diag=True, beta=0.0 if j0 == 0 else 1.0, base=None if j0 == 0 else image)
        if store is not None:
            store.update(0.0 if j0 == 0 else 1.0, Fj, lj)
    cost_ip = float(cip.sum().item()) if r > 64 else float(cip[0].item())
    stats = AggregateStats(trace, cost_ip, image)
    new_model = BundleModel(basis, stats, int(model.k_c), int(model.k_p), store)
    st = SolverState(y, nu, None, None, new_model,
                     last_primal=AggregateStats(trace, cost_ip, image.clone()),
                     scale_x=float(new_prob.scale_x), scale_c=float(new_prob.scale_c))
    st.device_problem = dp
    return st
