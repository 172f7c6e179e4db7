"""CPU oracle for the warm-start state container and padding -- TEST
INFRASTRUCTURE ONLY (imported by tests/ alone; the product never imports it).

Restates, in plain numpy, the reference's versioned ``USBS`` v1 state file
(specbundle bundle.py:541-700) and ``warm_start_pad`` (bundle.py:754-817).
Pinned against container bytes and padded states that oracle/make_golden.py
records by running the reference itself (tests/golden/state.npz; checked by
tests/test_state.py).
"""
from __future__ import annotations

import hashlib
import struct

import numpy as np

from .usbs_cpu import Dense, Model, Sketched, State, Stats, cost_ip, image_factor, sketch_apply, sketch_new

HEAD = "<4sI QQQQ II B II dd dd QQ dd"  # bundle.py:593-594 / 628


def fingerprint(n, m, n_ineq, b) -> tuple:
    """fingerprint_of (bundle.py:546-548)."""
    h = hashlib.sha256(np.ascontiguousarray(b, dtype="<f8").tobytes()).digest()
    return (int(n), int(m), int(n_ineq), int.from_bytes(h[:8], "little"))


def unpack(raw: bytes) -> dict:
    """load_state (bundle.py:625-700) into a plain dict."""
    size = struct.calcsize(HEAD)
    if len(raw) < size:
        raise ValueError("truncated state file")
    keys = ("magic", "version", "n", "m", "n_ineq", "b_hash", "k_c", "k_p", "kind", "rank", "psi_seed", "scale_x",
            "scale_c", "f_y", "lam_y", "descent", "null", "trace", "cost_ip")
    d = dict(zip(keys, struct.unpack(HEAD, raw[:size])))
    if d["magic"] != b"USBS":
        raise ValueError("not a solver state file")
    if d["version"] != 1:
        raise ValueError("unsupported state file version")
    pos = size

    def take(count):
        nonlocal pos
        a = np.frombuffer(raw, dtype="<f8", count=count, offset=pos).astype(float)
        pos += 8 * count
        return a

    n, m, k = d["n"], d["m"], d["k_c"] + d["k_p"]
    d["y"], d["nu"], d["a_xbar"] = take(m), take(m), take(m)
    d["basis"] = take(n * k).reshape(n, k)
    d["xbar"] = take(n * n).reshape(n, n) if d["kind"] == 1 else None
    d["sketch"] = take(n * d["rank"]).reshape(n, d["rank"]) if d["kind"] == 2 else None
    return d


def pack(d: dict) -> bytes:
    """save_state (bundle.py:578-622) from a dict as returned by unpack."""
    head = struct.pack(HEAD, b"USBS", 1, d["n"], d["m"], d["n_ineq"], d["b_hash"], d["k_c"], d["k_p"], d["kind"],
                       d["rank"], d["psi_seed"] & 0xFFFFFFFF, d["scale_x"], d["scale_c"], d["f_y"], d["lam_y"],
                       d["descent"], d["null"], d["trace"], d["cost_ip"])
    body = [np.ascontiguousarray(d[x], dtype="<f8").tobytes() for x in ("y", "nu", "a_xbar", "basis")]
    if d["kind"] == 1:
        body.append(np.ascontiguousarray(d["xbar"], dtype="<f8").tobytes())
    elif d["kind"] == 2:
        body.append(np.ascontiguousarray(d["sketch"], dtype="<f8").tobytes())
    return head + b"".join(body)


def to_state(d: dict) -> State:
    """record_to_state (bundle.py:703-729) into the oracle's State."""
    from .usbs_cpu import Sketch, psi_matrix
    if d["kind"] == 1:
        store = Dense(d["xbar"].copy())
    elif d["kind"] == 2:
        store = Sketched(Sketch(d["n"], d["rank"], d["psi_seed"], d["sketch"].copy(),
                                 psi_matrix(d["n"], d["rank"], d["psi_seed"])))
    else:
        store = None
    st = Stats(d["trace"], d["cost_ip"], d["a_xbar"].copy())
    f_y = None if np.isnan(d["f_y"]) else d["f_y"]
    lam_y = None if np.isnan(d["lam_y"]) else d["lam_y"]
    return State(d["y"].copy(), d["nu"].copy(), f_y, lam_y, Model(d["basis"].copy(), st, d["k_c"], d["k_p"], store),
                 descent_steps=d["descent"], null_steps=d["null"], last_primal=st.copy())


def pad(prev: State, prev_scale_x, new_prob, vmap, cmap, sketch_seed=None) -> State:
    """warm_start_pad (bundle.py:754-817): zero duals on new constraints,
    zero factor rows on new vertices, eigenvalues times
    prev_scale_x / new_scale_x, statistics recomputed on the new problem,
    store rebuilt from the padded factor."""
    vmap = np.asarray(vmap, dtype=np.int64)
    cmap = np.asarray(cmap, dtype=np.int64)
    if vmap.size and (vmap.min() < 0 or vmap.max() >= new_prob.n):
        raise ValueError("vertex mapping out of range")
    if cmap.size and (cmap.min() < 0 or cmap.max() >= new_prob.m):
        raise ValueError("constraint mapping out of range")
    model = prev.model
    if vmap.size != model.basis.shape[0] or cmap.size != prev.y.shape[0]:
        raise ValueError("mapping does not match the previous state dimensions")
    tau = prev_scale_x / new_prob.scale_x
    if model.store is not None:
        f_old, l_old = model.store.factorize()
    else:
        f_old, l_old = np.zeros((vmap.size, 1)), np.zeros(1)
    f = np.zeros((new_prob.n, f_old.shape[1]))
    f[vmap] = f_old
    lams = tau * l_old
    y = np.zeros(new_prob.m)
    y[cmap] = prev.y
    nu = np.zeros(new_prob.m)
    nu[cmap] = prev.nu
    basis = np.zeros((new_prob.n, model.basis.shape[1]))
    basis[vmap] = model.basis
    st = Stats(float(lams.sum()), cost_ip(new_prob, f, lams), image_factor(new_prob.constraints, f, lams))
    if isinstance(model.store, Dense):
        store = Dense((f * lams[None, :]) @ f.T)
    elif isinstance(model.store, Sketched):
        seed = sketch_seed if sketch_seed is not None else model.store.sk.seed
        sk = sketch_new(new_prob.n, min(model.store.sk.r, new_prob.n), seed)
        store = Sketched(sketch_apply(sk, 0.0, f, lams))
    else:
        store = None
    return State(y, nu, None, None, Model(basis, st, model.k_c, model.k_p, store), last_primal=st.copy())
