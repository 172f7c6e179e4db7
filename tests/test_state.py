"""Warm-start state files and padding.

Fixtures (tests/golden/state.npz, oracle/make_golden.py state_cases) hold the
reference's own save_state bytes of solved states, the bytes of its
warm_start_pad output into a graph with one more vertex (the construction of
the reference's test_bundle.py:373-394) and the trajectory of the solve
warm-started from it.

CPU: the oracle container and padding against those fixtures, the product's
load_state / fingerprint.  GPU: device states round-trip to identical bytes,
the device warm_start_pad against the reference's padded state, and the
warm-started solve against the reference trajectory.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import cuda_ok
from helpers import k3, load_npz
from oracle import state_cpu as OS
from paper_2312_11801_b200 import instances as inst
from paper_2312_11801_b200 import state as S

G = load_npz("state.npz")
BINS = ("k3_sketch/bin", "dense/bin", "sketch/bin", "dense/pad_bin", "sketch/pad_bin")


def _graph(which):
    return inst.Graph.from_arrays(10 if which == "big" else 9, G[f"{which}/eu"], G[f"{which}/ev"], G[f"{which}/ew"])


def _prob(which):
    if which == "k3":
        return inst.maxcut_problem(k3())
    return inst.maxcut_problem(_graph(which))


def _raw(key):
    return G[key].tobytes()


def _write(tmp_path, key):
    p = tmp_path / (key.replace("/", "_") + ".bin")
    p.write_bytes(_raw(key))
    return p


# ---------------------------------------------------------------- CPU: oracle
@pytest.mark.parametrize("key", BINS)
def test_oracle_container_round_trip(key):
    raw = _raw(key)
    assert OS.pack(OS.unpack(raw)) == raw


@pytest.mark.parametrize("key", BINS)
def test_load_state_matches_oracle(tmp_path, key):
    rec = S.load_state(_write(tmp_path, key))
    d = OS.unpack(_raw(key))
    assert (rec.n, rec.m, rec.n_ineq, rec.b_hash, rec.k_c, rec.k_p, rec.store_kind, rec.sketch_rank, rec.psi_seed) == \
        (d["n"], d["m"], d["n_ineq"], d["b_hash"], d["k_c"], d["k_p"], d["kind"], d["rank"], d["psi_seed"])
    for a, b in ((rec.y, d["y"]), (rec.nu, d["nu"]), (rec.a_xbar, d["a_xbar"]), (rec.basis, d["basis"])):
        np.testing.assert_array_equal(a, b)
    assert rec.trace == d["trace"] and rec.cost_ip == d["cost_ip"]
    if key.endswith("pad_bin"):
        assert rec.f_y is None and rec.lam_y is None  # padding leaves f, lambda unknown (NaN in the file)


@pytest.mark.parametrize("key,which", [("k3_sketch/bin", "k3"), ("dense/bin", "small"), ("sketch/bin", "small"),
                                       ("dense/pad_bin", "big"), ("sketch/pad_bin", "big")])
def test_fingerprint_of_rebuilt_problem(key, which):
    d = OS.unpack(_raw(key))
    p = _prob(which)
    assert S.fingerprint_of(p) == (d["n"], d["m"], d["n_ineq"], d["b_hash"])
    assert OS.fingerprint(p.n, p.m, 0, p.b) == S.fingerprint_of(p)


def test_bad_files(tmp_path):
    p = tmp_path / "junk.bin"
    p.write_bytes(b"NOPE" + b"\0" * 200)
    with pytest.raises(ValueError):
        S.load_state(p)
    p.write_bytes(b"USBS")
    with pytest.raises(ValueError):
        S.load_state(p)
    raw = bytearray(_raw("dense/bin"))
    raw[4] = 2  # version 2
    p.write_bytes(bytes(raw))
    with pytest.raises(ValueError):
        S.load_state(p)
    p.write_bytes(_raw("dense/bin")[:-8])  # one double short
    with pytest.raises(ValueError):
        S.load_state(p)


def _close(a, b, rtol):
    a, b = np.asarray(a, float), np.asarray(b, float)
    np.testing.assert_allclose(a, b, rtol=rtol, atol=rtol * max(1.0, float(np.abs(b).max(initial=0.0))))


@pytest.mark.parametrize("name", ["dense", "sketch"])
def test_oracle_pad_matches_reference(name):
    prev = OS.unpack(_raw(f"{name}/bin"))
    want = OS.unpack(_raw(f"{name}/pad_bin"))
    p_big = _prob("big")
    got = OS.pad(OS.to_state(prev), prev["scale_x"], p_big, np.arange(9), np.arange(9),
                 sketch_seed=5 if name == "sketch" else None)
    np.testing.assert_array_equal(got.y, want["y"])
    np.testing.assert_array_equal(got.nu, want["nu"])
    np.testing.assert_array_equal(got.model.basis, want["basis"])
    assert got.y[9] == 0.0 and np.all(got.model.basis[9] == 0.0)
    _close(got.model.stats.trace, want["trace"], 1e-13)
    _close(got.model.stats.cost_ip, want["cost_ip"], 1e-12)
    _close(got.model.stats.constr_image, want["a_xbar"], 1e-12)
    if name == "dense":
        _close(got.model.store.xbar, want["xbar"], 1e-12)
    else:
        _close(got.model.store.sk.p, want["sketch"], 1e-12)
    if name == "dense":  # the reference's rescale rule (exact store): trace x old / new normalisation
        assert got.model.stats.trace == pytest.approx(prev["trace"] * 9 / 10, rel=1e-9)


def test_oracle_pad_rejects_bad_mappings():
    prev = OS.to_state(OS.unpack(_raw("dense/bin")))
    p_big = _prob("big")
    with pytest.raises(ValueError):
        OS.pad(prev, 9.0, p_big, np.array([0, 1, 10, 3, 4, 5, 6, 7, 8]), np.arange(9))
    with pytest.raises(ValueError):
        OS.pad(prev, 9.0, p_big, np.arange(8), np.arange(9))


# ---------------------------------------------------------------- GPU
@pytest.mark.parametrize("key,which", [("k3_sketch/bin", "k3"), ("dense/bin", "small"), ("sketch/bin", "small"),
                                       ("dense/pad_bin", "big"), ("sketch/pad_bin", "big")])
@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")
def test_device_state_round_trips_reference_bytes(tmp_path, key, which):
    prob = _prob(which)
    st = S.state_from_record(S.load_state(_write(tmp_path, key)), prob)
    out = tmp_path / "again.bin"
    S.save_state(out, st, prob)
    assert out.read_bytes() == _raw(key)


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")
def test_fingerprint_mismatch(tmp_path):
    rec = S.load_state(_write(tmp_path, "dense/bin"))
    with pytest.raises(S.FingerprintMismatch):
        S.state_from_record(rec, _prob("big"))


@pytest.mark.parametrize("name", ["dense", "sketch"])
@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")
def test_device_pad_matches_reference(tmp_path, name):
    prev = S.record_to_state(S.load_state(_write(tmp_path, f"{name}/bin")))
    want = OS.unpack(_raw(f"{name}/pad_bin"))
    p_big = _prob("big")
    got = S.warm_start_pad(prev, p_big, S.Mapping(np.arange(9), np.arange(9)),
                           sketch_seed=5 if name == "sketch" else None)
    np.testing.assert_array_equal(got.y, want["y"])
    np.testing.assert_array_equal(got.nu, want["nu"])
    np.testing.assert_array_equal(got.model.basis, want["basis"])
    assert got.f_y is None and got.lam_y is None
    _close(got.model.stats.trace, want["trace"], 1e-12)
    _close(got.model.stats.cost_ip, want["cost_ip"], 1e-11)
    _close(got.model.stats.constr_image, want["a_xbar"], 1e-11)
    if name == "dense":
        _close(got.model.store.xbar, want["xbar"], 1e-11)
    else:
        assert got.model.store.psi_seed == 5 and got.model.store.r == want["rank"]
        _close(got.model.store.sketch_mat, want["sketch"], 1e-10)
    # the file written from the padded device state equals the reference's
    # up to the recomputed floating-point statistics
    out = tmp_path / "pad.bin"
    S.save_state(out, got, p_big)
    d = OS.unpack(out.read_bytes())
    assert (d["n"], d["m"], d["b_hash"], d["kind"], d["rank"], d["psi_seed"], d["k_c"], d["k_p"]) == \
        (want["n"], want["m"], want["b_hash"], want["kind"], want["rank"], want["psi_seed"], want["k_c"], want["k_p"])


@pytest.mark.parametrize("name", ["dense", "sketch"])
@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")
def test_warm_started_solve_tracks_reference(tmp_path, name):
    from paper_2312_11801_b200 import solver as SV
    prev = S.record_to_state(S.load_state(_write(tmp_path, f"{name}/bin")))
    p_big = _prob("big")
    padded = S.warm_start_pad(prev, p_big, S.Mapping(np.arange(9), np.arange(9)),
                              sketch_seed=5 if name == "sketch" else None)
    rec = []
    cfg = SV.SolverConfig(k_c=4, k_p=1, eps=1e-3, max_iters=500, seed=0, sketch_rank=3 if name == "sketch" else 0)
    st, _ = SV.solve(p_big, cfg, init=padded, callback=rec.append)
    f = np.array([r.f_y for r in rec])
    want = G[f"{name}/warm_f"]
    n0 = min(6, len(want))
    np.testing.assert_allclose(f[:n0], want[:n0], rtol=1e-8)
    assert [r.step == "descent" for r in rec[:n0]] == [bool(x) for x in G[f"{name}/warm_step"][:n0]]
    conv, iters, desc = G[f"{name}/warm_status"]
    assert st.status == "converged" and bool(conv)
    assert abs(st.iterations - int(iters)) <= max(3, int(iters) // 5)


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")
def test_device_pad_rejects_bad_mappings(tmp_path):
    prev = S.record_to_state(S.load_state(_write(tmp_path, "dense/bin")))
    p_big = _prob("big")
    with pytest.raises(ValueError):
        S.warm_start_pad(prev, p_big, S.Mapping(np.array([0, 1, 10, 3, 4, 5, 6, 7, 8]), np.arange(9)))
    with pytest.raises(ValueError):
        S.warm_start_pad(prev, p_big, S.Mapping(np.arange(9), np.arange(8)))


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")
def test_solve_accepts_host_state():
    """A host state with the reference's attribute names (here the oracle's
    restatement of a loaded dense record) initialises the device solve."""
    from paper_2312_11801_b200 import solver as SV
    host = OS.to_state(OS.unpack(_raw("dense/bin")))
    p_small = _prob("small")
    cfg = SV.SolverConfig(k_c=4, k_p=1, eps=1e-3, max_iters=3, seed=0)
    rec = []
    SV.solve(p_small, cfg, init=host, callback=rec.append)
    assert len(rec) >= 1 or host.f_y is not None
