"""Pin the CPU oracle (oracle/usbs_cpu.py) against fixtures recorded from the
unmodified reference by oracle/make_golden.py.  CPU only."""
from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN
from helpers import TRAJ_CFG, builders_json, load_npz, random_graph, random_qap, traj_problem
from oracle import usbs_cpu as O
from paper_2312_11801_b200 import instances as inst


def sha(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def digest(p):
    out = {"n": int(p.n), "m": int(p.m), "indptr": sha(p.cost.indptr), "indices": sha(p.cost.indices),
           "data": sha(p.cost.data), "b": sha(p.b), "ineq": sha(np.asarray(p.ineq_mask, dtype=bool)),
           "scale_c": float(p.scale_c).hex(), "scale_x": float(p.scale_x).hex(),
           "alpha": float(p.alpha), "sense": int(p.sense)}
    c = p.constraints
    if hasattr(c, "idx"):
        out.update({"idx": sha(c.idx), "rows": sha(c.rows), "cols": sha(c.cols), "vals": sha(c.vals)})
    return out


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4s", "C5s", "er_12_0", "er_60_3", "er_100_5", "qap_3_1"])
def test_builders_bit_exact(name):
    """Graph/CSR/b/scales/family arrays identical to the reference builders."""
    ref = builders_json()[name]
    if name in ("C1", "C2", "C3"):
        p = inst.baseline_config(name).problem
    elif name == "C4s":
        p = inst.baseline_config("C4", small=True).problem
    elif name == "C5s":
        p = inst.baseline_config("C5", small=True).problem
    elif name.startswith("er_"):
        _, n, s = name.split("_")
        pp = {"12": 0.4, "60": 0.2, "100": 0.1}[n]
        p = inst.maxcut_problem(random_graph(int(n), pp, int(s)))
    else:
        p = inst.qap_problem(random_qap(3, 1))
    assert digest(p) == ref


def test_quad_oracle_frozen_values():
    """The reference's own frozen projected-gradient values (1e-5, as in
    pkg/tests/test_subqp.py:236-246) and the reference IPM value (bitwise)."""
    g = json.loads((GOLDEN / "quad_oracle.json").read_text())
    for s, want in g["values"].items():
        c = g["coeffs"][s]
        q = O.Coeffs(np.array(c["quad_ss"]), np.array(c["quad_s_eta"]), c["quad_eta"], np.array(c["lin_s"]),
                     c["lin_eta"], True, 3)
        r = O.ipm(q)
        assert r.value == pytest.approx(want, abs=1e-5)
        assert r.value == g["ipm_value"][s]


def test_lanczos_matches_reference():
    z = load_npz("lanczos.npz")
    for name in ("dense200", "dense300", "degenerate62"):
        a = z[f"{name}/A"]
        kc, inner, rst, seed = (int(x) for x in z[f"{name}/args"])
        r = O.lanczos(O.Op(a.shape[0], lambda v: a @ v, lambda b: a @ b), kc, inner, rst, None, seed)
        np.testing.assert_array_equal(r.eigenvalues, z[f"{name}/vals"])
        np.testing.assert_array_equal(r.eigenvectors, z[f"{name}/vecs"])
        assert [int(r.converged), r.restarts] == z[f"{name}/meta"].tolist()
    p = inst.baseline_config("C1").problem
    r = O.lanczos(O.slack_op(p, z["c1/y"]), 10, seed=0)
    np.testing.assert_array_equal(r.eigenvalues, z["c1/vals"])
    np.testing.assert_array_equal(r.eigenvectors, z["c1/vecs"])
    np.testing.assert_array_equal(r.ritz_history, z["c1/hist"])


def test_ipm_matches_reference():
    z = load_npz("ipm.npz")
    for seed in range(4):
        pre = f"quad{seed}"
        qe, le, he, k = z[pre + "/scal"]
        q = O.Coeffs(z[pre + "/Q"], z[pre + "/q12"], float(qe), z[pre + "/h"], float(le), bool(he), int(k))
        r = O.ipm(q)
        np.testing.assert_array_equal(r.s_opt, z[pre + "/S"])
        assert [r.eta_opt, r.value, r.newton_iters, int(r.exact)] == z[pre + "/out"].tolist()
        e = O.ipm(O.linear_coeffs(q.lin_s, q.lin_eta, q.has_eta, q.k))
        np.testing.assert_array_equal(e.s_opt, z[pre + "/evalS"])


def test_constraint_ops_match_reference():
    z = load_npz("cons.npz")
    for tag, p in (("mc", inst.maxcut_problem(random_graph(12, 0.4, 0))), ("qap", inst.qap_problem(random_qap(3, 1)))):
        y, v, s, lam = z[f"{tag}/y"], z[f"{tag}/V"], z[f"{tag}/S"], z[f"{tag}/lam"]
        c = p.constraints
        np.testing.assert_array_equal(O.image_lowrank(c, v, s), z[f"{tag}/img_lowrank"])
        np.testing.assert_array_equal(O.image_factor(c, v, lam), z[f"{tag}/img_factor"])
        np.testing.assert_array_equal(O.adjoint_gram(c, y, v, p.n), z[f"{tag}/adj_gram"])
        np.testing.assert_array_equal(O.compressed(c, v), z[f"{tag}/compressed"])
        np.testing.assert_array_equal(O.cost_gram(p, v), z[f"{tag}/cost_quad"])
        assert O.cost_ip(p, v, lam) == z[f"{tag}/cost_ip"][0]
        np.testing.assert_array_equal(O.slack_op(p, y).matmat(v), z[f"{tag}/Zv"])


def test_sketch_matches_reference():
    z = load_npz("sketch.npz")
    assert O.sketch_seed(0) == int(z["derived_seed0"][0])
    sk = O.sketch_new(50, 6, int(z["seed"][0]))
    np.testing.assert_array_equal(sk.psi, z["psi"])
    for t in range(3):
        sk = O.sketch_apply(sk, float(z[f"step{t}/eta"][0]), z[f"step{t}/F"], z[f"step{t}/lam"])
        np.testing.assert_array_equal(sk.p, z[f"step{t}/P"])
    u, lam = O.sketch_factor(sk)
    np.testing.assert_array_equal(lam, z["lams"])
    np.testing.assert_array_equal(u, z["U"])


@pytest.mark.parametrize("name", list(TRAJ_CFG))
def test_solve_trajectory_matches_reference(name):
    """Free-running solve() trajectories are reproduced bit for bit (same
    numpy/scipy build); this pins every branch of the outer loop."""
    z = load_npz(f"traj_{name}.npz")
    p = traj_problem(name)
    cfg = O.Config(**TRAJ_CFG[name])
    rec = []
    st, _ = O.solve(p, cfg, callback=rec.append)
    np.testing.assert_array_equal([r.f_y for r in rec], z["f_y"])
    np.testing.assert_array_equal([r.f_cand for r in rec], z["f_cand"])
    np.testing.assert_array_equal([r.model_val for r in rec], z["model_val"])
    np.testing.assert_array_equal([1 if r.step == "descent" else 0 for r in rec], z["step"])
    np.testing.assert_array_equal([r.residuals.rel_infeas for r in rec], z["rel_infeas"])
    np.testing.assert_array_equal(st.y, z["y"])


def test_lockstep_snapshot_c1():
    """Inject the reference state at t=10 and reproduce iteration 11 exactly."""
    z = load_npz("lockstep_c1.npz")
    p = inst.baseline_config("C1").problem
    cfg = O.Config(rho=0.01, beta=0.25, k_c=10, k_p=1, sketch_rank=0, max_iters=1, seed=0)
    st = O.State(z["y"].copy(), z["nu"].copy(), float(z["f_y"]), float(z["lam_y"]),
                 O.Model(z["basis"].copy(), O.Stats(float(z["trace"]), float(z["cost_ip"]), z["image"].copy()),
                         10, 1, O.Dense(z["xbar"].copy())))
    st.last_primal = st.model.stats.copy()
    rec = []
    O.solve(p, cfg, init=st, callback=rec.append)
    r = rec[0]
    assert r.f_cand == float(z["n_f_cand"])
    assert r.model_val == float(z["n_model_val"])
    np.testing.assert_array_equal(r.y_cand, z["n_y_cand"])
    np.testing.assert_array_equal(r.primal.constr_image, z["n_image"])


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_builders_full_size_bit_exact(name):
    """Full-size C4 (n = 10^6 through GraphInstance.from_edges, problem.py:67-87)
    and C5 (n = 63,000, m = 1.37 M through build_from_families,
    problem.py:509-539): every array hash-equal to the reference builders'
    (builders_full.json, recorded by oracle/make_golden.py builders_full)."""
    ref = json.loads((GOLDEN / "builders_full.json").read_text())[name]
    assert digest(inst.baseline_config(name).problem) == ref
