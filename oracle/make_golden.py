"""Record golden fixtures by running the UNMODIFIED reference (test infrastructure).

Run in the authoring container, where /root/reference exists:

    python oracle/make_golden.py

It imports ``specbundle`` from /root/reference/pkg/src (read-only; nothing is
copied) and writes small .npz/.json fixtures under tests/golden/.  The GPU box
never sees /root/reference; the tests there compare the oracle and the device
path against these files.

Fixtures:
  builders.json      sha256 of every array the reference builders emit for
                     C1, C2, C3 and a small C4/C5, plus scale factors
  quad_oracle.json   the reference's own frozen projected-gradient values
                     (pkg/tests/data_quad_oracle.json) + its coefficient
                     generator outputs (pkg/tests/_oracles.py:105-127)
  lanczos.npz        lanczos_top outputs on dense and MaxCut operators
  ipm.npz            ipm_quad / ipm_eval outputs on seeded coefficients
  cons.npz           constraint-operator outputs (diag + QAP families)
  sketch.npz         sketch_update / reconstruct outputs
  traj_*.npz         per-iteration solve() trajectories of small problems
  lockstep_c1.npz    C1 state snapshot at t=10 and reference iteration 11
  rounding.npz       maxcut_round / qap_round (rounding.py) on seeded factors
  state.npz          USBS v1 state-file bytes (save_state) of solved states,
                     warm_start_pad outputs and the warm-started trajectory
  cli.json           front end: instance readers on valid/malformed files,
                     writers, perturb outputs, solve CSV rows and round output
"""
from __future__ import annotations

import copy
import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
OUT = ROOT / "tests" / "golden"

import specbundle as sb  # noqa: E402
from specbundle import bundle as sbb  # noqa: E402
from specbundle import problem as sbp  # noqa: E402
from specbundle import subqp as sbq  # noqa: E402
from specbundle import sketch as sbs  # noqa: E402
from specbundle.eigsolve import LinOp, lanczos_top  # noqa: E402

from paper_2312_11801_b200 import instances as inst  # noqa: E402


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def problem_digest(p) -> dict:
    out = {
        "n": int(p.n), "m": int(p.m),
        "indptr": sha(p.cost.indptr), "indices": sha(p.cost.indices), "data": sha(p.cost.data),
        "b": sha(p.b), "ineq": sha(np.asarray(p.ineq_mask, dtype=bool)),
        "scale_c": float(p.scale_c).hex(), "scale_x": float(p.scale_x).hex(),
        "alpha": float(p.alpha), "sense": int(p.sense),
    }
    c = p.constraints
    if hasattr(c, "idx"):
        out.update({"idx": sha(c.idx), "rows": sha(c.rows), "cols": sha(c.cols), "vals": sha(c.vals)})
    return out


def ref_problem(cfg_name: str):
    """Build the reference's SdpProblem for a config from the same raw inputs."""
    if cfg_name == "C1":
        from conftest import random_graph
        return sbp.build_maxcut(random_graph(800, 0.06, 0))
    if cfg_name == "C2":
        g = inst.torus_pm1(100, 1)
        edges = list(zip(g.eu.tolist(), g.ev.tolist(), g.ew.tolist()))
        # rebuild the raw (unsorted) edge list exactly as SURVEY 8d specifies
        side = 100
        raw = []
        for i in range(side):
            for j in range(side):
                v = side * i + j
                raw.append((v, side * ((i + 1) % side) + j))
                raw.append((v, side * i + (j + 1) % side))
        r = np.random.default_rng(1).random(len(raw))
        raw_w = [(a, b, 1.0 if r[e] < 0.5 else -1.0) for e, (a, b) in enumerate(raw)]
        del edges
        return sbp.build_maxcut(sbp.GraphInstance.from_edges(side * side, raw_w))
    if cfg_name == "C3":
        q = inst.qap_random(20, 2)
        return sbp.build_qap(sbp.QapInstance(q.weights, q.distances))
    if cfg_name == "C4s":
        g = inst.chung_lu(20_000, seed=3)
        gi = sbp.GraphInstance.from_edges(g.n, list(zip(g.eu.tolist(), g.ev.tolist(), g.ew.tolist())))
        return sbp.build_maxcut(gi)
    if cfg_name == "C4":
        # full size: from_edges over the de-duplicated Chung-Lu edge list
        g = inst.chung_lu(1_000_000, seed=3)
        gi = sbp.GraphInstance.from_edges(g.n, list(zip(g.eu.tolist(), g.ev.tolist(), g.ew.tolist())))
        return sbp.build_maxcut(gi)
    if cfg_name in ("C5s", "C5"):
        n, eu, ev, ew = (inst.knn_correlation(n=3000, clusters=100, seed=4) if cfg_name == "C5s"
                         else inst.knn_correlation(seed=4))
        import scipy.sparse as sp
        cost = sp.coo_matrix((np.concatenate([ew, ew]), (np.concatenate([eu, ev]), np.concatenate([ev, eu]))),
                             shape=(n, n)).tocsr()
        ne = eu.size
        d = np.arange(n)
        idx = np.concatenate([d, n + np.arange(ne)])
        rows = np.concatenate([d, eu])
        cols = np.concatenate([d, ev])
        vals = np.concatenate([np.ones(n), np.full(ne, -0.5)])
        b = np.concatenate([np.ones(n), np.zeros(ne)])
        ineq = np.concatenate([np.zeros(n, bool), np.ones(ne, bool)])
        return sbp.build_from_families(n, cost, (idx, rows, cols, vals), b, ineq, scale_x=float(n))
    raise KeyError(cfg_name)


def mine_problem(cfg_name: str):
    if cfg_name == "C4s":
        return inst.baseline_config("C4", small=True).problem
    if cfg_name == "C5s":
        return inst.baseline_config("C5", small=True).problem
    return inst.baseline_config(cfg_name).problem


def builders_full():
    """Full-size C4 (n = 10^6) and C5 (n = 63,000, m = 1.37 M) through the
    reference builders (from_edges / build_from_families), hashed like
    builders(); written to builders_full.json."""
    rec = {}
    for name in ("C4", "C5"):
        rp = ref_problem(name)
        rec[name] = problem_digest(rp)
        md = problem_digest(mine_problem(name))
        print(f"builders {name}: framework builder bit-exact vs reference = {md == rec[name]}", flush=True)
        del rp
    (OUT / "builders_full.json").write_text(json.dumps(rec, indent=1, sort_keys=True))


def builders():
    rec = {}
    for name in ("C1", "C2", "C3", "C4s", "C5s"):
        rp = ref_problem(name)
        rec[name] = problem_digest(rp)
        mp = mine_problem(name)
        md = problem_digest(mp)
        same = md == rec[name]
        print(f"builders {name}: framework builder bit-exact vs reference = {same}")
        if not same:
            for k in rec[name]:
                if rec[name][k] != md.get(k):
                    print("   differs:", k)
    # reference generators used by its own tests (conftest.py:25-41)
    from conftest import random_graph, random_qap
    for (n, p, s) in ((12, 0.4, 0), (60, 0.2, 3), (100, 0.1, 5)):
        rec[f"er_{n}_{s}"] = problem_digest(sbp.build_maxcut(random_graph(n, p, s)))
    rec["qap_3_1"] = problem_digest(sbp.build_qap(random_qap(3, 1)))
    (OUT / "builders.json").write_text(json.dumps(rec, indent=1, sort_keys=True))


def quad_oracle():
    from _oracles import random_quad_coeffs
    frozen = json.loads((REF / "tests" / "data_quad_oracle.json").read_text())
    out = {"source": "pkg/tests/data_quad_oracle.json (reference, frozen 1e6-step projected gradient)",
           "steps": frozen["steps"], "k": frozen["k"], "values": frozen["values"], "coeffs": {},
           "ipm_value": {}}
    for s in frozen["values"]:
        c = random_quad_coeffs(int(s))
        out["coeffs"][s] = {"quad_ss": c.quad_ss.tolist(), "quad_s_eta": c.quad_s_eta.tolist(),
                            "quad_eta": c.quad_eta, "lin_s": c.lin_s.tolist(), "lin_eta": c.lin_eta}
        out["ipm_value"][s] = sbq.ipm_quad(c).value
    (OUT / "quad_oracle.json").write_text(json.dumps(out))


def lanczos_cases():
    data = {}
    rng = np.random.default_rng(42)
    a = rng.standard_normal((200, 200)); a = 0.5 * (a + a.T)
    cases = {"dense200": (a, 5, 32, 10, 1)}
    rng = np.random.default_rng(3)
    b = rng.standard_normal((300, 300)); b = 0.5 * (b + b.T)
    cases["dense300"] = (b, 8, 16, 10, 0)
    d = np.array([4.0, 4.0] + [1.0] * 60)
    q, _ = np.linalg.qr(np.random.default_rng(5).standard_normal((62, 62)))
    cases["degenerate62"] = ((q * d[None, :]) @ q.T, 2, 32, 10, 0)
    for name, (mat, kc, inner, rst, seed) in cases.items():
        r = lanczos_top(LinOp(mat.shape[0], lambda v, m=mat: m @ v, lambda x, m=mat: m @ x), kc,
                        inner_iters=inner, max_restarts=rst, seed=seed)
        data[f"{name}/A"] = mat
        data[f"{name}/args"] = np.array([kc, inner, rst, seed])
        data[f"{name}/vals"] = r.eigenvalues
        data[f"{name}/vecs"] = r.eigenvectors
        data[f"{name}/res"] = r.residuals
        data[f"{name}/meta"] = np.array([int(r.converged), r.restarts])
        data[f"{name}/hist"] = np.array(r.ritz_history)
    # MaxCut C1 slack operator at a seeded dual (C1 arrays recomputed from builders on the box)
    p = ref_problem("C1")
    y = np.random.default_rng(1234).standard_normal(p.m) * 1e-3
    r = lanczos_top(sbp.dual_slack_operator(p, y), 10, seed=0)
    data["c1/y"] = y
    data["c1/vals"] = r.eigenvalues
    data["c1/vecs"] = r.eigenvectors
    data["c1/res"] = r.residuals
    data["c1/meta"] = np.array([int(r.converged), r.restarts])
    data["c1/hist"] = np.array(r.ritz_history)
    np.savez_compressed(OUT / "lanczos.npz", **data)


def ipm_cases():
    data = {}
    for seed, k, has_eta in ((0, 3, True), (1, 4, False), (2, 6, True), (3, 11, True)):
        rng = np.random.default_rng(100 + seed)
        d = k * (k + 1) // 2
        a = rng.standard_normal((d + 2, d))
        z = rng.standard_normal(d + 2)
        c = sbq.QuadCoeffs(quad_ss=a.T @ a / (d + 2), quad_s_eta=(a.T @ z / (d + 2)) if has_eta else np.zeros(d),
                           quad_eta=float(z @ z / (d + 2)) if has_eta else 0.0,
                           lin_s=rng.standard_normal(d), lin_eta=float(rng.standard_normal()) if has_eta else 0.0,
                           has_eta=has_eta, k=k)
        r = sbq.ipm_quad(c)
        pre = f"quad{seed}"
        data[pre + "/Q"] = c.quad_ss; data[pre + "/q12"] = c.quad_s_eta
        data[pre + "/scal"] = np.array([c.quad_eta, c.lin_eta, float(has_eta), k])
        data[pre + "/h"] = c.lin_s
        data[pre + "/S"] = r.s_opt; data[pre + "/out"] = np.array([r.eta_opt, r.value, r.newton_iters, int(r.exact)])
        e = sbq.ipm_eval(sbq.EvalCoeffs(lin_s=c.lin_s, lin_eta=c.lin_eta, has_eta=has_eta, k=k))
        data[pre + "/evalS"] = e.s_opt
        data[pre + "/evalout"] = np.array([e.eta_opt, e.value, e.newton_iters, int(e.exact)])
    np.savez_compressed(OUT / "ipm.npz", **data)


def cons_cases():
    from conftest import random_graph, random_qap
    data = {}
    for tag, p in (("mc", sbp.build_maxcut(random_graph(12, 0.4, 0))), ("qap", sbp.build_qap(random_qap(3, 1)))):
        rng = np.random.default_rng(5)
        y = rng.standard_normal(p.m)
        v, _ = np.linalg.qr(rng.standard_normal((p.n, 3)))
        s = rng.standard_normal((3, 3)); s = s @ s.T
        lam = np.abs(rng.standard_normal(3))
        c = p.constraints
        data[f"{tag}/y"] = y; data[f"{tag}/V"] = v; data[f"{tag}/S"] = s; data[f"{tag}/lam"] = lam
        data[f"{tag}/img_lowrank"] = c.primal_image_lowrank(v, s)
        data[f"{tag}/img_factor"] = c.primal_image_factor(v, lam)
        data[f"{tag}/adj_gram"] = c.adjoint_inner_lowrank(y, v)
        data[f"{tag}/compressed"] = c.compressed_rows(v)
        data[f"{tag}/cost_quad"] = p.cost_quad(v)
        data[f"{tag}/cost_ip"] = np.array([p.cost_factor_ip(v, lam)])
        data[f"{tag}/Zv"] = sbp.dual_slack_operator(p, y).matmat(v)
    np.savez_compressed(OUT / "cons.npz", **data)


def sketch_cases():
    data = {}
    n, r = 50, 6
    sk = sbs.sketch_init(n, r, 12345)
    rng = np.random.default_rng(9)
    for t in range(3):
        f, _ = np.linalg.qr(rng.standard_normal((n, 2)))
        lam = np.abs(rng.standard_normal(2))
        eta = 0.5 + 0.1 * t
        data[f"step{t}/F"] = f; data[f"step{t}/lam"] = lam; data[f"step{t}/eta"] = np.array([eta])
        sk = sbs.sketch_update(sk, eta, f, np.eye(2), lam)
        data[f"step{t}/P"] = sk.sketch_mat
    u, lam = sbs.reconstruct(sk)
    data["psi"] = sk.psi(); data["U"] = u; data["lams"] = lam
    data["seed"] = np.array([12345]); data["derived_seed0"] = np.array([sbb._derived_seeds(0)[0]], dtype=np.uint64)
    np.savez_compressed(OUT / "sketch.npz", **data)


def trajectory(name, prob, cfg, iters):
    rec = {k: [] for k in ("f_y", "f_cand", "model_val", "step", "rel_subopt", "rel_infeas",
                           "dual_feas", "lam_cand", "eta", "trace", "cost_ip")}

    def cb(info):
        rec["f_y"].append(info.f_y); rec["f_cand"].append(info.f_cand)
        rec["model_val"].append(info.model_val); rec["step"].append(1 if info.step == "descent" else 0)
        rec["rel_subopt"].append(info.residuals.rel_subopt); rec["rel_infeas"].append(info.residuals.rel_infeas)
        rec["dual_feas"].append(info.residuals.dual_feas); rec["lam_cand"].append(info.lam_cand)
        rec["eta"].append(info.eta); rec["trace"].append(info.primal.trace); rec["cost_ip"].append(info.primal.cost_ip)

    cfg.max_iters = iters
    st, out = sbb.solve(prob, cfg, callback=cb)
    data = {k: np.array(v, dtype=float) for k, v in rec.items()}
    data["y"] = st.y
    data["status"] = np.array([st.status == "converged", st.iterations, st.descent_steps])
    data["final_lams"] = out.lams
    np.savez_compressed(OUT / f"traj_{name}.npz", **data)
    print(f"trajectory {name}: {st.iterations} its, status {st.status}")


def trajectories():
    from conftest import make_k3, mixed_inequality_problem, random_graph
    trajectory("k3", sbp.build_maxcut(make_k3()), sbb.SolverConfig(k_c=1, k_p=1), 200)
    trajectory("er60", sbp.build_maxcut(random_graph(60, 0.2, 3)), sbb.SolverConfig(), 40)
    trajectory("er60_sketch", sbp.build_maxcut(random_graph(60, 0.2, 3)), sbb.SolverConfig(sketch_rank=5), 40)
    p, _ = mixed_inequality_problem(40, 2, n_ineq=8)
    trajectory("mixed40", p, sbb.SolverConfig(k_c=4, k_p=1, sketch_rank=4), 30)
    # the mixed problem arrays for reconstruction on the box
    c = p.constraints
    np.savez_compressed(OUT / "prob_mixed40.npz", n=p.n, m=p.m, indptr=p.cost.indptr, indices=p.cost.indices,
                        data=p.cost.data, b=p.b, ineq=p.ineq_mask, idx=c.idx, rows=c.rows, cols=c.cols,
                        vals=c.vals, scal=np.array([p.alpha, p.scale_c, p.scale_x]))
    from conftest import random_qap
    trajectory("qap4", sbp.build_qap(random_qap(4, 0)), sbb.SolverConfig(rho=0.005, k_c=4, k_p=0, sketch_rank=4), 20)


def lockstep():
    p = ref_problem("C1")
    cfg = sbb.SolverConfig(rho=0.01, beta=0.25, k_c=10, k_p=1, eps=1e-3, sketch_rank=0, max_iters=11, seed=0)
    snaps = {}

    def cb(info):
        if info.t == 9:
            s = copy.deepcopy(info.state)
            s.nu = info.nu_cand.copy()
            snaps["s"] = s
        if info.t == 10:
            snaps["next"] = (info.f_y, info.f_cand, info.model_val, info.step, info.y_cand.copy(),
                             info.primal.constr_image.copy(), info.primal.trace, info.primal.cost_ip,
                             info.residuals.rel_subopt, info.residuals.rel_infeas, info.lam_cand)

    sbb.solve(p, cfg, callback=cb)
    s = snaps["s"]
    nx = snaps["next"]
    np.savez_compressed(
        OUT / "lockstep_c1.npz",
        y=s.y, nu=s.nu, f_y=s.f_y, lam_y=s.lam_y, basis=s.model.basis, trace=s.model.stats.trace,
        cost_ip=s.model.stats.cost_ip, image=s.model.stats.constr_image, xbar=s.model.store.xbar,
        descent=s.descent_steps, null=s.null_steps,
        n_f_y=nx[0], n_f_cand=nx[1], n_model_val=nx[2], n_step=1 if nx[3] == "descent" else 0,
        n_y_cand=nx[4], n_image=nx[5], n_trace=nx[6], n_cost_ip=nx[7], n_rel_subopt=nx[8],
        n_rel_infeas=nx[9], n_lam_cand=nx[10])


def rounding_cases():
    """maxcut_round (rounding.py:34-51) and qap_round (rounding.py:72-93) of
    the unmodified reference on seeded factors (with exact zeros, which sign
    to +1)."""
    from conftest import random_graph, random_qap
    from specbundle import rounding as sbr
    data = {}
    graphs = {
        "er": random_graph(300, 0.05, 3),
        "torus": sbp.GraphInstance.from_edges(
            400, [(20 * i + j, 20 * ((i + 1) % 20) + j, 1.0 if k % 3 else -1.0)
                  for k, (i, j) in enumerate((i, j) for i in range(20) for j in range(20))] +
            [(20 * i + j, 20 * i + (j + 1) % 20, 1.0) for i in range(20) for j in range(20)]),
    }
    for name, g in graphs.items():
        rng = np.random.default_rng(11)
        u = rng.standard_normal((g.n, 7))
        u[rng.random(u.shape) < 0.05] = 0.0
        res = sbr.maxcut_round(u, g)
        data[f"{name}/eu"], data[f"{name}/ev"], data[f"{name}/ew"] = g.edges_u, g.edges_v, g.edges_w
        data[f"{name}/u"] = u
        data[f"{name}/x"] = res.assignment
        data[f"{name}/value"] = np.array([res.value])
        data[f"{name}/all"] = np.array([0.25 * float(np.where(u[:, j] >= 0, 1.0, -1.0) @ (
            g.laplacian() @ np.where(u[:, j] >= 0, 1.0, -1.0))) for j in range(u.shape[1])])
    for size, seed in ((4, 1), (6, 2)):
        q = random_qap(size, seed)
        rng = np.random.default_rng(5 + size)
        u = rng.standard_normal((size * size + 1, 5))
        res = sbr.qap_round(u, q)
        key = f"qap{size}"
        data[f"{key}/W"], data[f"{key}/D"], data[f"{key}/u"] = q.weights, q.distances, u
        data[f"{key}/perm"] = res.perm
        data[f"{key}/objective"] = np.array([res.objective])
    np.savez_compressed(OUT / "rounding.npz", **data)


def state_cases():
    """save_state bytes (bundle.py:578-622) of solved states, warm_start_pad
    (bundle.py:754-817) into a graph with one more vertex (the reference's
    test_bundle.py:373-394 construction), and the solve warm-started from it."""
    import tempfile
    from conftest import make_k3, random_graph
    data = {}

    def state_bytes(st, prob):
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "s.bin")
            sbb.save_state(path, st, prob)
            return np.frombuffer(open(path, "rb").read(), dtype=np.uint8).copy()

    k3p = sbp.build_maxcut(make_k3())
    st, _ = sbb.solve(k3p, sbb.SolverConfig(eps=1e-3, max_iters=200, seed=0, sketch_rank=2))
    data["k3_sketch/bin"] = state_bytes(st, k3p)
    g_small = random_graph(9, 0.5, 60)
    edges = list(zip(g_small.edges_u, g_small.edges_v, g_small.edges_w))
    edges.append((0, 9, 1.0))
    g_big = sbp.GraphInstance.from_edges(10, [(int(a), int(b), float(c)) for a, b, c in edges])
    data["big/eu"], data["big/ev"], data["big/ew"] = g_big.edges_u, g_big.edges_v, g_big.edges_w
    data["small/eu"], data["small/ev"], data["small/ew"] = g_small.edges_u, g_small.edges_v, g_small.edges_w
    p_small, p_big = sbp.build_maxcut(g_small), sbp.build_maxcut(g_big)
    for name, rank, seed in (("dense", 0, None), ("sketch", 3, 5)):
        cfg = sbb.SolverConfig(k_c=4, k_p=1, eps=1e-3, max_iters=500, seed=0, sketch_rank=rank)
        st, _ = sbb.solve(p_small, cfg)
        data[f"{name}/bin"] = state_bytes(st, p_small)
        padded = sbb.warm_start_pad(st, p_big, sbb.Mapping(np.arange(9), np.arange(9)), sketch_seed=seed)
        data[f"{name}/pad_bin"] = state_bytes(padded, p_big)
        fs = []
        cfg2 = sbb.SolverConfig(k_c=4, k_p=1, eps=1e-3, max_iters=500, seed=0, sketch_rank=rank)
        st2, _ = sbb.solve(p_big, cfg2, init=padded, callback=lambda i: fs.append((i.f_y, i.step == "descent")))
        data[f"{name}/warm_f"] = np.array([f for f, _ in fs])
        data[f"{name}/warm_step"] = np.array([d for _, d in fs], dtype=np.int8)
        data[f"{name}/warm_status"] = np.array([st2.status == "converged", st2.iterations, st2.descent_steps])
        print(f"state {name}: warm {st2.status} in {st2.iterations} its")
    np.savez_compressed(OUT / "state.npz", **data)


# instance files for the front-end fixtures: (name, text); valid and malformed
MM_FILES = [
    ("k3_pattern", "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 3\n2 1\n3 1\n3 2\n"),
    ("general_mirrored", "%%MatrixMarket matrix coordinate real general\n% a comment\n\n4 4 6\n1 2 0.5\n2 1 0.5\n"
     "3 4 -2.25\n4 3 -2.25\n2 2 7\n1 1 3\n"),
    ("integer_dups_diag", "%%MatrixMarket matrix coordinate integer symmetric\n5 5 6\n2 1 3\n1 2 4\n5 5 9\n"
     "4 3 -1\n5 1 2\n3 4 1\n"),
    ("empty", ""),
    ("no_header", "3 3 1\n2 1\n"),
    ("array", "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n"),
    ("complex", "%%MatrixMarket matrix coordinate complex symmetric\n2 2 1\n2 1 1 0\n"),
    ("hermitian", "%%MatrixMarket matrix coordinate real hermitian\n2 2 1\n2 1 1\n"),
    ("no_size", "%%MatrixMarket matrix coordinate real symmetric\n% only comments\n"),
    ("size_fields", "%%MatrixMarket matrix coordinate real symmetric\n3 3\n"),
    ("size_bad", "%%MatrixMarket matrix coordinate real symmetric\n3 x 1\n2 1 1\n"),
    ("not_square", "%%MatrixMarket matrix coordinate real symmetric\n3 4 1\n2 1 1\n"),
    ("few_fields", "%%MatrixMarket matrix coordinate real symmetric\n3 3 1\n2 1\n"),
    ("bad_value", "%%MatrixMarket matrix coordinate real symmetric\n3 3 1\n2 1 abc\n"),
    ("out_of_range", "%%MatrixMarket matrix coordinate real symmetric\n3 3 1\n4 1 1\n"),
    ("count", "%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n2 1 1\n"),
    ("no_mirror", "%%MatrixMarket matrix coordinate real general\n3 3 2\n2 1 1\n3 1 1\n"),
    ("mirror_mismatch", "%%MatrixMarket matrix coordinate real general\n3 3 2\n2 1 1\n1 2 2\n"),
]
QAP_FILES = [
    ("qap3", "3\n\n0 1 2\n1 0\n3\n2 3 0\n\n0 5 6 5 0 7\n6 7 0\n"),
    ("empty", ""),
    ("bad_size", "x\n0 1\n1 0\n"),
    ("nonpositive", "0\n"),
    ("short", "2\n0 1 1 0\n0 2\n"),
    ("trailing", "1\n0\n0\n5\n"),
    ("bad_entry", "2\n0 1 1 0\n0 2 q 0\n"),
    ("asymmetric", "2\n0 1 2 0\n0 2 2 0\n"),
]


def cli_cases():
    """Front end (cli.py, problem.py:546-681) of the unmodified reference:
    the readers on valid and malformed files (edges or the error text and
    line), the writers' bytes, perturb outputs, and solve/round runs (CSV
    rows without the time column, stdout)."""
    import contextlib
    import io
    import tempfile
    from conftest import random_graph, random_qap
    from specbundle import cli as sbc
    out = {"mm": {}, "qap": {}, "files": {"mm": MM_FILES, "qap": QAP_FILES}}
    with tempfile.TemporaryDirectory() as d:
        def put(name, text):
            path = os.path.join(d, name)
            with open(path, "w") as fh:
                fh.write(text)
            return path

        for name, text in MM_FILES:
            try:
                g = sbp.parse_graph_mm(put(name + ".mtx", text))
                out["mm"][name] = {"n": g.n, "u": g.edges_u.tolist(), "v": g.edges_v.tolist(), "w": g.edges_w.tolist()}
            except sbp.ParseError as exc:
                out["mm"][name] = {"error": str(exc), "line": exc.line}
        for name, text in QAP_FILES:
            try:
                q = sbp.parse_qaplib(put(name + ".dat", text))
                out["qap"][name] = {"W": q.weights.tolist(), "D": q.distances.tolist()}
            except sbp.ParseError as exc:
                out["qap"][name] = {"error": str(exc), "line": exc.line}
        g = random_graph(50, 0.2, 2)
        gp = os.path.join(d, "g.mtx")
        sbp.write_graph_mm(g, gp)
        out["write_graph"] = open(gp).read()
        q = random_qap(4, 1)
        qp = os.path.join(d, "q.dat")
        sbp.write_qaplib(q, qp)
        out["write_qap"] = open(qp).read()
        out["perturb"] = {}
        for kind, src, frac in (("maxcut", gp, "0.1"), ("qap", qp, "0.5")):
            si, sm = os.path.join(d, f"sub_{kind}"), os.path.join(d, f"map_{kind}.json")
            with contextlib.redirect_stdout(io.StringIO()) as so:
                rc = sbc.main(["perturb", "--problem", kind, "--input", src, "--fraction", frac,
                               "--out-instance", si, "--out-mapping", sm])
            out["perturb"][kind] = {"rc": rc, "instance": open(si).read(), "mapping": json.load(open(sm)),
                                    "stdout": so.getvalue().splitlines()[0]}
        k3 = put("k3.mtx", MM_FILES[0][1])
        q3 = put("q3.dat", QAP_FILES[0][1])
        out["solve"] = {}
        for tag, argv in (
                ("k3_round", ["solve", "--problem", "maxcut", "--input", k3, "--eps", "1e-3", "--round", "--seed", "5"]),
                ("k3_budget", ["solve", "--problem", "maxcut", "--input", k3, "--max-iters", "0"]),
                ("g50", ["solve", "--problem", "maxcut", "--input", gp, "--max-iters", "25", "--round"]),
                ("qap3", ["solve", "--problem", "qap", "--input", q3, "--max-iters", "20", "--round",
                          "--optimum", "40"])):
            csvp = os.path.join(d, tag + ".csv")
            st = os.path.join(d, tag + ".bin")
            with contextlib.redirect_stdout(io.StringIO()) as so:
                rc = sbc.main(argv + ["--out", csvp, "--save-state", st])
            rows = [r.split(",") for r in open(csvp).read().splitlines()]
            rows = [[c for i, c in enumerate(r) if i != 1] for r in rows]
            res = {"rc": rc, "rows": rows, "stdout": so.getvalue().splitlines()}
            kind = argv[2]
            with contextlib.redirect_stdout(io.StringIO()) as so2:
                res["round_rc"] = sbc.main(["round", "--problem", kind, "--input", argv[4], "--state", st])
            res["round_stdout"] = so2.getvalue().splitlines()
            out["solve"][tag] = res
    with open(OUT / "cli.json", "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    OUT.mkdir(parents=True, exist_ok=True)
    which = sys.argv[1:] or ["builders", "quad", "lanczos", "ipm", "cons", "sketch", "traj", "lockstep", "rounding", "state"]
    fn = {"builders": builders, "builders_full": builders_full, "quad": quad_oracle, "lanczos": lanczos_cases, "ipm": ipm_cases,
          "cons": cons_cases, "sketch": sketch_cases, "traj": trajectories, "lockstep": lockstep,
          "rounding": rounding_cases, "state": state_cases, "cli": cli_cases}
    for w in which:
        fn[w]()
        print("wrote", w)
