"""Shared test helpers: problem reconstruction for the golden fixtures.

The generators restate the reference's own test generators
(/root/reference/pkg/tests/conftest.py:21-41) so fixtures recorded from the
reference can be rebuilt without it.
"""
from __future__ import annotations

import json

import numpy as np
import scipy.sparse as sp

from paper_2312_11801_b200 import instances as inst

from conftest import GOLDEN


def random_graph(n, p, seed):
    """conftest.py:25-30."""
    return inst.erdos_renyi(n, p, seed)


def random_qap(n, seed, lo=0, hi=10):
    """conftest.py:33-41."""
    rng = np.random.default_rng(seed)
    w = rng.integers(lo, hi, (n, n)).astype(float)
    w = w + w.T
    np.fill_diagonal(w, 0.0)
    d = rng.integers(lo, hi, (n, n)).astype(float)
    d = d + d.T
    np.fill_diagonal(d, 0.0)
    return inst.Qap(w, d)


def k3():
    return inst.Graph.from_edge_list(3, [(0, 1, 1.0), (0, 2, 1.0), (1, 2, 1.0)])


def load_npz(name):
    z = np.load(GOLDEN / name, allow_pickle=False)
    return {k: z[k] for k in z.files}


def mixed40():
    z = load_npz("prob_mixed40.npz")
    n, m = int(z["n"]), int(z["m"])
    cost = sp.csr_matrix((z["data"], z["indices"], z["indptr"]), shape=(n, n))
    alpha, sc, sx = z["scal"]
    return inst.Problem(n=n, m=m, cost=cost,
                        constraints=inst.EntryFamilies(n, m, z["idx"], z["rows"], z["cols"], z["vals"]),
                        b=z["b"], ineq_mask=z["ineq"], alpha=float(alpha), scale_c=float(sc),
                        scale_x=float(sx), sense=1)


def builders_json():
    return json.loads((GOLDEN / "builders.json").read_text())


def traj_problem(name):
    if name == "k3":
        return inst.maxcut_problem(k3())
    if name in ("er60", "er60_sketch"):
        return inst.maxcut_problem(random_graph(60, 0.2, 3))
    if name == "mixed40":
        return mixed40()
    if name == "qap4":
        return inst.qap_problem(random_qap(4, 0))
    raise KeyError(name)


TRAJ_CFG = {
    "k3": dict(k_c=1, k_p=1, max_iters=200),
    "er60": dict(max_iters=40),
    "er60_sketch": dict(sketch_rank=5, max_iters=40),
    "mixed40": dict(k_c=4, k_p=1, sketch_rank=4, max_iters=30),
    "qap4": dict(rho=0.005, k_c=4, k_p=0, sketch_rank=4, max_iters=20),
}


_BASELINE_CACHE: dict = {}


def baseline_cached(name, small=False):
    """instances.baseline_config, built once per test session (C4 and C5 take
    seconds to tens of seconds on the host)."""
    key = (name, small)
    if key not in _BASELINE_CACHE:
        _BASELINE_CACHE[key] = inst.baseline_config(name, small=small)
    return _BASELINE_CACHE[key]
