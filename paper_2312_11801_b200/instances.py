"""Host-side problem construction (not on the device path).

The reference builds its scaled SDP data with numpy/scipy on the host and the
GPU path consumes exactly those arrays, so "graph and CSR construction are
bit-exact" holds by construction.  This module restates the reference
builders (same floating-point operations in the same order) so that the
framework does not need the reference package at run time, and adds the
seeded BASELINE workload generators C1..C5.

Reference anchors (paths relative to /root/reference):
  * ``Graph``            ~ pkg/src/specbundle/problem.py:57-108 (GraphInstance)
  * ``Qap``              ~ problem.py:111-137 (QapInstance)
  * ``DiagonalFamily``   ~ problem.py:144-176 (DiagonalConstraints; data only)
  * ``EntryFamilies``    ~ problem.py:179-243 (SparseConstraintFamilies; data only)
  * ``Problem``          ~ problem.py:250-289 (SdpProblem; data only)
  * ``maxcut_problem``   ~ problem.py:325-349 (build_maxcut)
  * ``qap_problem``      ~ problem.py:364-506 (qap_constraint_entries, build_qap)
  * ``family_problem``   ~ problem.py:509-539 (build_from_families)
Bit-exactness against the reference is pinned by tests/test_instances_golden.py
(golden hashes written by oracle/make_golden.py from the reference itself).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import scipy.sparse as sp

__all__ = [
    "Graph",
    "Qap",
    "DiagonalFamily",
    "EntryFamilies",
    "Problem",
    "maxcut_problem",
    "qap_problem",
    "family_problem",
    "erdos_renyi",
    "torus_pm1",
    "qap_random",
    "chung_lu",
    "knn_correlation",
    "baseline_config",
]


# ---------------------------------------------------------------------------
# graphs


@dataclass
class Graph:
    """Undirected weighted simple graph stored as sorted (u < v) edge arrays."""

    n: int
    eu: np.ndarray
    ev: np.ndarray
    ew: np.ndarray

    @classmethod
    def from_edge_list(cls, n: int, edges) -> "Graph":
        """Duplicates summed in input order, self loops dropped, keys sorted
        (problem.py:67-87).  Vectorised: bincount accumulates weights in the
        order they appear, which reproduces the dict accumulation bit for bit."""
        if n < 1:
            raise ValueError("graph needs at least one vertex")
        arr = list(edges)
        if not arr:
            z = np.zeros(0, dtype=np.int64)
            return cls(n, z, z.copy(), np.zeros(0))
        u = np.array([int(e[0]) for e in arr], dtype=np.int64)
        v = np.array([int(e[1]) for e in arr], dtype=np.int64)
        w = np.array([float(e[2]) for e in arr], dtype=float)
        return cls.from_arrays(n, u, v, w)

    @classmethod
    def from_arrays(cls, n: int, u, v, w) -> "Graph":
        u = np.asarray(u, dtype=np.int64)
        v = np.asarray(v, dtype=np.int64)
        w = np.asarray(w, dtype=float)
        keep = u != v
        u, v, w = u[keep], v[keep], w[keep]
        lo = np.minimum(u, v)
        hi = np.maximum(u, v)
        if lo.size and (lo.min() < 0 or hi.max() >= n):
            raise ValueError(f"edge out of range for n={n}")
        key = lo * n + hi
        uniq, inv = np.unique(key, return_inverse=True)
        acc = np.bincount(inv, weights=w, minlength=uniq.size) if uniq.size else np.zeros(0)
        return cls(n, (uniq // n).astype(np.int64), (uniq % n).astype(np.int64), acc.astype(float))

    @property
    def num_edges(self) -> int:
        return int(self.ew.size)

    def subgraph(self, keep: int) -> "Graph":
        """Induced subgraph on vertices 0 .. keep-1 (problem.py:104-108)."""
        sel = (self.eu < keep) & (self.ev < keep)
        return Graph.from_arrays(keep, self.eu[sel], self.ev[sel], self.ew[sel])

    def laplacian(self) -> sp.csr_matrix:
        # COO assembly order matches problem.py:93-102 so duplicate summation
        # inside tocsr() rounds identically
        n = self.n
        deg = np.zeros(n)
        np.add.at(deg, self.eu, self.ew)
        np.add.at(deg, self.ev, self.ew)
        diag = np.arange(n)
        r = np.concatenate([self.eu, self.ev, diag])
        c = np.concatenate([self.ev, self.eu, diag])
        d = np.concatenate([-self.ew, -self.ew, deg])
        return sp.coo_matrix((d, (r, c)), shape=(n, n)).tocsr()


@dataclass
class Qap:
    weights: np.ndarray
    distances: np.ndarray

    def __post_init__(self):
        w = np.asarray(self.weights, dtype=float)
        d = np.asarray(self.distances, dtype=float)
        if w.shape != d.shape or w.ndim != 2 or w.shape[0] != w.shape[1]:
            raise ValueError("weight and distance matrices must be square and the same size")
        for name, a in (("weight", w), ("distance", d)):
            if not np.allclose(a, a.T, atol=1e-12 * (1 + np.abs(a).max(initial=0.0))):
                raise ValueError(f"{name} matrix must be symmetric")
        self.weights, self.distances = w, d

    @property
    def size(self) -> int:
        return self.weights.shape[0]

    def shrink(self) -> "Qap":
        """The instance without its last facility/location (problem.py:131-133)."""
        return Qap(self.weights[:-1, :-1].copy(), self.distances[:-1, :-1].copy())


def qap_labels(q: Qap) -> list:
    """Labels of the lifted assignment constraints in builder order
    (problem.py:392-426): ("tr1", k, l), ("tr2", i, j), ("G", a, b),
    ("diagY", a), ("rowsum", k), ("colsum", i), ("B", a), ("corner",),
    ("trY",); used to map constraints between instance sizes."""
    l = q.size
    out = [("tr1", k, kk) for k in range(l) for kk in range(k, l)]
    out += [("tr2", i, j) for i in range(l) for j in range(i, l)]
    ka, kb = np.nonzero(np.kron(q.distances, q.weights))
    out += [("G", int(a), int(b)) for a, b in zip(ka, kb)]
    out += [("diagY", a) for a in range(l * l)]
    out += [("rowsum", k) for k in range(l)] + [("colsum", i) for i in range(l)]
    out += [("B", a) for a in range(l * l)] + [("corner",), ("trY",)]
    return out


# ---------------------------------------------------------------------------
# constraint data (device operators live in operators.py)


class DiagonalFamily:
    """A_i = e_i e_i^T (problem.py:144-176).  Pure data marker."""

    kind = "diag"

    def __init__(self, n: int):
        self.n = int(n)
        self.m = int(n)

    def frob_norms(self) -> np.ndarray:
        return np.ones(self.m)


class EntryFamilies:
    """Flat entry list: constraint idx[e] has A[rows[e], cols[e]] =
    A[cols[e], rows[e]] = vals[e], rows <= cols (problem.py:179-198)."""

    kind = "entries"

    def __init__(self, n, m, idx, rows, cols, vals):
        self.n, self.m = int(n), int(m)
        self.idx = np.asarray(idx, dtype=np.int64)
        self.rows = np.asarray(rows, dtype=np.int64)
        self.cols = np.asarray(cols, dtype=np.int64)
        self.vals = np.asarray(vals, dtype=float)
        if np.any(self.rows > self.cols):
            raise ValueError("entries must have rows <= cols")
        self._diag = self.rows == self.cols
        self._eff = np.where(self._diag, 1.0, 2.0) * self.vals

    def scaled(self, factors) -> "EntryFamilies":
        return EntryFamilies(self.n, self.m, self.idx, self.rows, self.cols,
                             self.vals * np.asarray(factors)[self.idx])

    def frob_norms(self) -> np.ndarray:
        sq = self.vals ** 2 * np.where(self._diag, 1.0, 2.0)
        return np.sqrt(np.bincount(self.idx, weights=sq, minlength=self.m))

    # host-side helpers used only by the operator-norm estimate at build time
    def _image_dense(self, x):
        return np.bincount(self.idx, weights=x[self.rows, self.cols] * self._eff, minlength=self.m)

    def _adjoint_dense(self, y):
        data = y[self.idx] * self.vals
        off = ~self._diag
        r = np.concatenate([self.rows, self.cols[off]])
        c = np.concatenate([self.cols, self.rows[off]])
        d = np.concatenate([data, data[off]])
        return sp.coo_matrix((d, (r, c)), shape=(self.n, self.n)).tocsr()


@dataclass
class Problem:
    """Scaled SDP data: maximise <cost, X> s.t. A X (<=|=) b, X psd,
    tr X <= alpha (problem.py:250-289).  Duck-compatible with the
    reference ``SdpProblem`` fields the solver reads."""

    n: int
    m: int
    cost: sp.csr_matrix
    constraints: object
    b: np.ndarray
    ineq_mask: np.ndarray
    alpha: float
    scale_c: float
    scale_x: float
    sense: int = 1
    labels: Optional[list] = None
    op_norm_estimate: Optional[float] = None
    kron_factors: Optional[tuple] = None  # (D, W): cost = -(0 (+) D (x) W) / scale_c (QAP)

    def __post_init__(self):
        self.b = np.asarray(self.b, dtype=float)
        self.ineq_mask = np.asarray(self.ineq_mask, dtype=bool)
        self._ineq_idx = np.flatnonzero(self.ineq_mask)

    @property
    def ineq_idx(self) -> np.ndarray:
        return self._ineq_idx

    @property
    def has_ineq(self) -> bool:
        return self._ineq_idx.size > 0

    def unscale_objective(self, v: float) -> float:
        return self.sense * v * self.scale_c * self.scale_x


def _frob(a) -> float:
    return float(np.sqrt((a.multiply(a)).sum()))


def maxcut_problem(g: Graph, alpha: float = 2.0, with_labels: bool = False) -> Problem:
    """build_maxcut (problem.py:325-349): C = L/4 / ||L/4||_F, b = 1/n."""
    if g.n < 1:
        raise ValueError("empty graph")
    n = g.n
    c_raw = (g.laplacian() / 4.0).tocsr()
    scale_c = _frob(c_raw) or 1.0
    cost = (c_raw / scale_c).tocsr()
    scale_x = float(n)
    return Problem(n=n, m=n, cost=cost, constraints=DiagonalFamily(n),
                   b=np.full(n, 1.0 / scale_x), ineq_mask=np.zeros(n, dtype=bool),
                   alpha=alpha, scale_c=scale_c, scale_x=scale_x, sense=1,
                   labels=[("diag", i) for i in range(n)] if with_labels else None)


def _qap_families(q: Qap):
    """Entry families of the lifted assignment relaxation, in the order of
    problem.py:392-426 (tr1, tr2, G, diagY, rowsum, colsum, B, corner, trY)."""
    l = q.size
    kron = np.kron(q.distances, q.weights)
    idx, rows, cols, vals, rhs, ineq = [], [], [], [], [], []

    def push(ent, b, is_ineq):
        ci = len(rhs)
        for r, c, v in ent:
            if r > c:
                r, c = c, r
            idx.append(ci); rows.append(r); cols.append(c); vals.append(v)
        rhs.append(b); ineq.append(is_ineq)

    for k in range(l):
        for kk in range(k, l):
            push([(1 + i * l + k, 1 + i * l + kk, 1.0 if k == kk else 0.5) for i in range(l)],
                 1.0 if k == kk else 0.0, False)
    for i in range(l):
        for j in range(i, l):
            push([(1 + i * l + k, 1 + j * l + k, 1.0 if i == j else 0.5) for k in range(l)],
                 1.0 if i == j else 0.0, False)
    ka, kb = np.nonzero(kron)
    for a, bb in zip(ka.tolist(), kb.tolist()):
        push([(1 + a, 1 + bb, -1.0 if a == bb else -0.5)], 0.0, True)
    for a in range(l * l):
        push([(1 + a, 1 + a, 1.0), (0, 1 + a, -0.5)], 0.0, False)
    for k in range(l):
        push([(0, 1 + i * l + k, 0.5) for i in range(l)], 1.0, False)
    for i in range(l):
        push([(0, 1 + i * l + k, 0.5) for k in range(l)], 1.0, False)
    for a in range(l * l):
        push([(0, 1 + a, -0.5)], 0.0, True)
    push([(0, 0, 1.0)], 1.0, False)
    push([(1 + a, 1 + a, 1.0) for a in range(l * l)], float(l), False)
    return (np.array(idx), np.array(rows), np.array(cols), np.array(vals, dtype=float),
            np.array(rhs, dtype=float), np.array(ineq, dtype=bool), kron)


def _power_norm(ops: EntryFamilies, n: int, tol=1e-6, max_iters=500, seed=0) -> float:
    """Operator-norm estimate by power iteration on A*A over symmetric
    matrices (problem.py:440-459); legacy MT19937 start."""
    x = np.random.RandomState(seed).standard_normal((n, n))
    x = 0.5 * (x + x.T)
    x /= np.linalg.norm(x)
    prev = 0.0
    lam = 0.0
    for _ in range(max_iters):
        yv = np.asarray(ops._adjoint_dense(ops._image_dense(x)).todense(), dtype=float)
        lam = float(np.linalg.norm(yv))
        if lam == 0.0:
            return 0.0
        x = yv / lam
        if abs(lam - prev) <= tol * lam:
            break
        prev = lam
    return float(np.sqrt(lam))


def qap_problem(q: Qap, alpha: float = 2.0) -> Problem:
    """build_qap (problem.py:462-506)."""
    l = q.size
    big = l * l + 1
    idx, rows, cols, vals, b_raw, ineq, kron = _qap_families(q)
    m = len(b_raw)
    ka, kb = np.nonzero(kron)
    c_raw = sp.coo_matrix((-kron[ka, kb], (1 + ka, 1 + kb)), shape=(big, big)).tocsr()
    scale_c = _frob(c_raw) or 1.0
    cost = (c_raw / scale_c).tocsr()
    scale_x = float(l + 1)
    b = b_raw / scale_x
    ops = EntryFamilies(big, m, idx, rows, cols, vals)
    norms = ops.frob_norms()
    if np.any(norms == 0):
        raise ValueError("degenerate constraint with zero norm")
    ops = ops.scaled(1.0 / norms)
    b = b / norms
    op_norm = _power_norm(ops, big)
    if op_norm > 0:
        ops = ops.scaled(np.full(m, 1.0 / op_norm))
        b = b / op_norm
    return Problem(n=big, m=m, cost=cost, constraints=ops, b=b, ineq_mask=ineq, alpha=alpha,
                   scale_c=scale_c, scale_x=scale_x, sense=-1, op_norm_estimate=op_norm,
                   kron_factors=(np.asarray(q.distances, dtype=float), np.asarray(q.weights, dtype=float)))


def family_problem(n, cost_raw, triples, b_raw, ineq_mask, alpha=2.0, scale_x=1.0) -> Problem:
    """build_from_families (problem.py:509-539)."""
    cost_raw = sp.csr_matrix(cost_raw)
    scale_c = _frob(cost_raw) or 1.0
    idx, rows, cols, vals = (np.asarray(a) for a in triples)
    m = len(b_raw)
    return Problem(n=n, m=m, cost=(cost_raw / scale_c).tocsr(),
                   constraints=EntryFamilies(n, m, idx, rows, cols, vals),
                   b=np.asarray(b_raw, dtype=float) / scale_x,
                   ineq_mask=np.asarray(ineq_mask, dtype=bool), alpha=alpha,
                   scale_c=scale_c, scale_x=scale_x, sense=1)


# ---------------------------------------------------------------------------
# seeded BASELINE generators


def erdos_renyi(n: int, p: float, seed: int) -> Graph:
    """pkg/tests/conftest.py:25-30: PCG64 default_rng(seed), one rng.random()
    per pair i<j in lexicographic order.  A single vectorised draw consumes
    the identical stream."""
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, 1)
    hit = rng.random(iu.size) < p
    if not hit.any():
        return Graph.from_arrays(n, [0], [1], [1.0])
    return Graph.from_arrays(n, iu[hit], ju[hit], np.ones(int(hit.sum())))


def torus_pm1(side: int = 100, seed: int = 1) -> Graph:
    """C2: side x side torus, vertex v = side*i + j; edges (v, down), (v, right)
    in (i, j) order; weight +1 if default_rng(seed).random(E)[e] < 0.5 else -1."""
    i, j = np.meshgrid(np.arange(side), np.arange(side), indexing="ij")
    i, j = i.ravel(), j.ravel()
    v = side * i + j
    down = side * ((i + 1) % side) + j
    right = side * i + (j + 1) % side
    u = np.stack([v, v], axis=1).ravel()
    w_to = np.stack([down, right], axis=1).ravel()
    r = np.random.default_rng(seed).random(u.size)
    wts = np.where(r < 0.5, 1.0, -1.0)
    return Graph.from_arrays(side * side, u, w_to, wts)


def qap_random(l: int = 20, seed: int = 2, hi: int = 11) -> Qap:
    """C3: W then D, each triu(integers(0, hi, (l,l)), 1) mirrored, one rng."""
    rng = np.random.default_rng(seed)
    mats = []
    for _ in range(2):
        a = np.triu(rng.integers(0, hi, (l, l)), 1).astype(float)
        mats.append(a + a.T)
    return Qap(mats[0], mats[1])


def chung_lu(n: int = 1_000_000, gamma: float = 2.5, mean_deg: float = 8.0, seed: int = 3) -> Graph:
    """C4: w_i = (i+1)^(-1/(gamma-1)) rescaled to mean ``mean_deg``;
    M = round(sum(w)/2) endpoint pairs drawn u then v from p = w/sum(w);
    self loops dropped, unordered duplicates removed (unit weights)."""
    w = np.arange(1, n + 1, dtype=float) ** (-1.0 / (gamma - 1.0))
    w *= mean_deg / w.mean()
    total = w.sum()
    mcount = int(round(total / 2.0))
    rng = np.random.default_rng(seed)
    p = w / total
    u = rng.choice(n, mcount, p=p)
    v = rng.choice(n, mcount, p=p)
    keep = u != v
    lo = np.minimum(u[keep], v[keep]).astype(np.int64)
    hi = np.maximum(u[keep], v[keep]).astype(np.int64)
    key = np.unique(lo * n + hi)
    return Graph(n, key // n, key % n, np.ones(key.size))


def knn_correlation(n: int = 63_000, clusters: int = 2000, dim: int = 64, knn: int = 32,
                    sigma: float = 0.3, zipf_s: float = 1.1, seed: int = 4):
    """C5 instance: Zipf cluster sizes (largest-remainder rounding, min 1),
    unit-norm Gaussian centres in ``dim`` dims, points = centre + sigma*N(0, I),
    exact cosine ``knn``-NN graph symmetrised by union, weights cos - 0.5.
    Returns (n, eu, ev, ew) with eu < ev sorted."""
    rng = np.random.default_rng(seed)
    raw = np.arange(1, clusters + 1, dtype=float) ** (-zipf_s)
    share = raw / raw.sum() * n
    size = np.maximum(np.floor(share).astype(np.int64), 1)
    short = n - int(size.sum())
    if short > 0:
        order = np.argsort(-(share - np.floor(share)), kind="stable")
        size[order[:short]] += 1
    elif short < 0:
        order = np.argsort(-size, kind="stable")
        t = 0
        while short < 0:
            c = order[t % clusters]
            if size[c] > 1:
                size[c] -= 1
                short += 1
            t += 1
    centres = rng.standard_normal((clusters, dim))
    centres /= np.linalg.norm(centres, axis=1, keepdims=True)
    lab = np.repeat(np.arange(clusters), size)
    pts = centres[lab] + sigma * rng.standard_normal((n, dim))
    pts /= np.linalg.norm(pts, axis=1, keepdims=True)
    nbr = np.empty((n, knn), dtype=np.int64)
    blk = 2048
    for s in range(0, n, blk):
        e = min(n, s + blk)
        sim = pts[s:e] @ pts.T
        sim[np.arange(e - s), np.arange(s, e)] = -np.inf
        part = np.argpartition(-sim, knn, axis=1)[:, :knn]
        nbr[s:e] = part
    src = np.repeat(np.arange(n, dtype=np.int64), knn)
    dst = nbr.ravel()
    lo = np.minimum(src, dst)
    hi = np.maximum(src, dst)
    key = np.unique(lo * n + hi)
    eu, ev = key // n, key % n
    ew = np.einsum("ij,ij->i", pts[eu], pts[ev]) - 0.5
    return n, eu, ev, ew


def correlation_problem(n, eu, ev, ew) -> Problem:
    """C5 problem via build_from_families: cost W (w_ij on kNN edges),
    diag(X) = 1 equalities, X_ij >= 0 on edges as -0.5 X_ij <= 0 rows."""
    cost = sp.coo_matrix((np.concatenate([ew, ew]), (np.concatenate([eu, ev]),
                                                      np.concatenate([ev, eu]))),
                         shape=(n, n)).tocsr()
    ne = eu.size
    diag = np.arange(n, dtype=np.int64)
    idx = np.concatenate([diag, n + np.arange(ne, dtype=np.int64)])
    rows = np.concatenate([diag, eu])
    cols = np.concatenate([diag, ev])
    vals = np.concatenate([np.ones(n), np.full(ne, -0.5)])
    b = np.concatenate([np.ones(n), np.zeros(ne)])
    ineq = np.concatenate([np.zeros(n, dtype=bool), np.ones(ne, dtype=bool)])
    return family_problem(n, cost, (idx, rows, cols, vals), b, ineq, scale_x=float(n))


@dataclass
class BaselineConfig:
    """One BASELINE.json config: the problem and the solver settings
    (SURVEY.md 7 item 11, 8d)."""

    name: str
    problem: Problem
    rho: float
    beta: float
    k_c: int
    k_p: int
    sketch_rank: int
    eps: float = 1e-3
    seed: int = 0
    extra: dict = field(default_factory=dict)


def baseline_config(name: str, small: bool = False) -> BaselineConfig:
    """Build C1..C5.  ``small`` shrinks C4/C5 for quick tests."""
    name = name.upper()
    if name == "C1":
        return BaselineConfig("C1", maxcut_problem(erdos_renyi(800, 0.06, 0)), 0.01, 0.25, 10, 1, 0)
    if name == "C2":
        return BaselineConfig("C2", maxcut_problem(torus_pm1(100, 1)), 0.01, 0.25, 10, 1, 10)
    if name == "C3":
        return BaselineConfig("C3", qap_problem(qap_random(20, 2)), 0.005, 0.25, 20, 0, 20)
    if name == "C4":
        n = 20_000 if small else 1_000_000
        return BaselineConfig("C4", maxcut_problem(chung_lu(n, seed=3)), 0.01, 0.25, 10, 1, 10)
    if name == "C5":
        if small:
            inst = knn_correlation(n=3000, clusters=100, seed=4)
        else:
            inst = knn_correlation(seed=4)
        return BaselineConfig("C5", correlation_problem(*inst), 0.01, 0.25, 20, 0, 20)
    raise ValueError(f"unknown config {name}")
