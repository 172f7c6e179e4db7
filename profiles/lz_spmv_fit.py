"""Per-block SpMV time of the TMA grid Lanczos vs the composition of the
block's work items (nonzeros, rows, long rows, items, pieces), least-squares
fit of the plan's cost model (usbs_lanczos_grid.cu lz_tma_plan)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_11801_b200 import eigen, instances  # noqa: E402
from paper_2312_11801_b200.runtime import DeviceProblem, runtime  # noqa: E402

SEG, SEGROWS, SHORT = 512, 64, 32


def items(rp):
    n = len(rp) - 1
    out = []  # (nnz, rows, long, piece)
    i = 0
    nz = np.diff(rp)
    while i < n:
        z = nz[i]
        if z > SEG:
            for q in range(rp[i], rp[i + 1], SEG):
                out.append((min(SEG, rp[i + 1] - q), 0, 0, 1))
            i += 1
        else:
            a0, nl = i, 0
            while i < n and i - a0 < SEGROWS and nz[i] <= SEG and rp[i + 1] - rp[a0] <= SEG:
                nl += nz[i] > SHORT
                i += 1
            out.append((rp[i] - rp[a0], i - a0, nl, 0))
    return np.array(out, dtype=float)


def plan(it, G, row_cost, item_cost, long_cost):
    cost = it[:, 0] + row_cost * it[:, 1] + long_cost * it[:, 2] + item_cost
    tot = cost.sum()
    acc = np.cumsum(cost)
    bounds = [0]
    for b in range(1, G):
        bounds.append(int(np.searchsorted(acc, tot * b / G, side="left")) + 1)
    bounds.append(len(it))
    return bounds


name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = instances.baseline_config(name)
p = cfg.problem
rt = runtime()
dp = DeviceProblem(p, rt)
y = np.random.default_rng(1234).standard_normal(p.m) * 1e-3
op = eigen.dual_slack_operator(dp, y)
import scipy.sparse as sp  # noqa: E402
z = (p.cost + sp.identity(p.n, format="csr")).tocsr()
z.sort_indices()
it = items(z.indptr.astype(np.int64))
G = 144
os.environ["USBS_LZ_PROF"] = "1"
buf = (C.c_ulonglong * 1024)()
r = eigen.lanczos_top(op, cfg.k_c, seed=0)
rt.lib.usbs_lanczos_profile(rt.h, buf, 1)
r = eigen.lanczos_top(op, cfg.k_c, seed=0)
rt.lib.usbs_lanczos_profile(rt.h, buf, 1)
spmv = np.array([buf[32 + 5 * b] for b in range(G)], dtype=float) / 1e3 / r.matvecs
bounds = plan(it, G, float(os.environ.get("USBS_LZG_ROWCOST", 2)), float(os.environ.get("USBS_LZG_ITEMCOST", 256)),
              float(os.environ.get("USBS_LZG_LONGCOST", 64)))
X = np.array([it[bounds[b]:bounds[b + 1]].sum(0).tolist() + [bounds[b + 1] - bounds[b]] for b in range(G)])
print("blocks: spmv us mean %.1f max %.1f min %.1f" % (spmv.mean(), spmv.max(), spmv.min()))
print("features: nnz, rows, long rows, pieces, items")
A = np.column_stack([X, np.ones(G)])
coef, *_ = np.linalg.lstsq(A, spmv, rcond=None)
print("fit us per unit:", np.round(coef, 6).tolist())
print("fit relative to nnz:", np.round(coef / coef[0], 2).tolist())
print("residual rms %.2f us" % np.sqrt(np.mean((A @ coef - spmv) ** 2)))
for b in list(np.argsort(-spmv)[:6]) + list(np.argsort(spmv)[:3]):
    print(b, "%.1f us" % spmv[b], X[b].astype(int).tolist())
