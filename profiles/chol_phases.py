"""Per-panel cycle split of the d = 210 Newton-matrix Cholesky (chol_p16): panel-row
solve, warp 0's look-ahead chain, trailing update of warps 1 / 8 / 15.  Needs a library
built with -DUSBS_CHOL_PROF (USBS_LIB=...) and USBS_IPM_PROF=1.  Diagnostic."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import torch
from paper_2312_11801_b200 import subproblem
from paper_2312_11801_b200.runtime import runtime
rng = np.random.default_rng(11)
k = 20; d = k * (k + 1) // 2
a = rng.standard_normal((d + 5, d)); z = rng.standard_normal(d + 5)
class Q: pass
q = Q()
q.quad_ss, q.quad_s_eta, q.quad_eta = a.T @ a / (d + 5), a.T @ z / (d + 5), float(z @ z / (d + 5))
q.lin_s, q.lin_eta, q.has_eta, q.k = rng.standard_normal(d), float(rng.standard_normal()), True, k
rt = runtime()
r = subproblem.ipm_quad(q)
out = (C.c_uint64 * 128)()
rt.lib.usbs_ipm_profile(rt.h, out, 1)
n = 3
for _ in range(n): r = subproblem.ipm_quad(q)
rt.lib.usbs_ipm_profile(rt.h, out, 1)
nn = n * r.newton_iters
print("newton", r.newton_iters, "chol us/newton", out[4] / 1e3 / nn)
print("panel  solve  w0chain  w1trail  w8trail  w15trail (cycles)")
for pn in range(14):
    print(pn, *[f"{out[16 + 16 * g + pn] / nn:8.0f}" for g in range(5)])
