"""A few d = 210 IPM solves (k = 20, random SPD quadratic as in
prof_kernels ipm) -- ncu target for k_ipm."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_11801_b200 import subproblem  # noqa: E402

rng = np.random.default_rng(0)
k = int(sys.argv[1]) if len(sys.argv) > 1 else 20
d = k * (k + 1) // 2


class Q:
    pass


q = Q()
a = rng.standard_normal((d + 5, d))
z = rng.standard_normal(d + 5)
q.quad_ss, q.quad_s_eta, q.quad_eta = a.T @ a / (d + 5), a.T @ z / (d + 5), float(z @ z / (d + 5))
q.lin_s, q.lin_eta, q.has_eta, q.k = rng.standard_normal(d), float(rng.standard_normal()), True, k
for _ in range(2):
    r = subproblem.ipm_quad(q)
print("ipm", d, r.value, r.newton_iters)
