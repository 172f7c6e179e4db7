"""One warm-up and one measured lanczos_top on a config (the ncu target)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_11801_b200 import eigen, instances  # noqa: E402
from paper_2312_11801_b200.runtime import DeviceProblem, runtime  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = instances.baseline_config(name)
p = cfg.problem
rt = runtime()
dp = DeviceProblem(p, rt)
y = np.random.default_rng(1234).standard_normal(p.m) * 1e-3
if dp.has_ineq:
    y[dp.ineq_idx] = np.abs(y[dp.ineq_idx])
op = eigen.dual_slack_operator(dp, y)
for _ in range(2):
    r = eigen.lanczos_top(op, cfg.k_c, seed=0)
rt.sync()
print(name, "matvecs", r.matvecs, "restarts", r.restarts, "lam0", r.eigenvalues[0])
