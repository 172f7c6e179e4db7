"""A few constraint-image evaluations A(V S V^T) at a config (ncu target)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_11801_b200 import instances  # noqa: E402
from paper_2312_11801_b200.engine import Engine  # noqa: E402
from paper_2312_11801_b200.runtime import DeviceProblem, runtime  # noqa: E402

bc = instances.baseline_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
rt = runtime()
dp = DeviceProblem(bc.problem, rt)
eng = Engine(dp)
k = bc.k_c + bc.k_p
rng = np.random.default_rng(3)
V = rt.upload(np.linalg.qr(rng.standard_normal((bc.problem.n, k)))[0])
a = rng.standard_normal((k, k))
S = rt.upload(a @ a.T)
out = rt.empty(bc.problem.m)
for _ in range(3):
    eng.image(V, S, out)
rt.sync()
print("ok")
