"""One K4 compressed Gram (d x d) on a config (ncu target)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_11801_b200 import instances  # noqa: E402
from paper_2312_11801_b200.engine import Engine  # noqa: E402
from paper_2312_11801_b200.runtime import DeviceProblem, runtime  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
bc = instances.baseline_config(name)
rt = runtime()
dp = DeviceProblem(bc.problem, rt)
eng = Engine(dp)
k = bc.k_c + bc.k_p
V = rt.upload(np.linalg.qr(np.random.default_rng(1234).standard_normal((bc.problem.n, k)))[0])
G = rt.empty(k * (k + 1) // 2, k * (k + 1) // 2)
for _ in range(2):
    eng.compressed(V, scale_gram=1.0, gram_out=G)
rt.sync()
print("ok")
