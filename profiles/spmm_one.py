"""One K1 apply Z V at k (default 11) on a config with the default SpMM
kernel (ncu target: k_spmm_g at C4)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_11801_b200 import instances  # noqa: E402
from paper_2312_11801_b200.runtime import DeviceProblem, runtime  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 11
name = sys.argv[2] if len(sys.argv) > 2 else "C4"
p = instances.baseline_config(name).problem
rt = runtime()
dp = DeviceProblem(p, rt)
dp.assemble(rt.upload(np.random.default_rng(1234).standard_normal(p.m) * 1e-3))
V = rt.upload(np.linalg.qr(np.random.default_rng(k).standard_normal((p.n, k)))[0])
Y = dp.apply(1, V)
dp.apply(1, V, out=Y)
rt.sync()
print("ok")
