"""One K1 apply at k on C4 with each SpMM kernel (ncu target)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_11801_b200 import instances  # noqa: E402
from paper_2312_11801_b200.runtime import DeviceProblem, runtime  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 11
p = instances.baseline_config("C4").problem
rt = runtime()
dp = DeviceProblem(p, rt)
dp.assemble(rt.upload(np.random.default_rng(1234).standard_normal(p.m) * 1e-3))
V = rt.upload(np.linalg.qr(np.random.default_rng(k).standard_normal((p.n, k)))[0])
for env in ("1", "0"):
    os.environ["USBS_SPMM_V1"] = env
    Y = dp.apply(1, V)
    dp.apply(1, V, out=Y)
rt.sync()
print("ok")
