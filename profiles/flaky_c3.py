"""Repeat the full-size C3 Lanczos of test_gpu_fullscale, interleaved with
C4/C5 operator applies and Lanczos calls, to reproduce an intermittent
non-finite matvec."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import usbs_cpu as O  # noqa: E402
from paper_2312_11801_b200 import eigen, instances, runtime  # noqa: E402

probs = {n: instances.baseline_config(n).problem for n in ("C3", "C4", "C5")}
bad = 0
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    for name in ("C4", "C5", "C3"):
        p = probs[name]
        y = np.random.default_rng(1234).standard_normal(p.m) * 1e-3
        if p.ineq_mask.any():
            y[p.ineq_mask] = np.abs(y[p.ineq_mask])
        dp = runtime.DeviceProblem(p)
        v = np.linalg.qr(np.random.default_rng(20).standard_normal((p.n, 20)))[0]
        dp.assemble(dp.rt.upload(y))
        dp.apply(1, dp.rt.upload(v))
        try:
            r = eigen.lanczos_top(eigen.dual_slack_operator(dp, y), 20 if name != "C4" else 10, seed=0)
            print(rep, name, "ok", r.matvecs, r.eigenvalues[0], flush=True)
        except Exception as e:
            bad += 1
            print(rep, name, "FAIL", type(e).__name__, e, flush=True)
        del dp
print("failures", bad)
