"""A/B of the TMA Lanczos switches on one config: SpMV tail pool share
(USBS_LZG_TAIL) and USBS_LZG_OPT bits (1: column sums from shared memory).
Measured and dropped this round: a shared-memory copy of x's 8192 leading
(highest-degree) entries in the free slots during the SpMV -- 8.71 vs
8.65 ms per C4 call (the hub lines already hit L1)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11801_b200 import eigen, instances, runtime as R  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = instances.baseline_config(name)
p = cfg.problem
rt = R.runtime()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=rt.device)
y = np.random.default_rng(1234).standard_normal(p.m) * 1e-3
buf = (C.c_ulonglong * 1024)()
for tail in sys.argv[2].split(",") if len(sys.argv) > 2 else ("0",):
    for opt in sys.argv[3].split(",") if len(sys.argv) > 3 else ("0", "1"):
        os.environ["USBS_LZG_TAIL"], os.environ["USBS_LZG_OPT"] = tail, opt
        os.environ.pop("USBS_LZ_PROF", None)
        dp = R.DeviceProblem(p, rt)  # fresh plan for the tail share
        op = eigen.dual_slack_operator(dp, y)
        r = eigen.lanczos_top(op, cfg.k_c, seed=0)
        ts = []
        for _ in range(3):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(rt.stream)
            r = eigen.lanczos_top(op, cfg.k_c, seed=0)
            e1.record(rt.stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        os.environ["USBS_LZ_PROF"] = "1"
        rt.lib.usbs_lanczos_profile(rt.h, buf, 1)
        eigen.lanczos_top(op, cfg.k_c, seed=0)
        rt.lib.usbs_lanczos_profile(rt.h, buf, 1)
        bw = np.array([[buf[32 + 5 * b + s] for s in range(5)] for b in range(144)], dtype=float) / 1e3 / r.matvecs
        print(f"tail {tail} opt {opt}: {np.median(ts):.3f} ms mv {r.matvecs} lam0 {r.eigenvalues[0]:.15f} mean "
              f"{np.round(bw.mean(0), 1).tolist()} max {np.round(bw.max(0), 1).tolist()}", flush=True)
        del dp
