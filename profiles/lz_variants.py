"""Time the TMA grid Lanczos kernel variants (USBS_LZG_VARIANT) on one config."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11801_b200 import eigen, instances  # noqa: E402
from paper_2312_11801_b200.runtime import DeviceProblem, runtime  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
variants = [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else "0,1,2,3,4".split(","))]
cfg = instances.baseline_config(name)
p = cfg.problem
rt = runtime()
dp = DeviceProblem(p, rt)
y = np.random.default_rng(1234).standard_normal(p.m) * 1e-3
if dp.has_ineq:
    y[dp.ineq_idx] = -np.abs(y[dp.ineq_idx])
dp.assemble(rt.upload(y))
op = eigen.dual_slack_operator(dp, y)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=rt.device)
import ctypes as C  # noqa: E402
buf = (C.c_ulonglong * 1024)()
for v in variants:
    os.environ["USBS_LZG_VARIANT"] = str(v)
    os.environ.pop("USBS_LZ_PROF", None)
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
    G = 144
    bw = np.array([[buf[32 + 5 * b + s] for s in range(5)] for b in range(G)], dtype=float) / 1e3 / r.matvecs
    print(f"variant {v}: {np.median(ts):.3f} ms matvecs {r.matvecs} lam0 {r.eigenvalues[0]:.15f} | per-block mean "
          f"{np.round(bw.mean(0), 1).tolist()} max {np.round(bw.max(0), 1).tolist()} | rr {buf[5]/1e3/r.matvecs:.1f} "
          f"restart {buf[6]/1e3/r.matvecs:.1f} us/step", flush=True)
