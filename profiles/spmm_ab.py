"""K1 on a config, CUDA-event medians with L2 flushed, achieved GB/s of
B_apply(k) = 12 nnz + 4 (n+1) + 16 n k, for each SpMM variant:
  g      grouped 16-byte-gather kernel (k <= 15, default)
  16x2   half-warp-per-nonzero kernel (USBS_SPMM_16X2=1)
  tiles  block CSR-stream kernel (USBS_SPMM_V1=0)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11801_b200 import instances  # noqa: E402
from paper_2312_11801_b200.runtime import DeviceProblem, runtime  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
p = instances.baseline_config(name).problem
rt = runtime()
dp = DeviceProblem(p, rt)
nnz = dp.info().nnz_z
y = np.random.default_rng(1234).standard_normal(p.m) * 1e-3
dp.assemble(rt.upload(y))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=rt.device)
VARIANTS = {"g": {}, "16x2": {"USBS_SPMM_16X2": "1"}, "tiles": {"USBS_SPMM_V1": "0"}}
for k in (2, 5, 11, 15, 20):
    V = rt.upload(np.linalg.qr(np.random.default_rng(k).standard_normal((p.n, k)))[0])
    out = {}
    for tag, env in VARIANTS.items():
        for key in ("USBS_SPMM_16X2", "USBS_SPMM_V1"):
            os.environ.pop(key, None)
        os.environ.update(env)
        Y = dp.apply(1, V)
        ts = []
        for _ in range(7):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(rt.stream)
            dp.apply(1, V, out=Y)
            e1.record(rt.stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[tag] = (float(np.median(ts)), Y.cpu().numpy())
    b = 12 * nnz + 4 * (p.n + 1) + 16 * p.n * k
    ref = out["16x2"][1]
    line = "  ".join(f"{t} {ms*1e3:.1f} us ({b/ms/1e6:.0f} GB/s, diff {np.abs(y_ - ref).max() / np.abs(ref).max():.0e})"
                     for t, (ms, y_) in out.items())
    print(f"{name} k={k}: {line}", flush=True)
