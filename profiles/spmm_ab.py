"""K1 at k = 1, 11, 20 on a config: the block-tiled SpMM vs the v1 warp-per-row
kernel (USBS_SPMM_V1=1); CUDA-event medians with L2 flushed, achieved GB/s of
B_apply(k) = 12 nnz + 4 (n+1) + 16 n k."""
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
for k in (11, 20):
    V = rt.upload(np.linalg.qr(np.random.default_rng(k).standard_normal((p.n, k)))[0])
    out = {}
    for tag, env in (("v1", "1"), ("tiles", "0")):
        os.environ["USBS_SPMM_L2"] = os.environ.get("L2", "1")
        os.environ["USBS_SPMM_V1"] = env
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
    d = np.abs(out["v1"][1] - out["tiles"][1]).max() / np.abs(out["v1"][1]).max()
    print(f"{name} k={k}: v1 {out['v1'][0]*1e3:.1f} us ({b/out['v1'][0]/1e6:.0f} GB/s)  tiles "
          f"{out['tiles'][0]*1e3:.1f} us ({b/out['tiles'][0]/1e6:.0f} GB/s)  max rel diff {d:.1e}", flush=True)
