"""usbs_rowgemm at n = 10^6: the row-per-thread kernel (default) vs the
entry-per-thread kernel (USBS_ROWGEMM_V1=1); CUDA-event medians, L2 flushed,
bytes = 8 n (ka + kb) (+ 8 n kb with Y0)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11801_b200 import instances  # noqa: E402
from paper_2312_11801_b200.engine import Engine  # noqa: E402
from paper_2312_11801_b200.runtime import DeviceProblem, runtime  # noqa: E402

rt = runtime()
dp = DeviceProblem(instances.maxcut_problem(instances.erdos_renyi(200, 0.1, 1)), rt)
eng = Engine(dp)
n = 1_000_000
flush = torch.empty(256 << 20, dtype=torch.uint8, device=rt.device)
rng = np.random.default_rng(0)
for ka, kb, y0 in ((11, 11, False), (11, 10, True), (1, 1, False), (33, 11, False), (20, 20, False)):
    X = rt.upload(rng.standard_normal((n, ka)))
    B = rt.upload(rng.standard_normal((ka, kb)))
    Y = rt.empty(n, kb)
    Y0 = rt.upload(rng.standard_normal((n, kb))) if y0 else None
    res = {}
    for tag, env in (("rt", "0"), ("v1", "1")):
        os.environ["USBS_ROWGEMM_V1"] = env
        ts = []
        for it in range(7):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(rt.stream)
            eng.rowgemm(X, B, Y, alpha=1.0, beta=0.5 if y0 else 0.0, Y0=Y0)
            e1.record(rt.stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[tag] = (float(np.median(ts[1:])), Y.cpu().numpy().copy())
    by = 8 * n * (ka + kb + (kb if y0 else 0))
    same = np.array_equal(res["rt"][1], res["v1"][1])
    print(f"ka={ka} kb={kb} Y0={y0}: row/thread {res['rt'][0]*1e3:.1f} us ({by/res['rt'][0]/1e6:.0f} GB/s)  "
          f"entry/thread {res['v1'][0]*1e3:.1f} us ({by/res['v1'][0]/1e6:.0f} GB/s)  bit-identical {same}", flush=True)
