"""K4 compressed Gram (d x d, DMMA) timing on C4 / C5 / C3: the pipelined
kernel (default) vs the round-1 kernel (USBS_K4_V1=1, strided tiles)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11801_b200 import instances  # noqa: E402
from paper_2312_11801_b200.engine import Engine  # noqa: E402
from paper_2312_11801_b200.runtime import DeviceProblem, runtime  # noqa: E402

peak = json.load(open(os.path.join(os.path.dirname(__file__), "fp64_peak.json")))["fp64_dmma_tflops"]
rt = runtime()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=rt.device)
for name in sys.argv[1:] or ["C4", "C5", "C3"]:
    bc = instances.baseline_config(name)
    p = bc.problem
    dp = DeviceProblem(p, rt)
    eng = Engine(dp)
    k = bc.k_c + bc.k_p
    d = k * (k + 1) // 2
    V = rt.upload(np.linalg.qr(np.random.default_rng(1234).standard_normal((p.n, k)))[0])
    G = rt.empty(d, d)
    res = {}
    for runs in ("0", "1"):
        os.environ["USBS_K4_V1"] = "1" if runs == "0" else "0"
        for _ in range(2):
            eng.compressed(V, scale_gram=1.0, gram_out=G)
        ts = []
        for _ in range(5):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(rt.stream)
            eng.compressed(V, scale_gram=1.0, gram_out=G)
            e1.record(rt.stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[runs] = (float(np.median(ts)), G.cpu().numpy().copy())
    flop = p.m * d * (d + 1)
    diff = np.abs(res["0"][1] - res["1"][1]).max() / np.abs(res["0"][1]).max()
    print(f"{name} d={d}: v1 {res['0'][0]:.3f} ms ({flop / res['0'][0] / 1e9:.1f} TF/s)  pipelined "
          f"{res['1'][0]:.3f} ms ({flop / res['1'][0] / 1e9:.1f} TF/s, {flop / res['1'][0] / 1e9 / peak:.0%} of "
          f"{peak} DMMA peak)  max rel diff {diff:.1e}", flush=True)
