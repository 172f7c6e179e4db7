"""A/B of the grid Lanczos kernels on one config: v1 (USBS_LZ_V1=1) vs the
TMA-pipelined variant; eigenvalues, matvec counts, CUDA-event time per call
and phase timers (USBS_LZ_PROF)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11801_b200 import eigen, instances  # noqa: E402
from paper_2312_11801_b200.runtime import DeviceProblem, runtime  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
small = len(sys.argv) > 2 and sys.argv[2] == "small"
t0 = time.time()
cfg = instances.baseline_config(name, small=small)
p = cfg.problem
rt = runtime()
dp = DeviceProblem(p, rt)
print(f"{name} n={p.n} build+upload {time.time()-t0:.1f}s", flush=True)
y = np.random.default_rng(1234).standard_normal(p.m) * 1e-3
if dp.has_ineq:
    y[dp.ineq_idx] = -np.abs(y[dp.ineq_idx])
dp.assemble(rt.upload(y))
op = eigen.dual_slack_operator(dp, y)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=rt.device)
out = {}
for tag, env in (("v1", "1"), ("tma", "0")):
    os.environ["USBS_LZ_V1"] = env
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
    out[tag] = {"ms": float(np.median(ts)), "matvecs": r.matvecs, "restarts": r.restarts,
                "vals": [float(v) for v in r.eigenvalues], "conv": bool(r.converged),
                "vec": r.eigenvectors[:, 0].copy()}
    print(tag, json.dumps({k: v for k, v in out[tag].items() if k != "vec"}), flush=True)
a, b = out["v1"], out["tma"]
dv = np.max(np.abs(np.array(a["vals"]) - np.array(b["vals"])) / np.maximum(1e-300, np.abs(a["vals"])))
v1, v2 = a["vec"], b["vec"]
print("max rel eig diff", dv, "vec0 |cos|", abs(v1 @ v2) / np.linalg.norm(v1) / np.linalg.norm(v2),
      "speedup", a["ms"] / b["ms"], flush=True)
# phase timers of the TMA kernel
os.environ["USBS_LZ_PROF"] = "1"
import ctypes as C  # noqa: E402
buf = (C.c_ulonglong * 1024)()
rt.lib.usbs_lanczos_profile(rt.h, buf, 1)
r = eigen.lanczos_top(op, cfg.k_c, seed=0)
rt.lib.usbs_lanczos_profile(rt.h, buf, 1)
names = ["spmv", "pass1", "gridsync", "pass2", "pass3", "rr", "restart", "cycle_end"]
steps = r.matvecs
print("phase us/step:", {nm: round(buf[i] / 1e3 / steps, 2) for i, nm in enumerate(names)}, flush=True)
G = dp.info().lanczos_blocks
import ctypes as C  # noqa: E402,F811
G = int(os.environ.get("LZG_G", "144"))
bw = np.array([[buf[32 + 5 * b + s] for s in range(5)] for b in range(G)], dtype=float) / 1e3 / steps
labels = ["spmv", "pass1", "sumsB", "pass2", "passC"]
print("per-block us/step  mean:", dict(zip(labels, np.round(bw.mean(0), 2))), flush=True)
print("per-block us/step   max:", dict(zip(labels, np.round(bw.max(0), 2))),
      "argmax:", dict(zip(labels, bw.argmax(0).tolist())), flush=True)
tot = bw.sum(1)
print("block totals: min %.1f mean %.1f max %.1f (block %d)" % (tot.min(), tot.mean(), tot.max(), tot.argmax()))
print("first blocks:", np.round(bw[:4], 1).tolist())
