"""Where the setup of a public solve() goes at C4 (problem upload and
planning, sketch test matrix, cold start, first iteration)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11801_b200 import instances, solver as S  # noqa: E402
from paper_2312_11801_b200.runtime import DeviceProblem, runtime  # noqa: E402

cfg_b = instances.baseline_config(sys.argv[1] if len(sys.argv) > 1 else "C4")
p = cfg_b.problem
rt = runtime()
torch.cuda.synchronize()
t = time.perf_counter()
marks = []


def mark(name):
    global t
    torch.cuda.synchronize()
    now = time.perf_counter()
    marks.append((name, 1e3 * (now - t)))
    t = now


for rep in range(2):
    marks.clear()
    t = time.perf_counter()
    dp = DeviceProblem(p, rt)
    mark("DeviceProblem (upload + merged pattern + SpMV plans)")
    cfg = S.SolverConfig(rho=cfg_b.rho, beta=cfg_b.beta, k_c=cfg_b.k_c, k_p=cfg_b.k_p, sketch_rank=cfg_b.sketch_rank,
                         eps=1e-12, max_iters=3, seed=cfg_b.seed)
    ds = S.DeviceSolver(p, cfg, dprob=dp)
    mark("DeviceSolver buffers")
    st = ds.cold_start()
    mark("cold_start (Lanczos on C + completion; Psi on a worker thread)")
    its = []
    ds.solve(init=st, callback=lambda info: its.append(time.perf_counter()))
    mark("3 iterations")
    print("rep", rep, [(n, round(v, 1)) for n, v in marks], flush=True)
