"""Variance of the e2e leg (public solve() at C4, 20 its, y read every iteration): 6 repetitions in one
process; first-callback time, sum of iteration intervals, exit time.  Diagnostic."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
import torch
from paper_2312_11801_b200 import instances, solver as S
bc = instances.baseline_config("C4")
p = bc.problem
for rep in range(6):
    cfg = S.SolverConfig(rho=bc.rho, beta=bc.beta, k_c=bc.k_c, k_p=bc.k_p, sketch_rank=bc.sketch_rank, eps=1e-12, max_iters=20, seed=bc.seed)
    st_ = []
    torch.cuda.synchronize(); t0 = time.perf_counter()
    def cb(info):
        t = time.perf_counter(); y = info.y; st_.append((t, time.perf_counter() - t))
    st, _ = S.solve(p, cfg, callback=cb)
    torch.cuda.synchronize(); tot = time.perf_counter() - t0
    ts = np.array([s[0] for s in st_]) - t0
    print(f"rep {rep}: total {tot*1e3:.0f} ms ({20/tot:.1f} it/s); first cb {ts[0]*1e3:.0f}; iters {1e3*(ts[-1]-ts[0]):.0f}; exit {1e3*(tot-ts[-1]):.0f}; y reads {1e3*sum(s[1] for s in st_):.0f} ms", flush=True)
