"""Diagnostic A/B (not a benchmark): C3 (QAP l = 20, IPM at d = 210) or C5
for a few iterations with the library named by USBS_LIB; prints seconds
per iteration and saves the f(y) trajectory so two builds can be checked
for bit-identical results.

    USBS_LIB=... python profiles/ab_c3.py C3 10 out.npy
"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main(name, iters, out):
    import torch
    from paper_2312_11801_b200 import instances as inst, solver as S
    cb = inst.baseline_config(name)
    cfg = S.SolverConfig(rho=cb.rho, beta=cb.beta, k_c=cb.k_c, k_p=cb.k_p, sketch_rank=cb.sketch_rank,
                         eps=1e-12, max_iters=iters, seed=cb.seed)
    fs, ts = [], []

    def cb_(info):
        torch.cuda.synchronize()
        fs.append(info.f_y)
        ts.append(time.perf_counter())

    S.solve(cb.problem, cfg, callback=cb_)
    dt = np.diff(ts[2:])
    np.save(out, np.array(fs))
    print(f"{name}: {len(fs)} iterations, {dt.mean() * 1e3:.2f} ms/iteration after 2 (min {dt.min() * 1e3:.2f})")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3])
