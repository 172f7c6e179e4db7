"""Where the e2e wall time of bench.py's public solve() goes at C4: setup
(problem upload + planning), cold start, then per-iteration wall times
(callback stamps), twice in one process.  Diagnostic, not a benchmark."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11801_b200 import instances, solver as S  # noqa: E402

bc = instances.baseline_config(sys.argv[1] if len(sys.argv) > 1 else "C4")
p = bc.problem
for rep in range(2):
    cfg = S.SolverConfig(rho=bc.rho, beta=bc.beta, k_c=bc.k_c, k_p=bc.k_p, sketch_rank=bc.sketch_rank, eps=1e-12,
                         max_iters=20, seed=bc.seed)
    stamps = []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st, _ = S.solve(p, cfg, callback=lambda info: stamps.append((time.perf_counter(), info.lanczos_matvecs,
                                                                 info.alt_passes, info.y.shape)))
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
    ts = np.array([s[0] for s in stamps]) - t0
    its = np.diff(np.concatenate([[0.0], ts]))
    print(f"rep {rep}: total {tot:.3f} s, {st.iterations} its, e2e {st.iterations / tot:.2f} it/s; first callback "
          f"at {ts[0]:.3f} s; iteration ms {np.round(its[1:] * 1e3, 1).tolist()}; matvecs "
          f"{[s[1] for s in stamps]}", flush=True)
