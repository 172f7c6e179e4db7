"""Exit-time reconstruct at C4 (n = 10^6, r = 10): device part vs the D2H of
the n x r half factor vs the host thin SVD.  Diagnostic."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11801_b200 import instances, solver as S  # noqa: E402

bc = instances.baseline_config("C4")
cfg = S.SolverConfig(rho=bc.rho, beta=bc.beta, k_c=bc.k_c, k_p=bc.k_p, sketch_rank=bc.sketch_rank, eps=1e-12,
                     max_iters=3, seed=bc.seed)
ds = S.DeviceSolver(bc.problem, cfg)
st, out = ds.solve()
store = st.model.store
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    u, lams = store.factorize()
    t1 = time.perf_counter()
    h = np.ascontiguousarray(u)
    t2 = time.perf_counter()
    a = np.linalg.svd(h, full_matrices=False)
    t3 = time.perf_counter()
    print(f"factorize {1e3 * (t1 - t0):.1f} ms (incl. D2H + host SVD); a second host SVD of the {h.shape} factor "
          f"{1e3 * (t3 - t2):.1f} ms; threads {os.cpu_count()}", flush=True)
