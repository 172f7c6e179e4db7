"""Warm per-call device time of the engine calls inside the alternating
passes (CUDA events around each call) and the wall time per pass, at a
config.  Diagnostic."""
import collections
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11801_b200 import instances, solver as S  # noqa: E402
from paper_2312_11801_b200.engine import Engine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
bc = instances.baseline_config(name)
cfg = S.SolverConfig(rho=bc.rho, beta=bc.beta, k_c=bc.k_c, k_p=bc.k_p, sketch_rank=bc.sketch_rank, eps=1e-12,
                     max_iters=4, seed=bc.seed)
rec = collections.defaultdict(list)
on = [False]


def wrap(nm):
    f = getattr(Engine, nm)

    def g(self, *a, **k):
        if not on[0]:
            return f(self, *a, **k)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(self.rt.stream)
        r = f(self, *a, **k)
        e1.record(self.rt.stream)
        rec[nm].append((e0, e1))
        return r
    setattr(Engine, nm, g)


for nm in ("vec", "compressed", "image", "dot_into", "ipm", "apply", "svec"):
    wrap(nm)
orig_alt = S.DeviceSolver.alternating_max
stats = []


def alt(self, *a, **k):
    torch.cuda.synchronize()
    on[0] = True
    t0 = time.perf_counter()
    r = orig_alt(self, *a, **k)
    torch.cuda.synchronize()
    stats.append((time.perf_counter() - t0, r[1]))
    on[0] = False
    return r


S.DeviceSolver.alternating_max = alt
S.solve(bc.problem, cfg)
torch.cuda.synchronize()
tot_wall = sum(w for w, _ in stats[1:])
tot_pass = sum(p for _, p in stats[1:])
print(f"{name}: alternating_max wall {tot_wall * 1e3:.1f} ms over {tot_pass} passes "
      f"({tot_wall / tot_pass * 1e6:.0f} us/pass incl. IPM)")
for nm, lst in rec.items():
    ms = [a.elapsed_time(b) for a, b in lst]
    print(f"  {nm:10s} calls {len(ms):5d}  mean {np.mean(ms) * 1e3:8.1f} us  total {np.sum(ms):8.2f} ms")
