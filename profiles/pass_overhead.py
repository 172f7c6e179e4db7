"""Per outer iteration at a config: wall time vs the summed IPM device time
(events around every ipm_quad call) and the number of alternating passes --
what the passes cost besides the IPM (launches, host syncs, K4w, images).
Diagnostic."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11801_b200 import instances, solver as S  # noqa: E402
from paper_2312_11801_b200.engine import Engine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 8
bc = instances.baseline_config(name)
cfg = S.SolverConfig(rho=bc.rho, beta=bc.beta, k_c=bc.k_c, k_p=bc.k_p, sketch_rank=bc.sketch_rank, eps=1e-12,
                     max_iters=its, seed=bc.seed)
ev = []
orig = Engine.ipm


def timed(self, *a, **k):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(self.rt.stream)
    orig(self, *a, **k)
    e1.record(self.rt.stream)
    ev.append((e0, e1, a[1] is not None))  # Q11 given: the quad solve


Engine.ipm = timed
rows = []
t_last = [None]


def cb(info):
    torch.cuda.synchronize()
    now = time.perf_counter()
    if t_last[0] is not None:
        rows.append((info.t, now - t_last[0], info.alt_passes, len(ev)))
    t_last[0] = now


S.solve(bc.problem, cfg, callback=cb)
prev = None
for t, wall, passes, nev in rows:
    cur = ev[:nev] if prev is None else ev[prev:nev]
    prev = nev
    ipm_ms = sum(a.elapsed_time(b) for a, b, quad in cur if quad)
    print(f"t={t}: wall {wall * 1e3:.1f} ms, passes {passes}, quad IPM {ipm_ms:.1f} ms, "
          f"rest {wall * 1e3 - ipm_ms:.1f} ms ({(wall * 1e3 - ipm_ms) / max(passes, 1) * 1e3:.0f} us/pass)", flush=True)
