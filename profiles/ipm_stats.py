"""Diagnostic (not a benchmark): per-iteration alternating passes, Newton
steps per IPM call and IPM time per call for a BASELINE config.

    python profiles/ipm_stats.py C3 12
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(name="C3", iters=12):
    import torch

    from paper_2312_11801_b200 import instances as inst, solver as S
    from paper_2312_11801_b200.engine import Engine

    cb_ = inst.baseline_config(name)
    cfg = S.SolverConfig(rho=cb_.rho, beta=cb_.beta, k_c=cb_.k_c, k_p=cb_.k_p, sketch_rank=cb_.sketch_rank,
                         eps=1e-12, max_iters=iters, seed=cb_.seed)
    calls = []
    orig = Engine.ipm

    def timed(self, k, has_eta, Q11, q12, lin_s, scal, warm, state_out, result, opts=None):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st = self.rt.stream
        e0.record(st)
        orig(self, k, has_eta, Q11, q12, lin_s, scal, warm, state_out, result, opts)
        e1.record(st)
        e1.synchronize()
        r = result.cpu().numpy()
        calls.append((Q11 is not None, warm is not None, int(r[1]), int(r[4]), e0.elapsed_time(e1)))

    Engine.ipm = timed
    rows = []

    def cb(info):
        rows.append((info.t, info.alt_passes, len(calls)))

    S.solve(cb_.problem, cfg, callback=cb)
    prev = 0
    for t, passes, ncalls in rows:
        cs = calls[prev:ncalls]
        prev = ncalls
        quad = [c for c in cs if c[0]]
        ev = [c for c in cs if not c[0]]
        nq = [c[2] for c in quad]
        print(f"t={t:3d} passes={passes:3d} quad calls={len(quad):3d} newton/call "
              f"min {min(nq) if nq else 0} med {int(np.median(nq)) if nq else 0} max {max(nq) if nq else 0} "
              f"sum {sum(nq)}  quad ms {sum(c[4] for c in quad):7.2f} ({np.mean([c[4] / max(c[2], 1) for c in quad]) if quad else 0:.3f} ms/newton)"
              f"  eval newton {[c[2] for c in ev]} ms {sum(c[4] for c in ev):.2f}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C3", int(sys.argv[2]) if len(sys.argv) > 2 else 12)
