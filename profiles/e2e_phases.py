"""Wall-clock phases of the public solve() at C4 (20 its from cold start):
the solver methods wrapped with a device sync and a timestamp.  Diagnostic
(the syncs serialise what would otherwise overlap)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11801_b200 import instances, runtime, solver as S  # noqa: E402

bc = instances.baseline_config("C4")
p = bc.problem
log = []
T0 = [0.0]


def wrap(cls, name):
    f = getattr(cls, name)

    def g(*a, **k):
        t = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        log.append((name, t - T0[0], time.perf_counter() - t))
        return r
    setattr(cls, name, g)


for nm in ("cold_start", "penalized_lanczos", "alternating_max", "model_update", "primal_output", "residuals"):
    wrap(S.DeviceSolver, nm)
wrap(runtime.DeviceProblem, "__init__")
wrap(S.DeviceSketchStore, "update")
for rep in range(2):
    cfg = S.SolverConfig(rho=bc.rho, beta=bc.beta, k_c=bc.k_c, k_p=bc.k_p, sketch_rank=bc.sketch_rank, eps=1e-12,
                         max_iters=20, seed=bc.seed)
    log.clear()
    torch.cuda.synchronize()
    T0[0] = time.perf_counter()
    S.solve(p, cfg)
    torch.cuda.synchronize()
    tot = time.perf_counter() - T0[0]
    agg = {}
    for name, start, dur in log:
        a = agg.setdefault(name, [0, 0.0, start])
        a[0] += 1
        a[1] += dur
    print(f"rep {rep}: total {tot * 1e3:.0f} ms; " + "; ".join(
        f"{k} x{v[0]} {v[1] * 1e3:.0f} ms (first at {v[2] * 1e3:.0f})" for k, v in agg.items()), flush=True)
