"""Wall-clock of the first outer iteration's phases in a warm process (second solve) at C4."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2312_11801_b200 import instances, solver as S
bc = instances.baseline_config("C4")
p = bc.problem
cfg = S.SolverConfig(rho=bc.rho, beta=bc.beta, k_c=bc.k_c, k_p=bc.k_p, sketch_rank=bc.sketch_rank, eps=1e-12, max_iters=3, seed=bc.seed)
log = []
def wrap(cls, name):
    f = getattr(cls, name)
    def g(*a, **k):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        log.append((name, (time.perf_counter() - t) * 1e3))
        return r
    setattr(cls, name, g)
for nm in ("cold_start", "penalized_lanczos", "alternating_max", "model_update", "_eval_at_candidate", "completion"):
    if hasattr(S.DeviceSolver, nm): wrap(S.DeviceSolver, nm)
if hasattr(S, "SketchStore"): wrap(S.SketchStore, "update")
for rep in range(2):
    log.clear()
    t0 = time.perf_counter()
    marks = []
    S.solve(p, cfg, callback=lambda i: marks.append(time.perf_counter() - t0))
    torch.cuda.synchronize()
    print("rep", rep, "callbacks at", [round(m * 1e3) for m in marks], "total", round((time.perf_counter() - t0) * 1e3))
    print("   ", [(n, round(v, 1)) for n, v in log])
