"""Free-running oracle (the reference algorithm restated, pinned to the
reference) solve of a BASELINE config to converged(1e-3) (bundle.py:154-158)
under a wall budget; writes profiles/r02_oracle_<cfg>.json with the
per-iteration objective/residual trace, time-to-1e-3 and the end state.
Run on the build container's host cores (not the GPU box)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import usbs_cpu as O  # noqa: E402
from paper_2312_11801_b200 import instances as inst  # noqa: E402

name = sys.argv[1]
budget = float(sys.argv[2]) if len(sys.argv) > 2 else 3600.0
t0 = time.time()
bc = inst.baseline_config(name)
p = bc.problem
build_s = time.time() - t0
cfg = O.Config(rho=bc.rho, beta=bc.beta, k_c=bc.k_c, k_p=bc.k_p, sketch_rank=bc.sketch_rank, eps=1e-3,
               max_iters=100000, max_time=budget, seed=bc.seed)
trace = []
first = {}


def cb(r):
    res = r.residuals
    trace.append([r.t, r.elapsed, r.f_y, res.rel_subopt, res.rel_infeas, res.dual_feas, r.step == "descent"])
    if "t" not in first and res.converged(1e-3):
        first.update(t=r.t + 1, seconds=r.elapsed)


st, _ = O.solve(p, cfg, callback=cb)
out = {"config": name, "n": p.n, "m": p.m, "cores": len(os.sched_getaffinity(0)),
       "threads": os.environ.get("OMP_NUM_THREADS"), "build_seconds": build_s, "budget_s": budget,
       "status": st.status, "iterations": st.iterations, "descent_steps": st.descent_steps,
       "f_y": st.f_y, "cost_ip": st.last_primal.cost_ip,
       "objective_unscaled": float(p.unscale_objective(st.last_primal.cost_ip)) if hasattr(p, "unscale_objective") else None,
       "residuals": vars(st.residuals), "time_to_1e-3": first or None,
       "seconds": trace[-1][1] if trace else 0.0, "trace": trace}
with open(os.path.join(ROOT, "profiles", f"r02_oracle_{name}.json"), "w") as f:
    json.dump(out, f)
print(name, st.status, st.iterations, first, flush=True)
