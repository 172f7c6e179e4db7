"""Run the device solver on each BASELINE config (C1..C5) for a bounded
number of outer iterations / seconds and report it/s and the residuals.

    python profiles/configs.py C1 C2 C3 C4 C5 [--iters N] [--budget S]

Outer iterations/s is measured after 3 warm-up iterations with CUDA-synced
wall clock (the same definition as bench.py's e2e, problem upload excluded).
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def run(name, iters, budget, eps):
    import torch

    from paper_2312_11801_b200 import instances as inst, solver as S

    t0 = time.perf_counter()
    cfg_b = inst.baseline_config(name)
    p = cfg_b.problem
    t_build = time.perf_counter() - t0
    cfg = S.SolverConfig(rho=cfg_b.rho, beta=cfg_b.beta, k_c=cfg_b.k_c, k_p=cfg_b.k_p, sketch_rank=cfg_b.sketch_rank,
                         eps=eps, max_iters=iters, seed=cfg_b.seed, max_time=budget)
    t0 = time.perf_counter()
    ds = S.DeviceSolver(p, cfg)
    st0 = ds.cold_start()
    torch.cuda.synchronize()
    t_up = time.perf_counter() - t0
    rec = {"t": [], "matvecs": [], "restarts": []}
    warm = 3

    def cb(info):
        torch.cuda.synchronize()
        rec["t"].append(time.perf_counter())
        rec["matvecs"].append(info.lanczos_matvecs)
        rec["restarts"].append(info.lanczos_restarts)

    t0 = time.perf_counter()
    st, _ = ds.solve(init=st0, callback=cb)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ts = rec["t"]
    its = len(ts)
    ips = (its - warm) / (ts[-1] - ts[warm - 1]) if its > warm + 1 else its / wall
    r = st.residuals
    return {"config": name, "n": p.n, "m": p.m, "nnz_c": int(p.cost.nnz), "build_s": t_build,
            "upload_and_cold_start_s": t_up, "iterations": its, "wall_s": wall, "iters_per_s": ips,
            "status": st.status, "rel_subopt": r.rel_subopt, "rel_infeas": r.rel_infeas, "dual_feas": r.dual_feas,
            "matvecs_per_iter": sum(rec["matvecs"]) / max(its, 1),
            "time_to_eps_s": (wall if st.status == "converged" else None),
            "f_y": st.f_y, "cost_ip": st.last_primal.cost_ip,
            "objective_unscaled": float(p.unscale_objective(st.last_primal.cost_ip)),
            "descent_steps": st.descent_steps, "null_steps": st.null_steps}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--iters", type=int, default=60)
    ap.add_argument("--budget", type=float, default=120.0)
    ap.add_argument("--eps", type=float, default=1e-3)
    a = ap.parse_args()
    for c in a.configs:
        try:
            print(json.dumps(run(c, a.iters, a.budget, a.eps)), flush=True)
        except Exception as e:  # report and continue with the next config
            print(json.dumps({"config": c, "error": f"{type(e).__name__}: {e}"}), flush=True)


if __name__ == "__main__":
    main()
