#!/usr/bin/env python
"""Benchmark of the USBS hot path on B200 (BASELINE.json metric: USBS iters/s
and time-to-1e-3; operator-apply HBM GB/s).

Workload (N=1): BASELINE.json names no config for its metric, so the line is
quoted on the largest single-GPU config, C4: MaxCut SDP on the Chung-Lu
power-law graph (n = 10^6, exponent 2.5, mean degree 8, unit weights,
seed 3), Nystrom sketch r = 10, k_c = 10, k_p = 1, rho = 0.01, beta = 0.25
(SURVEY 8d).  A "step" is one USBS outer iteration.  W warm-up iterations,
then K timed iterations, each timed with CUDA events on the launching
stream; the C4 working set (Z 108 MB, Lanczos basis 264 MB, V/P/Psi 88/80/80
MB) exceeds L2 and L2 is also flushed (256 MiB write) between timed
iterations.  For N > 1 (torchrun) each rank runs an independent replica
(scaling "weak", value = all ranks' iterations / max-over-ranks time): at
C4's size one GPU holds the whole problem and the single-GPU persistent
Lanczos beats the row-sharded path.  --mode sharded
runs ONE row-sharded solve over the N GPUs instead (dist.py: row blocks of
Z, V, Q, the sketch and the m-vectors per rank; NCCL allgather before each
SpMV, allreduces of the k x k / d x d Grams and norms; scaling "strong",
value = outer iterations of the whole problem per second).

--impl reference times the reference algorithm on the host cores (the CPU
oracle port of the pure-Python reference; the reference itself cannot travel
to the GPU box), rank 0 only, on the same C4 problem.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

UNIT = "iters/s"
WORKLOADS = {
    "C1": "C1: MaxCut SDP, Erdos-Renyi n=800 p=0.06 (seed 0), explicit store, k_c=10, k_p=1, rho=0.01, beta=0.25",
    "C2": "C2: MaxCut SDP, 100x100 torus +-1 weights (seed 1), n=10000, sketch r=10, k_c=10, k_p=1, rho=0.01, "
          "beta=0.25",
    "C3": "C3: QAP SDP, l=20 (n=401, m=126574), W, D ints in [0,10] (seed 2), sketch r=20, k_c=20, k_p=0, "
          "rho=0.005, beta=0.25",
    "C4": "C4: MaxCut SDP, Chung-Lu n=10^6 (exponent 2.5, mean degree 8, unit weights, seed 3), sketch r=10, "
          "k_c=10, k_p=1, rho=0.01, beta=0.25",
    "C5": "C5: correlation-clustering SDP, n=63000 points, 32-NN (seed 4), m=1366291, sketch r=20, k_c=20, "
          "k_p=0, rho=0.01, beta=0.25",
}


def metric_name(cfg_name):
    return f"USBS outer iterations/s ({cfg_name})"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def baseline(name):
    from paper_2312_11801_b200 import instances as inst
    return inst.baseline_config(name)


def lanczos_bytes(n, nnz, restarts, m=32, k_c=10):
    """SURVEY 8d algorithmic bytes of one lanczos_top call (fused 3-read CGS2):
    sum over steps j of B_apply(1) + 24 n (j+1) + 16 n, with
    B_apply(1) = 12 nnz + 4 (n+1) + 16 n (Z assembled once per call, no
    separate dual read)."""
    ell = max(1, min(k_c + 3, m - 2))
    b_apply = 12 * nnz + 4 * (n + 1) + 16 * n
    total = 0
    for cyc in range(restarts + 1):
        j0 = 0 if cyc == 0 else ell
        for j in range(j0, m):
            total += b_apply + 24 * n * (j + 1) + 16 * n
    return total


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def traffic_from_profile(cfg_name):
    """DRAM bytes per Lanczos launch from the committed ncu --set full capture
    (profiles/lanczos_dram.json, keyed by config), with the algorithmic bytes of
    that same captured launch so the ratio is meaningful."""
    p = ROOT / "profiles" / "lanczos_dram.json"
    if p.exists():
        try:
            d = json.loads(p.read_text()).get(cfg_name)
            if d:
                return d.get("dram_bytes_per_launch"), d.get("algorithmic_bytes_per_launch"), d.get("source")
        except Exception:
            pass
    return None, None, None


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------------------
# CPU baseline / reference arm


def cpu_run(cfg_b, steps, warmup, budget_s=120.0):
    """Oracle (port of the reference algorithm) on host cores: cold start and
    W untimed iterations, then up to K timed outer iterations (stopping early
    once budget_s of timed work has been spent)."""
    from oracle import usbs_cpu as O
    p = cfg_b.problem
    cfg = O.Config(rho=cfg_b.rho, beta=cfg_b.beta, k_c=cfg_b.k_c, k_p=cfg_b.k_p, sketch_rank=cfg_b.sketch_rank,
                   eps=1e-12, max_iters=warmup + steps, seed=cfg_b.seed)
    marks = []

    def cb(info):
        marks.append(time.perf_counter())
        if len(marks) > warmup and marks[-1] - marks[warmup - 1] > budget_s:
            raise StopIteration

    t0 = time.perf_counter()
    try:
        O.solve(p, cfg, callback=cb)
    except StopIteration:
        pass
    base = marks[warmup - 1] if warmup >= 1 else t0
    done = len(marks) - warmup
    dt = marks[-1] - base
    return done / dt, done, dt


def bench_config(name, world):
    """The `config` object of the JSON line -- identical for the device arm and
    the reference arm (the driver compares them key by key)."""
    return {"workload": WORKLOADS[name],
            "parallelism": f"replicas x{world}" if world > 1 else "single process",
            "l2": "inputs larger than L2; also flushed (256 MiB write) between timed iterations (device arm)",
            "step": "one USBS outer iteration"}


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg_b = baseline(args.config)
    warm = max(1, args.warmup)
    value, done, dt = cpu_run(cfg_b, args.steps, warm, budget_s=args.ref_budget)
    line = {
        "impl": "reference", "metric": metric_name(args.config), "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": done, "warmup": warm, "ms_per_step": 1e3 * dt / max(done, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args.config, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores(), "kind": "port",
                         "sample": f"{done} outer iterations (of {args.steps} asked; timed work capped at "
                                   f"{args.ref_budget:.0f} s) after cold start + {warm} warm-up iterations "
                                   f"(numpy/scipy oracle port of the reference, OpenBLAS threads = host cores; "
                                   f"scipy CSR SpMV single-threaded)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# device arm


def _solver_cfg(S, cfg_b, **kw):
    base = dict(rho=cfg_b.rho, beta=cfg_b.beta, k_c=cfg_b.k_c, k_p=cfg_b.k_p, sketch_rank=cfg_b.sketch_rank,
                seed=cfg_b.seed)
    base.update(kw)
    return S.SolverConfig(**base)


def timed_solve(S, rt, cfg_b, warmup, steps, flush, dp=None, world=1, clocks=None, comm=None):
    """W untimed then K timed outer iterations of a device-resident solve
    (problem uploaded and cold start done before timing); per-iteration CUDA
    events on the launching stream, L2 flushed before each timed iteration."""
    import torch
    p = cfg_b.problem
    cfg = _solver_cfg(S, cfg_b, eps=1e-12, max_iters=warmup + steps)
    ds = S.DeviceSolver(p, cfg, dprob=dp, comm=comm)
    ds.lz_probe = []
    evs = []
    launches0 = [None]
    stream = rt.stream
    state0 = ds.cold_start()

    def cb(info):
        t = info.t
        if t >= warmup:
            evs[-1][1].record(stream)
        if t == warmup - 1:
            torch.cuda.synchronize()
            if world > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            if clocks is not None:
                clocks.start()
            launches0[0] = rt.launches()
            ds.lz_probe.clear()
        if warmup - 1 <= t < warmup + steps - 1:
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            evs.append((e0, e1))

    ds.solve(init=state0, callback=cb)
    torch.cuda.synchronize()
    clk = clocks.stop() if clocks is not None else None
    launches = rt.launches() - (launches0[0] or 0)
    it_ms = [a.elapsed_time(b) for a, b in evs]
    return ds, it_ms, launches, clk


def run_device(args):
    import torch

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    from paper_2312_11801_b200 import solver as S
    from paper_2312_11801_b200.runtime import DeviceProblem, runtime

    rt = runtime()
    cfg_b = baseline(args.config)
    p = cfg_b.problem
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=rt.device)
    if args.warmup < 1:
        raise SystemExit("--warmup must be >= 1")

    # ---- timed run: device-resident problem (uploaded before timing)
    dp = DeviceProblem(p, rt)
    clocks = ClockSampler(local)
    ds, it_ms, launches, clk = timed_solve(S, rt, cfg_b, args.warmup, args.steps, flush, dp=dp, world=world,
                                           clocks=clocks)
    total_ms = float(np.sum(it_ms))
    if world > 1:
        t = torch.tensor([total_ms], device=rt.device, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    steps = len(it_ms)
    value = world * steps / (total_ms / 1e3)

    # ---- roofline of the dominant kernel (persistent Lanczos, one launch per lanczos_top)
    info = dp.info()
    lz = ds.lz_probe
    lz_ms = [a.elapsed_time(b) for a, b, _, _ in lz]
    k_c = cfg_b.k_c
    lz_bytes = [lanczos_bytes(p.n, info.nnz_z, r, m=max(32, k_c + 1), k_c=k_c) for _, _, r, _ in lz]
    avg_ms = float(np.mean(lz_ms)) if lz_ms else float("nan")
    avg_bytes = float(np.mean(lz_bytes)) if lz_bytes else float("nan")
    achieved = avg_bytes / (avg_ms / 1e3) / 1e9
    peak, peak_src = peaks()
    lz_share = float(np.sum(lz_ms)) / total_ms if total_ms else None
    tr, tr_alg, tr_src = traffic_from_profile(args.config)
    cs, rows = dp.lanczos_plan(max(32, k_c + 1))
    lz_kernel = (f"k_lanczos_cl (one {cs}-CTA thread-block cluster, Q resident in shared memory, "
                 f"{rows} rows per CTA; 1 launch per lanczos_top)" if cs else
                 "k_lanczos_tma (persistent cooperative grid, Q tiles streamed by cp.async.bulk; 1 launch per lanczos_top)")
    traffic = None
    if tr is not None and tr_alg:
        traffic = tr * (avg_bytes / tr_alg)  # captured DRAM/algorithmic ratio applied to the average launch

    # ---- e2e: public API from host buffers (problem upload + per-iteration y D2H inside the timed region)
    torch.cuda.synchronize()
    d2h = {"bytes": 0}

    e2e_marks = []

    def cb_e2e(info):
        yh = info.y  # D2H of the iteration's dual iterate
        d2h["bytes"] += yh.nbytes + 8 * 16
        e2e_marks.append(time.perf_counter())

    cfg_e = _solver_cfg(S, cfg_b, eps=1e-12, max_iters=args.steps)
    cost = p.cost
    h2d = (cost.indptr.size * 8 + cost.indices.size * 4 + cost.data.size * 8 + 4 * 8 * p.n + p.b.nbytes
           + p.n * cfg_b.sketch_rank * 8 + 8 * p.n)
    t0 = time.perf_counter()
    st_e, _ = S.solve(p, cfg_e, callback=cb_e2e)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if os.environ.get("USBS_BENCH_E2E_DEBUG") and e2e_marks:
        print(f"[e2e] total {e2e_s * 1e3:.0f} ms: first callback {1e3 * (e2e_marks[0] - t0):.0f}, iterations "
              f"{1e3 * (e2e_marks[-1] - e2e_marks[0]):.0f}, exit {1e3 * (t0 + e2e_s - e2e_marks[-1]):.0f}; intervals "
              f"{[round(1e3 * (b - a)) for a, b in zip(e2e_marks, e2e_marks[1:])]}", file=sys.stderr, flush=True)
    e2e_steps = st_e.iterations
    e2e_value = world * e2e_steps / e2e_s

    # ---- time to 1e-3 (free-running device solve to convergence, wall clock)
    ttg = None
    if args.ttg_budget > 0:
        cfg_t = _solver_cfg(S, cfg_b, eps=1e-3, max_iters=100000, max_time=args.ttg_budget)
        t0 = time.perf_counter()
        st_t, _ = S.DeviceSolver(p, cfg_t, dprob=dp).solve()
        torch.cuda.synchronize()
        ttg = {"seconds": time.perf_counter() - t0, "iterations": st_t.iterations, "status": st_t.status,
               "rel_subopt": st_t.residuals.rel_subopt, "rel_infeas": st_t.residuals.rel_infeas,
               "dual_feas": st_t.residuals.dual_feas, "budget_s": args.ttg_budget,
               "note": "cold start included, problem already resident"}

    # ---- operator apply (K1), one lanczos_top and the compressed Gram on this config
    opx = operator_apply(rt, dp, cfg_b, flush) if args.opapply else None

    # ---- context: the C2 line of round 1 (small, L2-resident config)
    ctx = None
    if args.context and args.config != "C2":
        cb2 = baseline("C2")
        dp2 = DeviceProblem(cb2.problem, rt)
        _, ms2, _, _ = timed_solve(S, rt, cb2, 5, 20, flush, dp=dp2)
        ctx = {"C2": {"value": len(ms2) / (np.sum(ms2) / 1e3), "unit": UNIT, "steps": len(ms2), "warmup": 5}}
        del dp2

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, done, dt = cpu_run(cfg_b, max(1, min(args.steps, 60)), 1, budget_s=args.cpu_budget)
        cpu = {"value": v, "unit": UNIT, "cores": cores(), "kind": "port",
               "sample": f"{done} {args.config} outer iterations after cold start + 1 warm-up on the numpy/scipy "
                         f"oracle port (timed work capped at {args.cpu_budget:.0f} s)"}
    if rank == 0:
        line = {
            "metric": metric_name(args.config), "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": total_ms / max(steps, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(args.config, world),
            "roofline": {"kernel": lz_kernel,
                         "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": avg_bytes, "avg_launch_ms": avg_ms,
                         "launches": len(lz), "share_of_step": lz_share,
                         "traffic_source": tr_src,
                         "note": "algorithmic bytes per launch = sum over the call's Lanczos steps j of "
                                 "12 nnz(Z) + 4(n+1) + 16n + 24n(j+1) + 16n (SURVEY 8d; fused 3-read CGS2); "
                                 "traffic = ncu dram__bytes of the captured launch scaled by its "
                                 "algorithmic bytes"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d / max(e2e_steps, 1),
                    "d2h_bytes_per_step": d2h["bytes"] / max(e2e_steps, 1),
                    "note": "public solve(prob_host, cfg) from cold start incl. problem upload and device "
                            "planning and a D2H of y every iteration; wall clock"},
            "time_to_1e-3": ttg,
            "gpu_launches": int(launches),
            "clocks": clk,
            "iter_ms": {"min": float(np.min(it_ms)), "median": float(np.median(it_ms)), "max": float(np.max(it_ms))},
            "lanczos_matvecs_per_iter": float(np.mean([mv for _, _, _, mv in lz])) if lz else None,
        }
        if opx is not None:
            line["operator_apply"] = opx
        if ctx is not None:
            line["context"] = ctx
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def run_sharded(args):
    """N > 1 on a sharded config: one row-sharded solve over all ranks."""
    import datetime

    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    # test hook: USBS_BENCH_GLOO=1 puts every rank on cuda:0 with a gloo group
    # (a real exchange through host memory; NCCL needs distinct devices)
    gloo = os.environ.get("USBS_BENCH_GLOO") == "1"
    if gloo:
        local = 0
    torch.cuda.set_device(local)
    # a stuck collective raises after 10 minutes instead of hanging the job
    tmo = datetime.timedelta(minutes=10)
    if gloo:
        dist.init_process_group("gloo", timeout=tmo)
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local), timeout=tmo)
    from paper_2312_11801_b200 import solver as S
    from paper_2312_11801_b200.dist import Comm, Shard, ShardedDeviceProblem
    from paper_2312_11801_b200.runtime import runtime

    rt = runtime()
    cfg_b = baseline(args.config)
    p = cfg_b.problem
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=rt.device)
    shard = Shard.balanced(p.cost.indptr, world, rank)
    comm = Comm(world)
    sdp = ShardedDeviceProblem(p, shard, comm)
    clocks = ClockSampler(local)
    _, it_ms, launches, clk = timed_solve(S, rt, cfg_b, max(1, args.warmup), args.steps, flush, dp=sdp, world=world,
                                          clocks=clocks, comm=comm)
    t = torch.tensor([float(np.sum(it_ms))], device=rt.device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    steps = len(it_ms)
    value = steps / (total_ms / 1e3)

    # e2e: shard upload + planning from the host problem, cold start and
    # the iterations with a D2H of the rank's dual block every iteration
    d2h = {"bytes": 0}

    def cb_e2e(info):
        d2h["bytes"] += info.y.nbytes + 8 * 16

    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    sdp_e = ShardedDeviceProblem(p, shard, comm)
    st_e, _ = S.DeviceSolver(p, _solver_cfg(S, cfg_b, eps=1e-12, max_iters=args.steps), dprob=sdp_e,
                             comm=comm).solve(callback=cb_e2e)
    torch.cuda.synchronize()
    te = torch.tensor([time.perf_counter() - t0], device=rt.device, dtype=torch.float64)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = st_e.iterations / float(te.item())
    rows = shard.rows
    nnz_local = int(p.cost.indptr[shard.r1] - p.cost.indptr[shard.r0])
    h2d = nnz_local * 12 + 8 * (rows + 1) + 4 * 8 * rows
    if rank == 0:
        line = {
            "metric": metric_name(args.config), "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": total_ms / max(steps, 1), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config],
                       "parallelism": f"row-sharded x{world} ({'gloo test group' if gloo else 'NCCL'} allgather per "
                                      f"SpMV, allreduce of Grams/norms)",
                       "l2": "inputs larger than L2; also flushed (256 MiB write) between timed iterations",
                       "step": "one USBS outer iteration of the whole problem",
                       "rows_per_rank": [int(x) for x in np.diff(shard.bounds)]},
            "roofline": None,
            "cpu_baseline": None,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d / max(st_e.iterations, 1),
                    "d2h_bytes_per_step": d2h["bytes"] / max(st_e.iterations, 1),
                    "note": "rank 0's shard upload + planning from the host problem, cold start and a D2H of its "
                            "dual block every iteration; wall clock, max over ranks"},
            "gpu_launches": int(launches),
            "clocks": clk,
            "iter_ms": {"min": float(np.min(it_ms)), "median": float(np.median(it_ms)), "max": float(np.max(it_ms))},
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def _event_time(rt, fn, flush, reps=5, warm=2):
    import torch
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(rt.stream)
        r = fn()
        e1.record(rt.stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), r


def operator_apply(rt, dp, cfg_b, flush):
    """K1 on this config: Y = Z V for k = 1 and k_c + k_p, L2 flushed between
    launches, B_apply(k) = 12 nnz + 4 (n+1) + 16 n k; one lanczos_top on the
    slack operator; the d x d compressed Gram (K4) against the FP64 DMMA peak."""
    from paper_2312_11801_b200 import eigen
    from paper_2312_11801_b200.engine import Engine
    p = cfg_b.problem
    info = dp.info()
    y = np.random.default_rng(1234).standard_normal(p.m) * 1e-3
    if dp.has_ineq:
        y[dp.ineq_idx] = np.abs(y[dp.ineq_idx])
    dp.assemble(rt.upload(y))
    out = {"n": p.n, "nnz_z": info.nnz_z}
    peak, _ = peaks()
    k = cfg_b.k_c + cfg_b.k_p
    for kk in sorted({1, k}):
        V = rt.upload(np.linalg.qr(np.random.default_rng(1234).standard_normal((p.n, kk)))[0])
        Y = rt.empty(p.n, kk)
        ms, _ = _event_time(rt, lambda: dp.apply(1, V, out=Y), flush, reps=6)
        b = 12 * info.nnz_z + 4 * (p.n + 1) + 16 * p.n * kk
        gbs = b / (ms / 1e3) / 1e9
        out[f"k{kk}"] = {"ms": ms, "algorithmic_bytes": b, "achieved_gbs": gbs, "frac_of_measured_peak": gbs / peak}
    op = eigen.dual_slack_operator(dp, y)
    ms, r = _event_time(rt, lambda: eigen.lanczos_top(op, cfg_b.k_c, seed=0), flush, reps=3, warm=1)
    m = max(32, cfg_b.k_c + 1)
    b = lanczos_bytes(p.n, info.nnz_z, r.restarts, m=m, k_c=cfg_b.k_c)
    cs, _ = dp.lanczos_plan(m)
    out["lanczos_top"] = {"ms": ms, "matvecs": r.matvecs, "restarts": r.restarts, "algorithmic_bytes": b,
                          "achieved_gbs": b / (ms / 1e3) / 1e9, "frac_of_measured_peak": b / (ms / 1e3) / 1e9 / peak,
                          "kernel": "k_lanczos_cl (cluster)" if cs else "k_lanczos_tma (grid)"}
    eng = Engine(dp)
    d = k * (k + 1) // 2
    vq, _ = np.linalg.qr(np.random.default_rng(1234).standard_normal((p.n, k)))
    V = rt.upload(vq)
    G = rt.empty(d, d)
    ms, _ = _event_time(rt, lambda: eng.compressed(V, scale_gram=1.0, gram_out=G), flush)
    flop = p.m * d * (d + 1)
    try:
        fp64 = json.loads((ROOT / "profiles" / "fp64_peak.json").read_text())["fp64_dmma_tflops"]
    except Exception:
        fp64 = None
    out["k4_compressed_gram"] = {"ms": ms, "m": p.m, "d": d, "flop": flop, "achieved_tflops": flop / (ms / 1e3) / 1e12,
                                 "peak_tflops": fp64, "peak_source": "measured FP64 DMMA (profiles/fp64_peak.json)",
                                 "frac": (flop / (ms / 1e3) / 1e12 / fp64) if fp64 else None,
                                 "kernel": "k_compressed_mma_pipe (mma.sync m8n8k4 f64, pipelined row generation)"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="device", choices=["device", "reference"])
    ap.add_argument("--config", default="C4", choices=sorted(WORKLOADS))
    ap.add_argument("--opapply", type=int, default=1, help="also report K1 / one lanczos_top / K4 on the config")
    ap.add_argument("--context", type=int, default=1, help="also report the C2 device line for context")
    ap.add_argument("--ttg-budget", type=float, default=90.0, help="wall budget (s) of the time-to-1e-3 run")
    ap.add_argument("--cpu-budget", type=float, default=25.0, help="timed CPU work of the cpu_baseline leg (s)")
    ap.add_argument("--ref-budget", type=float, default=120.0, help="timed CPU work of the reference arm (s)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--mode", default="replicas", choices=["sharded", "replicas"],
                    help="N > 1: independent replicas (default) or one row-sharded solve")
    args = ap.parse_args()
    _, world, _ = dist_env()
    if args.impl == "reference":
        run_reference(args)
    elif args.mode == "sharded":
        run_sharded(args)
    else:
        run_device(args)


if __name__ == "__main__":
    main()
