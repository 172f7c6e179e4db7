#!/usr/bin/env python
"""Benchmark of the USBS hot path on B200 (BASELINE.json metric: USBS iters/s
and time-to-1e-3; operator-apply HBM GB/s).

Workload (N=1): BASELINE configs[1] = C2, MaxCut SDP on the 100x100 +-1 torus
(n = 10,000), Nystrom sketch r = 10, k_c = 10, k_p = 1, rho = 0.01,
beta = 0.25.  A "step" is one USBS outer iteration.  W warm-up
iterations, then K timed iterations; L2 is flushed (256 MiB write) between
timed iterations and each iteration is timed with CUDA events on the
launching stream.  For N > 1 (torchrun) each rank runs an independent
replica (C2 is "replicas only"); value = all ranks' iterations /
max-over-ranks time.

--impl reference times the reference algorithm on the host cores (the CPU
oracle port of the pure-Python reference; the reference itself cannot travel
to the GPU box), rank 0 only.
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

METRIC = "USBS outer iterations/s (C2 torus n=10^4, sketch r=10)"
UNIT = "iters/s"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def c2_problem():
    from paper_2312_11801_b200 import instances as inst
    return inst.baseline_config("C2")


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


def traffic_from_profile():
    """DRAM bytes per Lanczos launch from the committed ncu --set full summary."""
    p = ROOT / "profiles" / "lanczos_dram.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return d.get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------------------
# CPU baseline / reference arm


def cpu_run(cfg_b, steps, warmup, budget_s=120.0):
    """Oracle (port of the reference algorithm) on host cores: W untimed then
    up to K timed outer iterations (bounded by budget_s)."""
    from oracle import usbs_cpu as O
    p = cfg_b.problem
    cfg = O.Config(rho=cfg_b.rho, beta=cfg_b.beta, k_c=cfg_b.k_c, k_p=cfg_b.k_p, sketch_rank=cfg_b.sketch_rank,
                   eps=1e-12, max_iters=warmup + steps, seed=cfg_b.seed)
    marks = []

    def cb(info):
        marks.append(time.perf_counter())
        if len(marks) > warmup and marks[-1] - marks[warmup - 1 if warmup else 0] > budget_s:
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


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg_b = c2_problem()
    value, done, dt = cpu_run(cfg_b, args.steps, args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": done, "warmup": args.warmup, "ms_per_step": 1e3 * dt / max(done, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2: MaxCut SDP, 100x100 torus +-1 weights (seed 1), n=10000, sketch r=10, "
                               "k_c=10, k_p=1, rho=0.01, beta=0.25", "parallelism": "host"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores(), "kind": "port",
                         "sample": f"{done} outer iterations after {args.warmup} warm-up (numpy/scipy oracle, "
                                   f"OpenBLAS threads = host cores; scipy CSR SpMV single-threaded)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# device arm


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
    cfg_b = c2_problem()
    p = cfg_b.problem
    cfg = S.SolverConfig(rho=cfg_b.rho, beta=cfg_b.beta, k_c=cfg_b.k_c, k_p=cfg_b.k_p, sketch_rank=cfg_b.sketch_rank,
                         eps=1e-12, max_iters=args.warmup + args.steps, seed=cfg_b.seed)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=rt.device)
    stream = rt.stream

    # ---- timed run: device-resident problem (uploaded before timing)
    ds = S.DeviceSolver(p, cfg)
    ds.lz_probe = []
    evs = []
    launches0 = [None]
    state0 = ds.cold_start()
    clocks = ClockSampler(local)
    marks = {"t": 0}

    def cb(info):
        t = info.t
        if t == args.warmup - 1 or (args.warmup == 0 and t == -1):
            pass
        if t >= args.warmup:
            evs[-1][1].record(stream)
        if t == args.warmup - 1:
            # warm-up done: enter the timed region
            torch.cuda.synchronize()
            if world > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            clocks.start()
            launches0[0] = rt.launches()
            ds.lz_probe.clear()
        if t >= args.warmup - 1 and t < args.warmup + args.steps - 1:
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            evs.append((e0, e1))

    if args.warmup == 0:
        raise SystemExit("--warmup must be >= 1")
    st, _ = ds.solve(init=state0, callback=cb)
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = rt.launches() - (launches0[0] or 0)
    it_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = float(np.sum(it_ms))
    if world > 1:
        t = torch.tensor([total_ms], device=rt.device, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    steps = len(it_ms)
    value = world * steps / (total_ms / 1e3)
    # ---- roofline of the dominant kernel (persistent Lanczos)
    info = ds.dp.info()
    lz = ds.lz_probe
    lz_ms = [a.elapsed_time(b) for a, b, _, _ in lz]
    lz_bytes = [lanczos_bytes(p.n, info.nnz_z, r) for _, _, r, _ in lz]
    avg_ms = float(np.mean(lz_ms)) if lz_ms else float("nan")
    avg_bytes = float(np.mean(lz_bytes)) if lz_bytes else float("nan")
    achieved = avg_bytes / (avg_ms / 1e3) / 1e9
    peak, peak_src = peaks()
    lz_share = float(np.sum(lz_ms)) / total_ms if total_ms else None
    tr = traffic_from_profile()
    cs, rows = ds.dp.lanczos_plan(max(32, cfg_b.k_c + 1))
    lz_kernel = (f"k_lanczos_cl (one {cs}-CTA thread-block cluster, Q resident in shared memory, "
                 f"{rows} rows per CTA; 1 launch per lanczos_top)" if cs else
                 "k_lanczos (persistent cooperative grid; 1 launch per lanczos_top)")

    # ---- e2e: public API from host buffers (problem upload + per-iteration y D2H inside the timed region)
    torch.cuda.synchronize()
    d2h = {"bytes": 0}

    def cb_e2e(info):
        yh = info.y  # D2H of the iteration's dual iterate
        d2h["bytes"] += yh.nbytes + 8 * 16

    cfg_e = S.SolverConfig(rho=cfg_b.rho, beta=cfg_b.beta, k_c=cfg_b.k_c, k_p=cfg_b.k_p,
                           sketch_rank=cfg_b.sketch_rank, eps=1e-12, max_iters=args.steps, seed=cfg_b.seed)
    cost = p.cost
    h2d = (cost.indptr.size * 8 + cost.indices.size * 4 + cost.data.size * 8 + 4 * 8 * p.n + p.b.nbytes
           + p.n * cfg_b.sketch_rank * 8 + 8 * p.n)
    t0 = time.perf_counter()
    st_e, _ = S.solve(p, cfg_e, callback=cb_e2e)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    e2e_steps = st_e.iterations
    e2e_value = world * e2e_steps / e2e_s

    # ---- time to 1e-3 (free-running device solve to convergence)
    cfg_t = S.SolverConfig(rho=cfg_b.rho, beta=cfg_b.beta, k_c=cfg_b.k_c, k_p=cfg_b.k_p,
                           sketch_rank=cfg_b.sketch_rank, eps=1e-3, max_iters=3000, seed=cfg_b.seed)
    t0 = time.perf_counter()
    st_t, _ = S.solve(p, cfg_t)
    torch.cuda.synchronize()
    ttg = time.perf_counter() - t0

    # ---- C4-scale operator apply (K1) HBM roofline, if requested
    c4 = None
    if args.c4:
        c4 = c4_operator_apply(rt)

    cpu = None
    if rank == 0 and not args.no_cpu:
        v, done, dt = cpu_run(cfg_b, max(5, min(args.steps, 60)), 2, budget_s=25.0)
        cpu = {"value": v, "unit": UNIT, "cores": cores(), "kind": "port",
               "sample": f"{done} C2 outer iterations after 2 warm-up on the numpy/scipy oracle port"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": total_ms / max(steps, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C2: MaxCut SDP, 100x100 torus +-1 weights (seed 1), n=10000, sketch r=10, "
                                   "k_c=10, k_p=1, rho=0.01, beta=0.25",
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                       "l2": "flushed (256 MiB write) between timed iterations",
                       "step": "one USBS outer iteration"},
            "roofline": {"kernel": lz_kernel,
                         "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": tr, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": avg_bytes, "avg_launch_ms": avg_ms,
                         "launches": len(lz), "share_of_step": lz_share,
                         "note": "C2 working set (Z 0.7 MB, Q 2.6 MB) lives in shared memory / L2: the HBM "
                                 "fraction is low by construction; the kernel is latency-bound (3 cluster "
                                 "barriers per step, Rayleigh-Ritz per cycle), see DESIGN.md"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d / max(e2e_steps, 1),
                    "d2h_bytes_per_step": d2h["bytes"] / max(e2e_steps, 1),
                    "note": "public solve(prob_host, cfg) from cold start incl. problem upload and a D2H of y "
                            "every iteration; wall clock"},
            "time_to_1e-3": {"seconds": ttg, "iterations": st_t.iterations, "status": st_t.status,
                             "rel_subopt": st_t.residuals.rel_subopt, "rel_infeas": st_t.residuals.rel_infeas,
                             "dual_feas": st_t.residuals.dual_feas},
            "gpu_launches": int(launches),
            "clocks": clk,
            "iter_ms": {"min": float(np.min(it_ms)), "median": float(np.median(it_ms)), "max": float(np.max(it_ms))},
        }
        if c4 is not None:
            line["c4_operator_apply"] = c4
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def c4_operator_apply(rt):
    """K1 on C4 (n = 10^6 Chung-Lu, nnz(Z) ~ 9.98M): Y = Z V for k = 1 and 11,
    L2 flushed between launches; B_apply(k) = 12 nnz + 4 (n+1) + 16 n k."""
    import torch
    from paper_2312_11801_b200 import instances as inst
    from paper_2312_11801_b200.runtime import DeviceProblem

    cfg = inst.baseline_config("C4")
    p = cfg.problem
    dp = DeviceProblem(p, rt)
    info = dp.info()
    y = np.random.default_rng(1234).standard_normal(p.m) * 1e-3
    dp.assemble(rt.upload(y))
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=rt.device)
    out = {"n": p.n, "nnz_z": info.nnz_z}
    peak, _ = peaks()
    for k in (1, 11):
        V = rt.upload(np.linalg.qr(np.random.default_rng(1234).standard_normal((p.n, k)))[0])
        Y = rt.empty(p.n, k)
        ts = []
        for it in range(8):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(rt.stream)
            dp.apply(1, V, out=Y)
            e1.record(rt.stream)
            torch.cuda.synchronize()
            if it >= 2:
                ts.append(e0.elapsed_time(e1))
        b = 12 * info.nnz_z + 4 * (p.n + 1) + 16 * p.n * k
        ms = float(np.median(ts))
        gbs = b / (ms / 1e3) / 1e9
        out[f"k{k}"] = {"ms": ms, "algorithmic_bytes": b, "achieved_gbs": gbs, "frac_of_measured_peak": gbs / peak}
    # one lanczos_top on the C4 slack operator (grid kernel, Q streamed from HBM)
    from paper_2312_11801_b200 import eigen
    op = eigen.dual_slack_operator(dp, y)
    eigen.lanczos_top(op, 10, seed=0)
    ts, r = [], None
    for _ in range(3):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(rt.stream)
        r = eigen.lanczos_top(op, 10, seed=0)
        e1.record(rt.stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    b = lanczos_bytes(p.n, info.nnz_z, r.restarts)
    out["lanczos_top"] = {"ms": ms, "matvecs": r.matvecs, "restarts": r.restarts, "algorithmic_bytes": b,
                          "achieved_gbs": b / (ms / 1e3) / 1e9, "frac_of_measured_peak": b / (ms / 1e3) / 1e9 / peak,
                          "kernel": "k_lanczos (grid)"}
    # K4: the d x d compressed Gram (SYRK over m generated rows) on the FP64
    # tensor cores, against the measured FP64 DMMA peak (profiles/fp64_peak.json)
    from paper_2312_11801_b200.engine import Engine
    eng = Engine(dp)
    k = cfg.k_c + cfg.k_p
    d = k * (k + 1) // 2
    vq, _ = np.linalg.qr(np.random.default_rng(1234).standard_normal((p.n, k)))
    V = rt.upload(vq)
    G = rt.empty(d, d)
    for _ in range(2):
        eng.compressed(V, scale_gram=1.0, gram_out=G)
    ts = []
    for _ in range(5):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(rt.stream)
        eng.compressed(V, scale_gram=1.0, gram_out=G)
        e1.record(rt.stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    flop = p.m * d * (d + 1)
    try:
        fp64 = json.loads((ROOT / "profiles" / "fp64_peak.json").read_text())["fp64_dmma_tflops"]
    except Exception:
        fp64 = None
    out["k4_compressed_gram"] = {"ms": ms, "m": p.m, "d": d, "flop": flop, "achieved_tflops": flop / (ms / 1e3) / 1e12,
                                 "peak_tflops": fp64, "peak_source": "measured FP64 DMMA (profiles/fp64_peak.json)",
                                 "frac": (flop / (ms / 1e3) / 1e12 / fp64) if fp64 else None,
                                 "kernel": "k_compressed_mma (mma.sync m8n8k4 f64)"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="device", choices=["device", "reference"])
    ap.add_argument("--c4", type=int, default=1, help="also measure K1 on the C4 graph (n=1e6)")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_device(args)


if __name__ == "__main__":
    main()
