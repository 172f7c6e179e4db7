"""Small driver for ncu captures of individual kernels (not a benchmark).

    python profiles/prof_kernels.py lanczos   # k_lanczos on C2 slack operator
    python profiles/prof_kernels.py ipm       # k_ipm (d = 66) on a C2-like subproblem
    python profiles/prof_kernels.py spmm      # K1 on C4 (n = 1e6), k = 1 and 11
    python profiles/prof_kernels.py lanczos4  # k_lanczos on the C4 slack operator (HBM-resident Q)
    python profiles/prof_kernels.py compressed  # K4 compressed d x d Gram on C3, C4, C5 (FP64 roofline)
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(which):
    import torch

    from paper_2312_11801_b200 import eigen, instances as inst, subproblem
    from paper_2312_11801_b200.runtime import DeviceProblem

    if which in ("lanczos", "lanczos4"):
        p = inst.baseline_config("C2" if which == "lanczos" else "C4").problem
        dp = DeviceProblem(p)
        y = np.random.default_rng(1234).standard_normal(p.m) * 1e-3
        import ctypes as C
        import os
        import time
        for _ in range(4):
            r = eigen.lanczos_top(eigen.dual_slack_operator(dp, y), 10, seed=0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = 10
        for _ in range(reps):
            r = eigen.lanczos_top(eigen.dual_slack_operator(dp, y), 10, seed=0)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps
        print("lanczos", r.eigenvalues[0], r.restarts, r.matvecs, f"{dt * 1e3:.3f} ms/call",
              f"{dt / r.matvecs * 1e6:.2f} us/step", "blocks", dp.info().lanczos_blocks,
              "plan", dp.lanczos_plan(max(32, 11)))
        # step j moves B_apply(1) + 24 n (j+1) + 16 n bytes (fused 3-read CGS2)
        nnz = dp.info().nnz_z
        bapp = 12 * nnz + 4 * (p.n + 1) + 8 * p.n + 16 * p.n
        m, ell, tot, j0 = 32, 13, 0, 0
        for c in range(r.restarts + 1):
            for j in range(j0, m):
                tot += bapp + 24 * p.n * (j + 1) + 16 * p.n
            j0 = ell
        print(f"  algorithmic {tot / 1e9:.3f} GB/call -> {tot / dt / 1e9:.0f} GB/s")
        if os.environ.get("USBS_LZ_PROF"):
            out = (C.c_uint64 * 1024)()
            dp.rt.lib.usbs_lanczos_profile(dp.rt.h, out, 1)
            names = ["phaseA", "barriers", "phaseB", "phaseC", "endcycle", "rayleigh_ritz", "restart",
                     "spmv(cluster)"]
            tot = sum(out[:8])
            for nm, v in zip(names, out[:8]):
                print(f"  {nm:14s} {v / 1e6 / (reps + 4):8.3f} ms/call  {100 * v / max(tot, 1):5.1f}%")
            nrr = (reps + 4) * (r.restarts + 1)
            for nm, v in zip(["setup", "bisection", "inverse-it", "output"], out[8:12]):
                print(f"    rr {nm:12s} {v / 1e3 / nrr:8.2f} us per Rayleigh-Ritz")
            G = dp.info().lanczos_blocks
            pb = np.array([[out[32 + 4 * b + q] for q in range(4)] for b in range(G)], float)
            pb /= 1e3 * (reps + 4) * r.matvecs
            if pb.sum() > 0:
                for q, nm in enumerate(["spmv", "Q^T w", "phase B", "phase C"]):
                    print(f"  per-block {nm:8s} us/step: mean {pb[:, q].mean():6.1f} max {pb[:, q].max():6.1f} "
                          f"(b={pb[:, q].argmax()}) min {pb[:, q].min():6.1f}")
        if os.environ.get("USBS_LZ_SWEEP"):
            for g in (8, 16, 32, 64, 148):
                os.environ["USBS_LZ_BLOCKS"] = str(g)
                dpg = DeviceProblem(p)
                eigen.lanczos_top(eigen.dual_slack_operator(dpg, y), 10, seed=0)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for _ in range(5):
                    r = eigen.lanczos_top(eigen.dual_slack_operator(dpg, y), 10, seed=0)
                torch.cuda.synchronize()
                dt = (time.perf_counter() - t0) / 5
                print(f"  G={g:4d}: {dt * 1e3:.3f} ms/call")
    elif which == "ipm":
        rng = np.random.default_rng(11)
        k = 11
        d = k * (k + 1) // 2
        a = rng.standard_normal((d + 5, d))
        z = rng.standard_normal(d + 5)

        class Q:
            pass

        q = Q()
        q.quad_ss, q.quad_s_eta, q.quad_eta = a.T @ a / (d + 5), a.T @ z / (d + 5), float(z @ z / (d + 5))
        q.lin_s, q.lin_eta, q.has_eta, q.k = rng.standard_normal(d), float(rng.standard_normal()), True, k
        import time
        for _ in range(4):
            r = subproblem.ipm_quad(q)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            r = subproblem.ipm_quad(q)
        dt = (time.perf_counter() - t0) / 10
        print("ipm d=66", r.value, r.newton_iters, f"{dt * 1e3:.3f} ms/solve (incl. host copies)")
        import ctypes as C
        import os
        if os.environ.get("USBS_IPM_PROF"):
            from paper_2312_11801_b200.runtime import runtime
            rt = runtime()
            out = (C.c_uint64 * 10)()
            rt.lib.usbs_ipm_profile(rt.h, out, 1)
            names = ["stationarity", "S^-1", "rd/rhs", "M build", "Cholesky", "solves", "Eds/dirs", "line search",
                     "update"]
            tot = sum(out[:9])
            for nm, v in zip(names, out[:9]):
                print(f"  {nm:14s} {v / 1e3 / (14 * 14):8.2f} us/newton  {100 * v / max(tot, 1):5.1f}%")
        k = 20
        d = k * (k + 1) // 2
        a = rng.standard_normal((d + 5, d))
        z = rng.standard_normal(d + 5)
        q.quad_ss, q.quad_s_eta, q.quad_eta = a.T @ a / (d + 5), a.T @ z / (d + 5), float(z @ z / (d + 5))
        q.lin_s, q.lin_eta, q.k = rng.standard_normal(d), float(rng.standard_normal()), k
        r = subproblem.ipm_quad(q)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            r = subproblem.ipm_quad(q)
        dt = (time.perf_counter() - t0) / 3
        print("ipm d=210", r.value, r.newton_iters, f"{dt * 1e3:.3f} ms/solve (incl. host copies)")
        if os.environ.get("USBS_IPM_PROF"):
            out = (C.c_uint64 * 10)()
            rt.lib.usbs_ipm_profile(rt.h, out, 1)
            tot = sum(out[:9])
            nn = 4 * r.newton_iters
            for nm, v in zip(names, out[:9]):
                print(f"  {nm:14s} {v / 1e3 / nn:8.2f} us/newton  {100 * v / max(tot, 1):5.1f}%")
    elif which == "compressed":
        import json
        from paper_2312_11801_b200.engine import Engine
        peak = json.loads((ROOT / "profiles" / "fp64_peak.json").read_text())["fp64_dmma_tflops"]
        for name in ("C3", "C4", "C5"):
            cb = inst.baseline_config(name)
            p = cb.problem
            dp = DeviceProblem(p)
            eng = Engine(dp)
            k = cb.k_c + cb.k_p
            d = k * (k + 1) // 2
            v, _ = np.linalg.qr(np.random.default_rng(1234).standard_normal((p.n, k)))
            V = dp.rt.upload(v)
            G = dp.rt.empty(d, d)
            for _ in range(2):
                eng.compressed(V, scale_gram=1.0, gram_out=G)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 5
            e0.record(dp.rt.stream)
            for _ in range(reps):
                eng.compressed(V, scale_gram=1.0, gram_out=G)
            e1.record(dp.rt.stream)
            e1.synchronize()
            ms = e0.elapsed_time(e1) / reps
            flop = p.m * d * (d + 1)  # lower triangle incl. diagonal, multiply-add = 2 flop
            print(json.dumps({"config": name, "m": p.m, "d": d, "ms": ms, "gflop": flop / 1e9,
                              "tflops": flop / (ms * 1e-3) / 1e12, "frac_of_fp64_dmma_peak": flop / (ms * 1e-3) / 1e12 / peak}))
    elif which == "spmm":
        p = inst.baseline_config("C4").problem
        dp = DeviceProblem(p)
        dp.assemble(dp.rt.upload(np.random.default_rng(1).standard_normal(p.m) * 1e-3))
        nnz = dp.info().nnz_z
        for k in (1, 11):
            V = dp.rt.upload(np.random.default_rng(2).standard_normal((p.n, k)))
            out = dp.rt.empty(p.n, k)
            for _ in range(3):
                dp.apply(1, V, out=out)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 20
            e0.record()
            for _ in range(reps):
                dp.apply(1, V, out=out)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / reps
            b = 12 * nnz + 4 * (p.n + 1) + 8 * p.n + 16 * p.n * k  # SURVEY 8(d) B_apply(k)
            print(f"spmm C4 k={k}: {us:.1f} us/apply  {b / us / 1e3:.0f} GB/s (B_apply = {b / 1e6:.1f} MB, L2-warm)")
        print("spmm done")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "lanczos")
