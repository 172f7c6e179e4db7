"""Per-iteration GPU timeline of the C2 solve (torch.profiler / CUPTI):
kernel time per name, GPU busy vs wall, i.e. how much of an outer iteration
is host-side gaps.  Not a benchmark (profiler overhead)."""
from __future__ import annotations

import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(name="C2", iters=30, skip=10):
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2312_11801_b200 import instances as inst, solver as S

    cfg_b = inst.baseline_config(name)
    cfg = S.SolverConfig(rho=cfg_b.rho, beta=cfg_b.beta, k_c=cfg_b.k_c, k_p=cfg_b.k_p, sketch_rank=cfg_b.sketch_rank,
                         eps=1e-12, max_iters=skip + iters, seed=cfg_b.seed)
    ds = S.DeviceSolver(cfg_b.problem, cfg)
    st0 = ds.cold_start()
    marks = {}

    def cb(info):
        if info.t == skip - 1:
            torch.cuda.synchronize()
            marks["t0"] = time.perf_counter()
            prof.start()
        if info.t == skip - 1 + iters:
            torch.cuda.synchronize()
            marks["t1"] = time.perf_counter()
            prof.stop()

    prof = profile(activities=[ProfilerActivity.CUDA], record_shapes=False)
    ds.solve(init=st0, callback=cb)
    wall = marks["t1"] - marks["t0"]
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    tot = {}
    spans = []
    for e in ev:
        nm = e.name.split("(")[0]
        d = e.time_range.end - e.time_range.start
        tot[nm] = tot.get(nm, 0.0) + d
        spans.append((e.time_range.start, e.time_range.end))
    spans.sort()
    busy, cur_s, cur_e = 0.0, None, None
    for s, e in spans:
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        busy += cur_e - cur_s
    print(f"{iters} iterations: wall {wall * 1e3 / iters:.3f} ms/it, GPU busy (union) {busy / 1e3 / iters:.3f} ms/it")
    # idle gaps between consecutive kernels (main + aux streams merged),
    # attributed to the (previous -> next) kernel pair
    evs = sorted(((e.time_range.start, e.time_range.end, e.name.split("(")[0]) for e in ev), key=lambda x: x[0])
    gaps, last_end, last_name = {}, None, None
    for st_, en_, nm in evs:
        if last_end is not None and st_ > last_end:
            key = (last_name[-28:], nm[-28:])
            gaps[key] = gaps.get(key, 0.0) + (st_ - last_end)
        if last_end is None or en_ > last_end:
            last_end, last_name = en_, nm
    print("  largest idle gaps (us/it): previous kernel -> next kernel")
    for (a_, b_), g in sorted(gaps.items(), key=lambda x: -x[1])[:12]:
        print(f"    {g / iters:8.1f}  {a_:>28s} -> {b_}")
    for nm, t in sorted(tot.items(), key=lambda x: -x[1])[:20]:
        print(f"  {t / 1e3 / iters:8.3f} ms/it  {nm}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C2", int(sys.argv[2]) if len(sys.argv) > 2 else 30,
         int(sys.argv[3]) if len(sys.argv) > 3 else 10)
