import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2312_11801_b200 import instances
from paper_2312_11801_b200.runtime import DeviceProblem, runtime
cfg_b = instances.baseline_config("C4")
p = cfg_b.problem
rt = runtime()
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    dp = DeviceProblem(p, rt)
    torch.cuda.synchronize()
    print("rep", rep, "DeviceProblem %.1f ms" % ((time.perf_counter() - t) * 1e3), flush=True)
    t = time.perf_counter(); dp.lanczos_plan(32); torch.cuda.synchronize()
    print("   lanczos_plan %.1f ms" % ((time.perf_counter() - t) * 1e3), flush=True)
    del dp
