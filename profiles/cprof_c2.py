import cProfile, pstats, sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2312_11801_b200 import instances as inst, solver as S
cb = inst.baseline_config("C2")
cfg = S.SolverConfig(rho=cb.rho, beta=cb.beta, k_c=cb.k_c, k_p=cb.k_p, sketch_rank=cb.sketch_rank, eps=1e-12, max_iters=60, seed=0)
ds = S.DeviceSolver(cb.problem, cfg)
st0 = ds.cold_start()
S.DeviceSolver(cb.problem, S.SolverConfig(rho=cb.rho, beta=cb.beta, k_c=cb.k_c, k_p=cb.k_p, sketch_rank=cb.sketch_rank, eps=1e-12, max_iters=5, seed=0)).solve()
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
ds.solve(init=st0)
pr.disable()
torch.cuda.synchronize()
print("wall per it ms", (time.perf_counter() - t0) / 60 * 1e3)
ps = pstats.Stats(pr).sort_stats("tottime")
ps.sort_stats("cumulative").print_stats(40)
