"""Diagnostic: C2 to 1e-3 through S.solve versus DeviceSolver.cold_start + solve(init)."""
import sys
sys.path.insert(0, "/root/repo")
from paper_2312_11801_b200 import instances as inst, solver as S
cb = inst.baseline_config("C2")
mk = lambda: S.SolverConfig(rho=cb.rho, beta=cb.beta, k_c=cb.k_c, k_p=cb.k_p, sketch_rank=cb.sketch_rank, eps=1e-3, max_iters=3000, seed=0)
st, _ = S.solve(cb.problem, mk())
print("S.solve", st.iterations)
ds = S.DeviceSolver(cb.problem, mk())
st0 = ds.cold_start()
st, _ = ds.solve(init=st0)
print("cold_start + solve(init)", st.iterations)
ds = S.DeviceSolver(cb.problem, mk())
ds.lz_probe = []
st, _ = ds.solve()
print("lz_probe", st.iterations)
