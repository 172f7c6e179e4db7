"""Diagnostic: does the C2 solve depend on what ran before it in the process?"""
import sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2312_11801_b200 import instances as inst, solver as S
cb = inst.baseline_config("C2")
def run():
    cfg = S.SolverConfig(rho=cb.rho, beta=cb.beta, k_c=cb.k_c, k_p=cb.k_p, sketch_rank=cb.sketch_rank, eps=1e-3, max_iters=3000, seed=0)
    fs = []
    st, _ = S.solve(cb.problem, cfg, callback=lambda i: fs.append(i.f_y))
    return st.iterations, np.array(fs)
a = run()
# something else first: a C1 solve and a few C2 iterations with other settings
S.solve(inst.baseline_config("C1").problem, S.SolverConfig(k_c=10, k_p=1, eps=1e-3, max_iters=50, seed=3))
S.solve(cb.problem, S.SolverConfig(sketch_rank=10, eps=1e-12, max_iters=20, seed=5))
b = run()
n = min(len(a[1]), len(b[1]))
d = np.nonzero(a[1][:n] != b[1][:n])[0]
print("iterations", a[0], b[0], "first differing iteration:", d[0] if d.size else None)
