import sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2312_11801_b200 import instances as inst, solver as S
cb = inst.baseline_config("C2")
res = []
for rep in range(3):
    cfg = S.SolverConfig(rho=cb.rho, beta=cb.beta, k_c=cb.k_c, k_p=cb.k_p, sketch_rank=cb.sketch_rank, eps=1e-3, max_iters=3000, seed=0)
    fs = []
    st, _ = S.solve(cb.problem, cfg, callback=lambda i: fs.append(i.f_y))
    res.append((st.iterations, np.array(fs)))
    print(rep, st.iterations, repr(fs[-1]))
for rep in range(1, 3):
    n = min(len(res[0][1]), len(res[rep][1]))
    d = np.nonzero(res[0][1][:n] != res[rep][1][:n])[0]
    print("first differing iteration vs run 0:", d[0] if d.size else None)
