"""A few device USBS iterations of a BASELINE config (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_11801_b200 import instances, solver as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 2
bc = instances.baseline_config(name)
cfg = S.SolverConfig(rho=bc.rho, beta=bc.beta, k_c=bc.k_c, k_p=bc.k_p, sketch_rank=bc.sketch_rank, eps=1e-12,
                     max_iters=its, seed=bc.seed)
st, _ = S.solve(bc.problem, cfg)
print(name, "iterations", st.iterations, "f_y", st.f_y)
