"""cProfile of the public solve() at C4 from the host problem, 20 its
(the bench's e2e leg), after one warm-up solve.  Diagnostic."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11801_b200 import instances, solver as S  # noqa: E402

bc = instances.baseline_config("C4")
p = bc.problem
cfg = S.SolverConfig(rho=bc.rho, beta=bc.beta, k_c=bc.k_c, k_p=bc.k_p, sketch_rank=bc.sketch_rank, eps=1e-12,
                     max_iters=20, seed=bc.seed)
S.solve(p, cfg, callback=lambda i: i.y)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
S.solve(p, cfg, callback=lambda i: i.y)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(40)
