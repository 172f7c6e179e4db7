"""Row-sharded (multi-GPU) host logic under a world_size-2 gloo group on CPU.

The device kernels are replaced by the numpy engine of tests/cpu_backend.py;
what is tested is the sharding itself: the row partition, which reductions
are allreduced, the gathers before each SpMV, the replicated k x k work and
the distributed Lanczos -- against the single-process CPU oracle."""
from __future__ import annotations

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import random_graph
from oracle import usbs_cpu as O
from paper_2312_11801_b200 import instances as inst


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(kind="maxcut"):
    if kind == "entries":  # correlation SDP: diag equalities + edge inequalities (C5 family)
        return inst.correlation_problem(*inst.knn_correlation(n=90, clusters=6, dim=8, knn=5, seed=4))
    return inst.maxcut_problem(random_graph(120, 0.08, 3))


def _minrow(p):
    c = p.constraints
    mr = np.full(p.m, np.iinfo(np.int64).max, dtype=np.int64)
    np.minimum.at(mr, np.asarray(c.idx), np.asarray(c.rows))
    return mr


def _worker(rank, world, port, outdir, what):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(__file__))
        from cpu_backend import CpuEngine, CpuRuntime, CpuShardProblem
        from paper_2312_11801_b200.dist import Comm, Shard, lanczos_sharded
        from paper_2312_11801_b200.solver import DeviceSolver, SolverConfig

        p = _problem("entries" if what == "solve_entries" else "maxcut")
        shard = Shard.balanced(p.cost.indptr, world, rank)
        comm = Comm(world)
        rt = CpuRuntime()
        dp = CpuShardProblem(p, shard, comm, rt)
        eng = CpuEngine(dp, comm)
        if what == "lanczos":
            y = np.random.default_rng(9).standard_normal(p.m) * 1e-2
            dp.assemble(rt.upload(y[shard.r0:shard.r1]))
            r = lanczos_sharded(eng, dp, 1, 6, seed=0)
            full = torch.empty(p.n, 6, dtype=torch.float64)
            comm.allgather_rows(r.eigenvectors_dev, full, shard)
            np.savez(os.path.join(outdir, f"r{rank}.npz"), vals=r.eigenvalues, vecs=full.numpy(),
                     meta=np.array([r.restarts, r.matvecs, int(r.converged)]))
        else:
            cfg = SolverConfig(sketch_rank=5, max_iters=8, seed=0)
            ds = DeviceSolver(p, cfg, dprob=dp, comm=comm, engine=eng)
            rec = []
            st, out = ds.solve(callback=rec.append)
            if what == "solve_entries":  # owned duals back to global constraint order
                from paper_2312_11801_b200.dist import _allgather_var
                cat = torch.zeros(p.m, dtype=torch.float64)
                _allgather_var(comm, st.y_dev, dp.plan.counts, cat)
                order = np.argsort(np.searchsorted(shard.bounds, _minrow(p), side="right") - 1, kind="stable")
                yg = np.empty(p.m)
                yg[order] = cat.numpy()
                yfull = torch.from_numpy(yg).view(-1, 1)
            else:
                yfull = torch.empty(p.n, 1, dtype=torch.float64)
                comm.allgather_rows(st.y_dev.view(-1, 1), yfull, shard)
            np.savez(os.path.join(outdir, f"r{rank}.npz"), f_y=np.array([r.f_y for r in rec]),
                     f_cand=np.array([r.f_cand for r in rec]), model_val=np.array([r.model_val for r in rec]),
                     steps=np.array([r.step == "descent" for r in rec]), y=yfull.numpy().ravel(), lams=out.lams,
                     bounds=shard.bounds)
    finally:
        dist.destroy_process_group()


def _run(what):
    outdir = tempfile.mkdtemp()
    mp.spawn(_worker, args=(2, _free_port(), outdir, what), nprocs=2, join=True)
    return [dict(np.load(os.path.join(outdir, f"r{r}.npz"))) for r in range(2)]


def test_shard_partition_balanced():
    from paper_2312_11801_b200.dist import Shard
    p = inst.maxcut_problem(inst.chung_lu(5000, seed=3))
    nnz = np.diff(p.cost.indptr)
    for world in (2, 4, 8):
        s = Shard.balanced(p.cost.indptr, world, 0)
        assert s.bounds[0] == 0 and s.bounds[-1] == p.n and np.all(np.diff(s.bounds) > 0)
        loads = [nnz[s.bounds[i]:s.bounds[i + 1]].sum() + 4 * (s.bounds[i + 1] - s.bounds[i]) for i in range(world)]
        assert max(loads) <= 1.25 * (sum(loads) / world) + nnz.max()


def test_sharded_lanczos_gloo_world2():
    res = _run("lanczos")
    p = _problem()
    y = np.random.default_rng(9).standard_normal(p.m) * 1e-2
    ro = O.lanczos(O.slack_op(p, y), 6, seed=0)
    for r in res:
        np.testing.assert_allclose(r["vals"], ro.eigenvalues, rtol=1e-10, atol=1e-12)
        assert int(r["meta"][0]) == ro.restarts and int(r["meta"][1]) == ro.matvecs
        pe = np.linalg.norm(r["vecs"] @ r["vecs"].T - ro.eigenvectors @ ro.eigenvectors.T)
        assert pe <= 1e-7
    np.testing.assert_array_equal(res[0]["vals"], res[1]["vals"])  # replicated results identical


def test_sharded_solve_gloo_world2():
    res = _run("solve")
    p = _problem()
    rec = []
    ost, oout = O.solve(p, O.Config(sketch_rank=5, max_iters=8, seed=0), callback=rec.append)
    f_y = np.array([r.f_y for r in rec])
    for r in res:
        np.testing.assert_allclose(r["f_y"][:4], f_y[:4], rtol=1e-8)
        np.testing.assert_array_equal(r["steps"][:4], [x.step == "descent" for x in rec][:4])
        assert len(r["f_y"]) == len(f_y)
        np.testing.assert_allclose(r["f_y"][-1], f_y[-1], rtol=1e-3)
    np.testing.assert_array_equal(res[0]["f_y"], res[1]["f_y"])  # every rank took the same decisions
    np.testing.assert_array_equal(res[0]["y"], res[1]["y"])


def test_entry_shard_plan_covers_every_entry():
    """Every entry lands on the owners of its rows exactly once per half, the
    owned sets partition the constraints, ghosts point at their owners."""
    from paper_2312_11801_b200.dist import EntryShardPlan, Shard
    p = _problem("entries")
    c = p.constraints
    world = 3
    plans = [EntryShardPlan(p, Shard.balanced(p.cost.indptr, world, r)) for r in range(world)]
    owned = np.concatenate([pl.owned for pl in plans])
    assert np.array_equal(np.sort(owned), np.arange(p.m))
    halves = sum(pl.d_vals.size for pl in plans)
    assert halves == c.vals.size + int(np.sum(np.asarray(c.rows) != np.asarray(c.cols)))
    cat = np.concatenate([pl.owned for pl in plans])
    for pl in plans:
        np.testing.assert_array_equal(cat[pl.ghost_pos], pl.ghost)
        assert pl.o_vals.size == int(np.isin(np.asarray(c.idx), pl.owned).sum())


def test_sharded_entry_solve_gloo_world2():
    """C5-family (entry constraints with inequalities) row-sharded over two
    gloo ranks: the first iterations match the single-process oracle, all
    decisions identical, both ranks bit-identical."""
    res = _run("solve_entries")
    p = _problem("entries")
    rec = []
    ost, oout = O.solve(p, O.Config(sketch_rank=5, max_iters=8, seed=0), callback=rec.append)
    f_y = np.array([r.f_y for r in rec])
    for r in res:
        np.testing.assert_allclose(r["f_y"][:4], f_y[:4], rtol=1e-8)
        np.testing.assert_array_equal(r["steps"], [x.step == "descent" for x in rec])
        assert len(r["f_y"]) == len(f_y)
        np.testing.assert_allclose(r["f_y"][-1], f_y[-1], rtol=1e-6)
        np.testing.assert_allclose(r["y"], ost.y, rtol=1e-5, atol=1e-8 * np.abs(ost.y).max())
    np.testing.assert_array_equal(res[0]["f_y"], res[1]["f_y"])
    np.testing.assert_array_equal(res[0]["y"], res[1]["y"])
