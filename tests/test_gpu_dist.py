"""GPU checks of the row-shard kernels (usbs_problem_create_shard, rectangular
operator apply) and of the host-driven sharded Lanczos / solve on one GPU
(world size 1), against the oracle and the persistent single-GPU path."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import cuda_ok
from helpers import random_graph
from oracle import usbs_cpu as O
from paper_2312_11801_b200 import instances as inst

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


def _sharded(p):
    from paper_2312_11801_b200.dist import Comm, ShardedDeviceProblem, Shard
    shard = Shard.balanced(p.cost.indptr, 1, 0)
    comm = Comm(1)
    return ShardedDeviceProblem(p, shard, comm), comm


def test_shard_problem_apply_matches_oracle():
    p = inst.maxcut_problem(inst.chung_lu(20000, seed=3))
    sdp, comm = _sharded(p)
    rt = sdp.rt
    rng = np.random.default_rng(3)
    y = rng.standard_normal(p.m) * 1e-3
    v = rng.standard_normal((p.n, 11))
    sdp.assemble(rt.upload(y))
    out = rt.download(sdp.apply(1, rt.upload(v)))
    want = O.slack_op(p, y).matmat(v)
    np.testing.assert_allclose(out, want, rtol=1e-12, atol=1e-13 * np.abs(want).max())


def test_sharded_lanczos_matches_oracle():
    from paper_2312_11801_b200.dist import lanczos_sharded
    from paper_2312_11801_b200.engine import Engine
    p = inst.baseline_config("C2").problem
    sdp, comm = _sharded(p)
    eng = Engine(sdp, comm)
    y = np.random.default_rng(4).standard_normal(p.m) * 1e-3
    sdp.assemble(sdp.rt.upload(y))
    r = lanczos_sharded(eng, sdp, 1, 10, seed=0)
    ro = O.lanczos(O.slack_op(p, y), 10, seed=0)
    assert abs(r.eigenvalues[0] - ro.eigenvalues[0]) <= 1e-11 * abs(ro.eigenvalues[0])
    assert r.restarts == ro.restarts and r.matvecs == ro.matvecs


def test_sharded_solve_matches_single_gpu_path():
    from paper_2312_11801_b200 import solver as S
    p = inst.maxcut_problem(random_graph(300, 0.05, 7))
    cfg = S.SolverConfig(sketch_rank=8, max_iters=12, seed=0)
    rec1 = []
    S.solve(p, cfg, callback=rec1.append)
    sdp, comm = _sharded(p)
    rec2 = []
    S.DeviceSolver(p, cfg, dprob=sdp, comm=comm).solve(callback=rec2.append)
    f1 = np.array([r.f_y for r in rec1])
    f2 = np.array([r.f_y for r in rec2])
    np.testing.assert_allclose(f2[:4], f1[:4], rtol=1e-8)
    assert len(f1) == len(f2)
    assert abs(f2[-1] - f1[-1]) <= 3e-2 * (1 + abs(f1[-1]))


class _FakeComm:
    """Two-rank stand-in on one GPU: the gathers return the global arrays the
    test provides, reductions stay local (the test compares per-rank partials)."""

    world = 2
    group = None

    def __init__(self, vfull):
        self.vfull = vfull

    def allreduce_sum(self, t):
        return t

    def allreduce_max(self, t):
        return t

    def allgather_rows(self, local, out, shard):
        out.copy_(self.vfull[:, : out.shape[1]])
        return out


@pytest.mark.parametrize("rank", [0, 1])
def test_entry_shard_kernels_with_ghosts(rank, monkeypatch):
    """One rank of a 2-way entry-family (C5) shard on one GPU: ghost duals
    through usbs_gather, the directed slack rows, and the owned-constraint
    image / compressed sums on the allgathered basis, against the oracle."""
    import paper_2312_11801_b200.dist as D
    from paper_2312_11801_b200.engine import Engine
    p = inst.correlation_problem(*inst.knn_correlation(n=400, clusters=12, dim=8, knn=6, seed=4))
    shard = D.Shard.balanced(p.cost.indptr, 2, rank)
    rng = np.random.default_rng(5)
    y = rng.standard_normal(p.m) * 1e-2
    v = rng.standard_normal((p.n, 7))
    owner = np.searchsorted(shard.bounds, _minrow(p), side="right") - 1
    ycat = y[np.argsort(owner, kind="stable")]
    from paper_2312_11801_b200.runtime import runtime
    rt = runtime()
    comm = _FakeComm(rt.upload(v))
    monkeypatch.setattr(D, "_allgather_var", lambda c, local, counts, out: out.copy_(rt.upload(ycat)))
    sdp = D.ShardedDeviceProblem(p, shard, comm)
    plan = sdp.plan
    if rank == 1:
        assert plan.ghost.size > 0  # edges from rank-0 rows: the ghost path is exercised
    sdp.assemble(rt.upload(y[plan.owned]))
    r0, r1 = shard.r0, shard.r1
    out = rt.download(sdp.apply(1, rt.upload(v[r0:r1])))
    want = (O.slack_op(p, y).matmat(v))[r0:r1]
    np.testing.assert_allclose(out, want, rtol=1e-12, atol=1e-12 * np.abs(want).max())
    eng = Engine(sdp, comm)
    k = v.shape[1]
    s = rng.standard_normal((k, k))
    s = s + s.T
    img = rt.download(eng.image(rt.upload(v[r0:r1]), rt.upload(s), rt.empty(plan.m_own)))
    want_img = O.image_lowrank(p.constraints, v, s)[plan.owned]
    np.testing.assert_allclose(img, want_img, rtol=1e-11, atol=1e-12 * np.abs(want_img).max())
    w = rng.standard_normal(p.m)
    d = k * (k + 1) // 2
    wo = rt.empty(d)
    eng.compressed(rt.upload(v[r0:r1]), w=rt.upload(w[plan.owned]), scale_w=1.0, w_out=wo)
    want_w = O.compressed(p.constraints, v)[plan.owned].T @ w[plan.owned]
    np.testing.assert_allclose(rt.download(wo), want_w, rtol=1e-10, atol=1e-11 * np.abs(want_w).max())


def _minrow(p):
    c = p.constraints
    mr = np.full(p.m, np.iinfo(np.int64).max, dtype=np.int64)
    np.minimum.at(mr, np.asarray(c.idx), np.asarray(c.rows))
    return mr


def test_entry_shard_solve_world1_matches_single_gpu():
    """An entry-family problem through the sharded device path (world 1):
    same trajectory as the single-GPU solver."""
    from paper_2312_11801_b200 import solver as S
    from paper_2312_11801_b200.dist import Comm, Shard, ShardedDeviceProblem
    p = inst.correlation_problem(*inst.knn_correlation(n=300, clusters=10, dim=8, knn=6, seed=4))
    cfg = S.SolverConfig(sketch_rank=6, k_c=6, k_p=0, max_iters=10, seed=0)
    rec1, rec2 = [], []
    S.solve(p, cfg, callback=rec1.append)
    sdp = ShardedDeviceProblem(p, Shard.balanced(p.cost.indptr, 1, 0), Comm(1))
    S.DeviceSolver(p, cfg, dprob=sdp, comm=Comm(1)).solve(callback=rec2.append)
    f1 = np.array([r.f_y for r in rec1])
    f2 = np.array([r.f_y for r in rec2])
    np.testing.assert_allclose(f2[:4], f1[:4], rtol=1e-8)
    assert [r.step for r in rec1] == [r.step for r in rec2]


class _ForcedComm:
    """A Comm whose collectives always go through torch.distributed (a
    one-rank NCCL group here), so the sharded Lanczos's allreduces and
    allgathers really run on NCCL."""

    def __init__(self):
        from paper_2312_11801_b200.dist import Comm
        self._c = Comm(2)  # world > 1: collectives issued
        self.world = 1     # but the engine treats it as the (single) rank's communicator
        self.group = None

    def allreduce_sum(self, t):
        import torch.distributed as dist
        dist.all_reduce(t)
        return t

    def allreduce_max(self, t):
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t

    def allgather_rows(self, local, out, shard):
        import torch.distributed as dist
        dist.all_gather_into_tensor(out, local.contiguous())
        return out


def test_sharded_lanczos_cycle_issues_no_host_sync():
    """within a restart cycle the sharded
    Lanczos enqueues SpMV, NCCL allgather / allreduces and the step epilogue
    without a synchronising call (torch sync-debug mode 'error' raises on any
    .item() / .cpu() / blocking copy); results equal the oracle's."""
    import os

    import torch
    import torch.distributed as dist

    from paper_2312_11801_b200.dist import ShardedDeviceProblem, Shard, lanczos_sharded
    from paper_2312_11801_b200.engine import Engine
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29617")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    p = inst.baseline_config("C4", small=True).problem
    shard = Shard.balanced(p.cost.indptr, 1, 0)
    comm = _ForcedComm()
    sdp = ShardedDeviceProblem(p, shard, comm)
    eng = Engine(sdp, None)
    eng.comm = comm  # collectives through NCCL
    y = np.random.default_rng(4).standard_normal(p.m) * 1e-3
    sdp.assemble(sdp.rt.upload(y))
    torch.cuda.synchronize()

    class Strict:
        def __enter__(self):
            torch.cuda.set_sync_debug_mode("error")

        def __exit__(self, *exc):
            torch.cuda.set_sync_debug_mode("default")

    with Strict():  # the guard does catch a synchronising call
        with pytest.raises(RuntimeError):
            torch.ones(1, device="cuda").item()
    r = lanczos_sharded(eng, sdp, 1, 10, seed=0, sync_guard=Strict)
    ro = O.lanczos(O.slack_op(p, y), 10, seed=0)
    assert r.restarts == ro.restarts and r.matvecs == ro.matvecs
    np.testing.assert_allclose(r.eigenvalues, ro.eigenvalues, rtol=1e-12)
