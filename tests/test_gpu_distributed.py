"""The sharded engine on real kernels: two ranks (gloo, both on cuda:0 -- the
test boxes have one GPU) run distributed.ShardedALS on nnz-balanced row shards
and all-gather after each half; the factors must equal the single-rank run bit
for bit (every row's solve is independent and deterministic)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SHAPE = (3000, 700, 90_000)  # m, n, ratings
F = 32
ITERS = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(rank, world, solver, peer=False):
    import paper_1808_03843_b200 as cmfb
    from paper_1808_03843_b200.distributed import ShardedALS
    torch.cuda.set_device(0)
    m, n, nnz = SHAPE
    train, _ = cmfb.gen_synthetic_device(m, n, F, nnz, 0.1, 0.1, seed=3)
    x = torch.from_numpy(cmfb.init_factors(m, F, 0.1, [0, 0])).cuda()
    th = torch.from_numpy(cmfb.init_factors(n, F, 0.1, [0, 1])).cuda()
    method, prec = {"cg16": ("cg", "fp16"), "exact": ("exact", "fp32")}[solver]
    eng = ShardedALS(train, F, lam=0.05, solver=cmfb.SolverConfig(method, precision=prec),
                     rank=rank, world=world)
    if peer:
        assert eng.attach_replicas(x, th) == (solver == "cg16")
    for _ in range(ITERS):
        eng.iteration(x, th)
    torch.cuda.synchronize()
    out = x.cpu().numpy(), th.cpu().numpy(), eng.local_rows()
    if peer:
        dist.barrier()  # nobody unmaps before every rank has read its factors
        eng.detach_replicas()
    return out


def _worker(rank, world, port, out, solver, peer=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, th, rows = _run(rank, world, solver, peer)
        np.savez(f"{out}_{rank}.npz", x=x, th=th, xr=rows["x"], tr=rows["t"])
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("solver,peer", [("cg16", False), ("exact", False), ("cg16", True)])
def test_two_rank_engine_equals_single_rank(tmp_path, solver, peer):
    """peer=True: the fused kernel stores each solved row into the other rank's
    replica through a CUDA-IPC mapping (cmf_fused_cg_update_peers) instead of
    an all-gather."""
    out = str(tmp_path / "r")
    mp.spawn(_worker, args=(2, _free_port(), out, solver, peer), nprocs=2, join=True)
    x1, th1, _ = _run(0, 1, solver)
    parts = [np.load(f"{out}_{r}.npz") for r in range(2)]
    assert parts[0]["xr"] > 0 and parts[1]["xr"] > 0  # both ranks solved rows
    for p in parts:  # every rank holds the full, identical factors
        assert np.array_equal(p["x"], x1)
        assert np.array_equal(p["th"], th1)
