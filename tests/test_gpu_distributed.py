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


def _run(rank, world, solver, peer=False, per_rank=False):
    import paper_1808_03843_b200 as cmfb
    from paper_1808_03843_b200.distributed import ShardedALS, ShardedRatings, shard_ratings
    torch.cuda.set_device(0)
    m, n, nnz = SHAPE
    if per_rank == "stream":
        # the streaming generator: each rank generates only its CSR rows / CSC columns
        ub = [s * m // world for s in range(world + 1)]
        vb = [s * n // world for s in range(world + 1)]
        sh = cmfb.gen_stream_shard(m, n, F, nnz, 0.1, 0.1, 3, users=(ub[rank], ub[rank + 1]),
                                   items=(vb[rank], vb[rank + 1]))
        if world == 1:
            train = cmfb.DeviceRatings(m, n, int(sh.x_view[1].numel()), *sh.x_view, *sh.t_view)
        else:
            tot = torch.tensor([sh.x_view[1].numel()], dtype=torch.int64)
            dist.all_reduce(tot)
            train = ShardedRatings(m, n, int(tot.item()), ub, vb, sh.x_view, sh.t_view)
    elif per_rank:
        # reference protocol on the host, each rank builds only its shards
        t, _ = cmfb.gen_synthetic(m, n, F, nnz / (m * n), 0.1, 3)
        train = shard_ratings(t, m, n, rank, world)
    else:
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


def _worker(rank, world, port, out, solver, peer=False, per_rank=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, th, rows = _run(rank, world, solver, peer, per_rank)
        np.savez(f"{out}_{rank}.npz", x=x, th=th, xr=rows["x"], tr=rows["t"])
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("solver,peer,per_rank", [("cg16", False, False), ("exact", False, False),
                                                  ("cg16", True, False), ("cg16", True, True),
                                                  ("cg16", True, "stream"), ("exact", False, "stream")])
def test_two_rank_engine_equals_single_rank(tmp_path, solver, peer, per_rank):
    """peer=True: the fused kernel stores each solved row into the other rank's
    replica through a CUDA-IPC mapping (cmf_fused_cg_update_peers) instead of
    an all-gather.  per_rank=True: each rank builds only its own shards from the
    host triples (distributed.shard_ratings); "stream": each rank generates only
    its own shards (gen_stream_shard, row-balanced ranges)."""
    out = str(tmp_path / "r")
    mp.spawn(_worker, args=(2, _free_port(), out, solver, peer, per_rank), nprocs=2, join=True)
    x1, th1, _ = _run(0, 1, solver, per_rank=per_rank)
    parts = [np.load(f"{out}_{r}.npz") for r in range(2)]
    assert parts[0]["xr"] > 0 and parts[1]["xr"] > 0  # both ranks solved rows
    for p in parts:  # every rank holds the full, identical factors
        assert np.array_equal(p["x"], x1)
        assert np.array_equal(p["th"], th1)


def test_per_rank_shards_concatenate_to_build(cuda_device):
    """shard_ratings for k ranks: the CSR / CSC slices each rank builds on its
    own concatenate to the single-device build byte for byte (incl. duplicate
    triples, last wins, and empty rows)."""
    import paper_1808_03843_b200 as cmfb
    from paper_1808_03843_b200.distributed import shard_ratings
    rng = np.random.default_rng(11)
    m, n, k = 500, 300, 20_000
    u = rng.integers(0, m - 3, k)
    v = rng.integers(0, n, k)
    t = cmfb.Triples(u, v, rng.standard_normal(k).astype(np.float32))
    full = cmfb.build(t, m, n)
    for world in (1, 2, 3, 5):
        parts = [shard_ratings(t, m, n, r, world) for r in range(world)]
        for side, ref in (("x_view", (full.row_ptr, full.col_idx, full.csr_val)),
                          ("t_view", (full.col_ptr, full.row_idx, full.csc_val))):
            ptrs, idxs, vals = [], [], []
            for p in parts:
                ptr, idx, val = (a.cpu().numpy() for a in getattr(p, side))
                ptrs.append(ptr[1:] + (ptrs[-1][-1] if ptrs else 0))
                idxs.append(idx)
                vals.append(val)
            assert np.array_equal(np.concatenate([[0]] + ptrs), ref[0])
            assert np.array_equal(np.concatenate(idxs), ref[1])
            assert np.array_equal(np.concatenate(vals).view(np.uint32), ref[2].view(np.uint32))


def _run_rs(rank, world):
    """The reduce-scatter exchange (distributed.ReduceScatterALS) on streamed
    shards: X stays sharded, partial item Grams are summed across ranks."""
    import paper_1808_03843_b200 as cmfb
    from paper_1808_03843_b200.distributed import ReduceScatterALS
    torch.cuda.set_device(0)
    m, n, nnz = SHAPE
    ub = [s * m // world for s in range(world + 1)]
    sh = cmfb.gen_stream_shard(m, n, F, nnz, 0.1, 0.1, 3, users=(ub[rank], ub[rank + 1]), local_csc=True)
    eng = ReduceScatterALS(sh, F, lam=0.05, solver=cmfb.SolverConfig("cg", precision="fp16"), rank=rank,
                           world=world)
    x = torch.from_numpy(cmfb.init_factors(m, F, 0.1, [0, 0])).cuda()[ub[rank]:ub[rank + 1]].contiguous()
    th = torch.from_numpy(cmfb.init_factors(n, F, 0.1, [0, 1])).cuda()
    for _ in range(ITERS):
        eng.iteration(x, th)
    eng.check()
    torch.cuda.synchronize()
    te = sh.test
    local = cmfb.Triples(te.user - ub[rank], te.item, te.rating)
    sse = cmfb.rmse(x, th, local) ** 2 * len(te)
    return x.cpu().numpy(), th.cpu().numpy(), sse, len(te)


def _worker_rs(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, th, sse, cnt = _run_rs(rank, world)
        np.savez(f"{out}_{rank}.npz", x=x, th=th, sse=sse, cnt=cnt)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_reduce_scatter_exchange(tmp_path):
    """world = 1: the reduce-scatter route (pass 1 -> partial -> pass 2) equals
    the replicated engine bit for bit (the partial is the full fp32
    accumulator).  world = 2 (gloo, one device): X sharded, partial item Grams
    summed across ranks -- same factors up to fp32 summation order and the same
    test RMSE to 1e-6."""
    import paper_1808_03843_b200 as cmfb
    from paper_1808_03843_b200.distributed import ShardedALS
    m, n, nnz = SHAPE
    x1, th1, sse1, cnt1 = _run_rs(0, 1)
    # the replicated single-rank engine on the same matrix
    full, _ = cmfb.gen_synthetic_stream(m, n, F, nnz, 0.1, 0.1, 3)
    eng = ShardedALS(full, F, lam=0.05, solver=cmfb.SolverConfig("cg", precision="fp16"))
    x = torch.from_numpy(cmfb.init_factors(m, F, 0.1, [0, 0])).cuda()
    th = torch.from_numpy(cmfb.init_factors(n, F, 0.1, [0, 1])).cuda()
    for _ in range(ITERS):
        eng.iteration(x, th)
    assert np.array_equal(x.cpu().numpy(), x1) and np.array_equal(th.cpu().numpy(), th1)
    out = str(tmp_path / "rs")
    mp.spawn(_worker_rs, args=(2, _free_port(), out), nprocs=2, join=True)
    parts = [np.load(f"{out}_{r}.npz") for r in range(2)]
    x2 = np.concatenate([p["x"] for p in parts])
    assert np.array_equal(parts[0]["th"], parts[1]["th"])
    rel = np.linalg.norm(x2 - x1) / np.linalg.norm(x1)
    assert rel < 1e-4, rel
    rmse1 = np.sqrt(sse1 / cnt1)
    rmse2 = np.sqrt(sum(float(p["sse"]) for p in parts) / sum(int(p["cnt"]) for p in parts))
    assert abs(rmse2 - rmse1) < 1e-6
