"""Multi-rank host logic of the sharded driver (CPU, gloo, world_size 2).

The CUDA kernels cannot run here, so each rank solves its shard with the CPU
oracle (test-only) and the driver's own shard planning and RowGather assemble
the result.  Checks: shards are byte-exact slices whose concatenation is the
reference arrays, and the all-gathered half-update equals the single-process
update."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1808_03843_b200.distributed import RowGather, shard_bounds, shard_view


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _instance():
    from oracle import oracle as o
    t, _, _ = o.gen_synthetic(120, 70, 6, 0.2, 0.1, 5)
    r = o.build(t, 121, 70)  # one empty user row at the end
    theta = o.init_factors(70, 6, 0.1, [0, 1])
    x = o.init_factors(121, 6, 0.1, [0, 0])
    return o, r, theta, x


def test_shard_bounds_and_views_are_exact():
    o, r, _, _ = _instance()
    for world in (1, 2, 3, 4, 7):
        b = shard_bounds(r.row_ptr, world)
        assert b[0] == 0 and b[-1] == r.m and all(b[i] <= b[i + 1] for i in range(world))
        ptrs, idxs, vals = [], [], []
        for s in range(world):
            p, i, v = shard_view(r.row_ptr, r.col_idx, r.csr_val, b[s], b[s + 1])
            assert p[0] == 0 and p[-1] == len(i) == len(v)
            ptrs.append(p[1:] + (ptrs[-1][-1] if ptrs else 0))
            idxs.append(i)
            vals.append(v)
        assert np.array_equal(np.concatenate([[0]] + ptrs), r.row_ptr)
        assert np.array_equal(np.concatenate(idxs), r.col_idx)
        assert np.array_equal(np.concatenate(vals), r.csr_val)
        # nnz balance: no shard exceeds its share by more than one row's ratings
        share = r.nnz / world
        maxrow = int(np.diff(r.row_ptr).max())
        for s in range(world):
            assert r.row_ptr[b[s + 1]] - r.row_ptr[b[s]] <= share + maxrow


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o, r, theta, x = _instance()
    b = shard_bounds(r.row_ptr, world)
    lo, hi = b[rank], b[rank + 1]
    p, i, v = shard_view(r.row_ptr, r.col_idx, r.csr_val, lo, hi)
    local = x[lo:hi].copy()
    o.update_side((p, i, v, hi - lo, r.n), theta, local, 0.05, "cg", "fp32")
    full = torch.from_numpy(x.copy())
    full[lo:hi] = torch.from_numpy(local)
    RowGather(b, x.shape[1], torch.device("cpu"))(full, rank)
    if rank == 0:
        np.save(out_path, full.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_half_update_equals_single_process(tmp_path, world):
    out = str(tmp_path / "x.npy")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    o, r, theta, x = _instance()
    ref = x.copy()
    o.update_side(r.csr(), theta, ref, 0.05, "cg", "fp32")
    got = np.load(out)
    assert np.array_equal(got, ref)
    assert np.array_equal(got[120], x[120])  # the empty row is untouched
