"""Streaming synthetic generator (csrc/gen.cu): the device CSR/CSC
shards equal the oracle's data.build (data.py:205-249) of the triples the
numpy restatement of the generator writes, byte for byte; shards of any split
tile the global arrays; the held-out triples match."""
import numpy as np
import pytest
import torch

import paper_1808_03843_b200 as cmfb

pytestmark = pytest.mark.gpu

KEYS = ("row_ptr", "col_idx", "csr_val", "col_ptr", "row_idx", "csc_val")


@pytest.mark.parametrize("m,n,f,nnz,seed", [(300, 200, 16, 9000, 0), (517, 1031, 13, 40_000, 7),
                                            (64, 3000, 100, 20_000, 3)])
def test_stream_generator_matches_oracle_build(oracle, cuda_device, m, n, f, nnz, seed):
    thr_c, thr_t, scale = cmfb.stream_params(m, n, nnz, 0.1, 0.1)
    tr, te, X, T = oracle.gen_stream_triples(seed, m, n, f, thr_c, thr_t, scale)
    perm = np.random.default_rng(1).permutation(len(tr))  # any file order builds the same arrays
    ref = oracle.build(oracle.OTriples(tr.user[perm], tr.item[perm], tr.rating[perm]), m, n)
    dr, test = cmfb.gen_synthetic_stream(m, n, f, nnz, 0.1, 0.1, seed)
    for k in KEYS:
        a, b = getattr(dr, k).cpu().numpy(), getattr(ref, k)
        assert a.dtype == b.dtype and np.array_equal(a, b), k
    assert abs(dr.nnz - nnz) < 6 * np.sqrt(nnz)
    order = np.lexsort((test.item.cpu().numpy(), test.user.cpu().numpy()))
    for got, want in ((test.user, te.user), (test.item, te.item), (test.rating, te.rating)):
        assert np.array_equal(got.cpu().numpy()[order], want)
    sh = cmfb.gen_stream_shard(m, n, f, nnz, 0.1, 0.1, seed)
    assert np.array_equal(sh.x_true.cpu().numpy(), X) and np.array_equal(sh.t_true.cpu().numpy(), T)


def test_stream_shards_tile_the_matrix(cuda_device):
    m, n, f, nnz = 1000, 700, 24, 60_000
    full, test = cmfb.gen_synthetic_stream(m, n, f, nnz, 0.1, 0.1, 5)
    world = 3
    ub = [s * m // world for s in range(world + 1)]
    vb = [s * n // world for s in range(world + 1)]
    rows, cols, tests = [], [], 0
    for s in range(world):
        sh = cmfb.gen_stream_shard(m, n, f, nnz, 0.1, 0.1, 5, users=(ub[s], ub[s + 1]), items=(vb[s], vb[s + 1]))
        rp, ci, cv = sh.x_view
        assert torch.equal(rp, full.row_ptr[ub[s]:ub[s + 1] + 1] - full.row_ptr[ub[s]])
        assert torch.equal(ci, full.col_idx[full.row_ptr[ub[s]]:full.row_ptr[ub[s + 1]]])
        assert torch.equal(cv, full.csr_val[full.row_ptr[ub[s]]:full.row_ptr[ub[s + 1]]])
        cp, ri, rv = sh.t_view
        assert torch.equal(cp, full.col_ptr[vb[s]:vb[s + 1] + 1] - full.col_ptr[vb[s]])
        assert torch.equal(ri, full.row_idx[full.col_ptr[vb[s]]:full.col_ptr[vb[s + 1]]])
        assert torch.equal(rv, full.csc_val[full.col_ptr[vb[s]]:full.col_ptr[vb[s + 1]]])
        tests += len(sh.test)
    assert tests == len(test)


def test_stream_generator_trains(cuda_device):
    """A generated matrix is a valid ALS input: CG training lowers the test RMSE."""
    m, n, f = 2000, 1500, 16
    dr, test = cmfb.gen_synthetic_stream(m, n, f, 200_000, 0.1, 0.1, 2)
    cfg = cmfb.AlsConfig(f=f, lam=0.05, epochs=4, solver=cmfb.SolverConfig("cg", precision="fp16"))
    _, _, rep = cmfb.train(dr, test, cfg)
    r = [e.rmse for e in rep.epochs]
    assert r[-1] < r[0]
