"""CSR/CSC construction on the device (cmf_build, build.cu) vs the oracle's
restatement of data.build (data.py:205-249) -- bit-exact, per SURVEY 8(a13).

Edge cases the reference's own build tests cover (tests/test_data.py::TestBuild):
duplicates collapse to the LAST occurrence in file order, empty rows and columns,
no triples at all, the first out-of-range triple named in DataError, m/n
defaulting to max id + 1.  Plus the radix sort's own edges: more than one
8-bit pass, more than one 4096-key tile per digit run, 1-row / 1-column
matrices, int32 ids.
"""
import numpy as np
import pytest
import torch

import paper_1808_03843_b200 as cmfb
from paper_1808_03843_b200 import _native as nat

pytestmark = pytest.mark.gpu

KEYS = ("row_ptr", "col_idx", "csr_val", "col_ptr", "row_idx", "csc_val")


def _same(ours, ref, tag=""):
    assert ours.m == ref.m and ours.n == ref.n and ours.nnz == ref.nnz, tag
    for k in KEYS:
        a, b = getattr(ours, k), getattr(ref, k)
        assert a.dtype == b.dtype and np.array_equal(a, b), (tag, k)


def _triples(rng, k, m, n, dup_frac=0.0):
    u = rng.integers(0, m, size=k, dtype=np.int64)
    v = rng.integers(0, n, size=k, dtype=np.int64)
    if dup_frac > 0:  # re-use earlier (user, item) pairs at later file positions
        nd = int(dup_frac * k)
        src = rng.integers(0, k, size=nd)
        dst = rng.integers(0, k, size=nd)
        u[dst], v[dst] = u[src], v[src]
    r = rng.standard_normal(k).astype(np.float32)
    return u, v, r


@pytest.mark.parametrize("k,m,n,dup", [
    (1, 1, 1, 0.0),
    (37, 5, 7, 0.5),             # tiny, heavy duplicates
    (5000, 1, 9000, 0.1),        # one row: every key in one digit run
    (5000, 9000, 1, 0.1),        # one column: CSC bits = 0
    (200_000, 3000, 70_000, 0.05),   # 28-bit keys: four passes, many tiles
    (300_000, 480, 178, 0.0),    # dense-ish small matrix, long runs per digit
    (1_000_000, 48_019, 17_770, 0.01),
])
def test_build_matches_oracle(oracle, cuda_device, k, m, n, dup):
    rng = np.random.default_rng(k + m + n)
    u, v, r = _triples(rng, k, m, n, dup)
    ref = oracle.build(oracle.OTriples(u, v, r), m, n)
    _same(cmfb.build(cmfb.Triples(u, v, r), m, n), ref, (k, m, n))


def test_build_last_occurrence_wins(cuda_device):
    t = [(1, 2, 1.0), (0, 0, 5.0), (1, 2, 2.0), (0, 0, 6.0), (1, 2, 3.0)]
    sr = cmfb.build(t, 2, 3)
    assert sr.nnz == 2
    assert sr.row_ptr.tolist() == [0, 1, 2]
    assert sr.col_idx.tolist() == [0, 2] and sr.csr_val.tolist() == [6.0, 3.0]
    assert sr.col_ptr.tolist() == [0, 1, 1, 2]
    assert sr.row_idx.tolist() == [0, 1] and sr.csc_val.tolist() == [6.0, 3.0]


def test_build_defaults_and_empty(oracle, cuda_device):
    rng = np.random.default_rng(3)
    u, v, r = _triples(rng, 1000, 77, 55)
    sr = cmfb.build(cmfb.Triples(u, v, r))
    _same(sr, oracle.build(oracle.OTriples(u, v, r), int(u.max()) + 1, int(v.max()) + 1))
    e = cmfb.build(cmfb.Triples(np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0, np.float32)), 4, 3)
    assert e.nnz == 0 and e.row_ptr.tolist() == [0] * 5 and e.col_ptr.tolist() == [0] * 4
    e0 = cmfb.build(cmfb.Triples(np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0, np.float32)))
    assert (e0.m, e0.n, e0.nnz) == (0, 0, 0)


def test_build_names_first_bad_triple(cuda_device):
    t = [(0, 0, 1.0), (2, 9, 4.5), (3, 0, 2.0), (-1, 0, 1.0)]
    with pytest.raises(cmfb.DataError, match=r"triple \(2, 9, 4\.5\) out of range for a 3x5 matrix"):
        cmfb.build(t, 3, 5)
    with pytest.raises(cmfb.DataError, match=r"\(-1, 0, 1\.0\)"):
        cmfb.build([(0, 0, 1.0), (-1, 0, 1.0)], 3, 5)


def test_build_device_int32_ids_and_determinism(oracle, cuda_device):
    """The C ABI takes int32 ids too; two builds of the same triples are bitwise equal."""
    rng = np.random.default_rng(11)
    k, m, n = 400_000, 20_000, 5_000
    u, v, r = _triples(rng, k, m, n, 0.02)
    ref = oracle.build(oracle.OTriples(u, v, r), m, n)
    ud, vd = torch.from_numpy(u.astype(np.int32)).cuda(), torch.from_numpy(v.astype(np.int32)).cuda()
    rd = torch.from_numpy(r).cuda()
    import ctypes
    ws = torch.empty(int(nat.lib().cmf_build_workspace_bytes(k)), dtype=torch.uint8, device="cuda")
    outs = []
    for _ in range(2):
        mn = (ctypes.c_int64 * 2)(m, n)
        rp = torch.empty(m + 1, dtype=torch.int64, device="cuda")
        cp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        ci, ri = (torch.empty(k, dtype=torch.int32, device="cuda") for _ in range(2))
        cv, rv = (torch.empty(k, dtype=torch.float32, device="cuda") for _ in range(2))
        nnz, bad = ctypes.c_int64(0), ctypes.c_int64(0)
        nat.call("cmf_build", nat.ptr(ud), nat.ptr(vd), 0, nat.ptr(rd), k, mn, nat.ptr(rp), nat.ptr(ci),
                 nat.ptr(cv), nat.ptr(cp), nat.ptr(ri), nat.ptr(rv), nat.ptr(ws), ws.numel(),
                 ctypes.byref(nnz), ctypes.byref(bad), nat.stream_ptr())
        z = nnz.value
        assert z == ref.nnz and bad.value == -1
        got = dict(row_ptr=rp, col_idx=ci[:z], csr_val=cv[:z], col_ptr=cp, row_idx=ri[:z], csc_val=rv[:z])
        for key in KEYS:
            assert np.array_equal(got[key].cpu().numpy(), getattr(ref, key)), key
        outs.append([got[key].cpu().numpy() for key in KEYS])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


def test_build_netflix_shape_properties(cuda_device):
    """BASELINE configs[2] scale (99M ratings), size-independent properties:
    sorted rows/columns, pointer arrays consistent, CSC a permutation of CSR
    (checksums of (row, col, value) agree), no duplicates."""
    train, _ = cmfb.gen_synthetic_device(480_189, 17_770, 100, 99_000_000, 0.1, 0.1, seed=0)
    trip_u = torch.repeat_interleave(torch.arange(train.m, device="cuda"), torch.diff(train.row_ptr))
    trip_v = train.col_idx.long()
    # rebuild from the triples in a shuffled file order: same arrays
    perm = torch.randperm(train.nnz, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    sr = cmfb.data.build_device(cmfb.Triples(trip_u[perm], trip_v[perm], train.csr_val[perm]), train.m, train.n)
    for key in KEYS:
        assert torch.equal(getattr(sr, key), getattr(train, key)), key
    key = trip_u * train.n + trip_v
    assert bool((key[1:] > key[:-1]).all())
