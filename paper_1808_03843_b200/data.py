"""Rating data: triples, the paired CSR/CSC structure, and the synthetic
generators the benchmark protocol uses.

Mirrors the reference's data.py (Triples, RowView, SparseRatings, build,
split_holdout, gen_synthetic; data.py:52-130, :205-302).  ``build`` runs on the
GPU (stable device sorts + bincount scans) and is bit-identical to the
reference's lexsort/bincount construction: the CSR order is (user, item,
position) with the LAST duplicate kept, the CSC order is (item, user).
``gen_synthetic``/``split_holdout`` keep the reference's numpy PCG64 draw
sequence (identical inputs are part of the parity contract), while
``gen_synthetic_device`` is the fast on-GPU generator used for benchmark
shapes that the reference generator cannot reach (Netflix and up).

A ``DeviceRatings`` holds the same six arrays as CUDA tensors; it is what the
training loop keeps resident in HBM.
"""

from __future__ import annotations

import ctypes
import math
import struct
from dataclasses import dataclass
from typing import Iterable, NamedTuple

import numpy as np
import torch

from . import _native as nat
from .errors import DataError, FormatError, ParseError
from .factors import predict_pairs


class RatingTriple(NamedTuple):
    user: int
    item: int
    rating: float


@dataclass
class Triples:
    """Flat (user, item, rating) arrays in file order (int64, int64, float32)."""

    user: object
    item: object
    rating: object

    @classmethod
    def from_iter(cls, triples: Iterable) -> "Triples":
        rows = list(triples)
        u = np.array([t[0] for t in rows], dtype=np.int64)
        v = np.array([t[1] for t in rows], dtype=np.int64)
        r = np.array([t[2] for t in rows], dtype=np.float32)
        return cls(u, v, r)

    def __len__(self):
        return int(self.user.shape[0])

    def __getitem__(self, i):
        return RatingTriple(int(self.user[i]), int(self.item[i]), float(self.rating[i]))

    def __iter__(self):
        for k in range(len(self)):
            yield self[k]

    def to_device(self) -> "Triples":
        return Triples(nat.to_dev(self.user, torch.int64), nat.to_dev(self.item, torch.int64),
                       nat.to_dev(self.rating, torch.float32))


class RowView(NamedTuple):
    """One orientation of the rating matrix (data.py:79-86)."""

    indptr: object
    indices: object
    values: object
    nrows: int
    ncols: int


@dataclass(frozen=True)
class SparseRatings:
    """Host copy of the paired CSR + CSC structure (data.py:89-130)."""

    m: int
    n: int
    nnz: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    csr_val: np.ndarray
    col_ptr: np.ndarray
    row_idx: np.ndarray
    csc_val: np.ndarray

    def csr_view(self) -> RowView:
        return RowView(self.row_ptr, self.col_idx, self.csr_val, self.m, self.n)

    def csc_view(self) -> RowView:
        return RowView(self.col_ptr, self.row_idx, self.csc_val, self.n, self.m)

    def row(self, u: int):
        lo, hi = int(self.row_ptr[u]), int(self.row_ptr[u + 1])
        return self.col_idx[lo:hi], self.csr_val[lo:hi]

    def col(self, v: int):
        lo, hi = int(self.col_ptr[v]), int(self.col_ptr[v + 1])
        return self.row_idx[lo:hi], self.csc_val[lo:hi]

    def to_triples(self) -> Triples:
        users = np.repeat(np.arange(self.m, dtype=np.int64), np.diff(self.row_ptr))
        return Triples(users, self.col_idx.astype(np.int64), self.csr_val.copy())

    @property
    def nbytes(self) -> int:
        return int(sum(getattr(self, k).nbytes for k in _ARRAYS))

    def to_device(self) -> "DeviceRatings":
        dt = {"row_ptr": torch.int64, "col_ptr": torch.int64, "col_idx": torch.int32,
              "row_idx": torch.int32, "csr_val": torch.float32, "csc_val": torch.float32}
        return DeviceRatings(self.m, self.n, self.nnz,
                             **{k: nat.to_dev(getattr(self, k), dt[k]) for k in _ARRAYS})


_ARRAYS = ("row_ptr", "col_idx", "csr_val", "col_ptr", "row_idx", "csc_val")


@dataclass(frozen=True)
class DeviceRatings:
    """The same six arrays resident in HBM (torch CUDA tensors)."""

    m: int
    n: int
    nnz: int
    row_ptr: torch.Tensor
    col_idx: torch.Tensor
    csr_val: torch.Tensor
    col_ptr: torch.Tensor
    row_idx: torch.Tensor
    csc_val: torch.Tensor

    def csr_view(self) -> RowView:
        return RowView(self.row_ptr, self.col_idx, self.csr_val, self.m, self.n)

    def csc_view(self) -> RowView:
        return RowView(self.col_ptr, self.row_idx, self.csc_val, self.n, self.m)

    @property
    def nbytes(self) -> int:
        return int(sum(t.numel() * t.element_size() for t in (getattr(self, k) for k in _ARRAYS)))

    def to_host(self) -> SparseRatings:
        return SparseRatings(self.m, self.n, self.nnz,
                             **{k: nat.to_host(getattr(self, k)) for k in _ARRAYS})

    def to_device(self) -> "DeviceRatings":
        return self


@dataclass
class SyntheticTruth:
    x_true: np.ndarray
    theta_true: np.ndarray
    noise_sigma: float


# ------------------------------------------------------------------- build

def _as_triples(triples) -> Triples:
    return triples if isinstance(triples, Triples) else Triples.from_iter(triples)


def build_device(triples, m: int | None = None, n: int | None = None) -> DeviceRatings:
    """CSR + CSC on the GPU (``cmf_build``: hand-written stable radix sorts,
    build.cu); bit-identical to reference data.build (data.py:205-249),
    including the collapse of duplicate (user, item) pairs to the last
    occurrence and the DataError naming the first out-of-range triple."""
    t = _as_triples(triples)
    dev = nat.device()
    user = nat.to_dev(t.user, torch.int64, dev)
    item = nat.to_dev(t.item, torch.int64, dev)
    val = nat.to_dev(t.rating, torch.float32, dev)
    k = int(user.shape[0])
    # an explicit negative extent puts every id out of range, as in the reference
    mn = (ctypes.c_int64 * 2)(-1 if m is None else max(int(m), 0), -1 if n is None else max(int(n), 0))
    if m is not None and int(m) < 0 and k == 0:
        raise DataError(f"negative matrix extent m={m}")
    if n is not None and int(n) < 0 and k == 0:
        raise DataError(f"negative matrix extent n={n}")
    ws = torch.empty(int(nat.lib().cmf_build_workspace_bytes(k)), dtype=torch.uint8, device=dev)
    nnz, bad = ctypes.c_int64(0), ctypes.c_int64(-1)
    args = (nat.ptr(user), nat.ptr(item), 1, nat.ptr(val), k, mn)
    tail = (nat.ptr(ws), ws.numel(), ctypes.byref(nnz), ctypes.byref(bad), nat.stream_ptr())
    if m is None or n is None:  # size the outputs: resolve max id + 1 first
        nat.call("cmf_build", *args, None, None, None, None, None, None, *tail)
    M, N = int(mn[0]), int(mn[1])
    row_ptr = torch.empty(M + 1, dtype=torch.int64, device=dev)
    col_ptr = torch.empty(N + 1, dtype=torch.int64, device=dev)
    col_idx = torch.empty(k, dtype=torch.int32, device=dev)
    row_idx = torch.empty(k, dtype=torch.int32, device=dev)
    csr_val = torch.empty(k, dtype=torch.float32, device=dev)
    csc_val = torch.empty(k, dtype=torch.float32, device=dev)
    rc = nat.lib().cmf_build(*args, nat.ptr(row_ptr), nat.ptr(col_idx), nat.ptr(csr_val), nat.ptr(col_ptr),
                             nat.ptr(row_idx), nat.ptr(csc_val), *tail)
    nat.LAUNCHES[0] += 1
    if rc != nat.CMF_OK and bad.value >= 0:
        i = int(bad.value)
        raise DataError(f"triple ({int(t.user[i])}, {int(t.item[i])}, {float(t.rating[i])}) "
                        f"out of range for a {m if m is not None else M}x{n if n is not None else N} matrix")
    nat.check(rc, "cmf_build")
    del ws
    z = int(nnz.value)
    if z < k:  # duplicates collapsed: trim the worst-case allocations
        col_idx, row_idx = col_idx[:z].clone(), row_idx[:z].clone()
        csr_val, csc_val = csr_val[:z].clone(), csc_val[:z].clone()
    return DeviceRatings(M, N, z, row_ptr, col_idx, csr_val, col_ptr, row_idx, csc_val)


def build(triples, m: int | None = None, n: int | None = None) -> SparseRatings:
    """Reference-compatible ``build``: device construction, host arrays back."""
    return build_device(triples, m, n).to_host()


# ------------------------------------------------------------- text / cache I/O
# File formats of the reference (data.py:1-26): text COO "user<d>item<d>rating"
# per line (tab or comma, '#' comments and blank lines skipped), and the
# little-endian binary CMFR cache (magic, u32 version, u64 m, n, nnz, then
# row_ptr u64[m+1], col_idx u32[nnz], csr_val f32[nnz], col_ptr u64[n+1],
# row_idx u32[nnz], csc_val f32[nnz]).  Files written by either package load
# in the other.

CACHE_MAGIC = b"CMFR"
CACHE_VERSION = 1
_DELIMS = {"tsv": "\t", "csv": ","}
_HEADER = struct.Struct("<IQQQ")


def parse_coo(lines, fmt: str = "tsv", m: int | None = None, n: int | None = None):
    """Text triples -> (Triples, m, n); m, n default to max index + 1
    (data.py:142-190).  Malformed lines raise ParseError with the 1-based line."""
    if fmt not in _DELIMS:
        raise DataError(f"unknown format {fmt!r}; expected 'tsv' or 'csv'")
    delim = _DELIMS[fmt]
    us, vs, rs = [], [], []
    for line_no, raw in enumerate(lines, 1):
        text = raw.strip()
        if not text or text[0] == "#":
            continue
        fields = text.split(delim)
        if len(fields) != 3:
            raise ParseError(f"expected 3 fields separated by {delim!r}, got {len(fields)}", line_no)
        try:
            u, v, r = int(fields[0]), int(fields[1]), float(fields[2])
        except ValueError as exc:
            raise ParseError(str(exc), line_no) from None
        if not math.isfinite(r):
            raise ParseError(f"non-finite rating {fields[2]!r}", line_no)
        if u < 0 or v < 0:
            raise ParseError(f"negative index ({u}, {v})", line_no)
        us.append(u)
        vs.append(v)
        rs.append(r)
    t = Triples(np.array(us, dtype=np.int64), np.array(vs, dtype=np.int64),
                np.array(rs, dtype=np.float64).astype(np.float32))
    if m is None:
        m = int(t.user.max()) + 1 if len(t) else 0
    if n is None:
        n = int(t.item.max()) + 1 if len(t) else 0
    return t, m, n


def load_coo(path, fmt: str = "tsv", m=None, n=None):
    with open(path, "r", encoding="utf-8") as fh:
        return parse_coo(fh, fmt=fmt, m=m, n=n)


def save_coo(path, triples: Triples, fmt: str = "tsv") -> None:
    """One line per triple, ratings with 9 significant digits (round-trips f32)."""
    if fmt not in _DELIMS:
        raise DataError(f"unknown format {fmt!r}; expected 'tsv' or 'csv'")
    d = _DELIMS[fmt]
    u, v, r = (np.asarray(a) for a in (triples.user, triples.item, triples.rating))
    with open(path, "w", encoding="utf-8") as fh:
        fh.writelines(f"{a}{d}{b}{d}{c:.9g}\n" for a, b, c in zip(u.tolist(), v.tolist(), r.tolist()))


_CACHE_LAYOUT = (("row_ptr", "<u8", np.int64), ("col_idx", "<u4", np.int32), ("csr_val", "<f4", np.float32),
                 ("col_ptr", "<u8", np.int64), ("row_idx", "<u4", np.int32), ("csc_val", "<f4", np.float32))


def save_cache(path, sr) -> None:
    """Write the CMFR cache (data.py:305-314); a DeviceRatings is copied to the host."""
    sr = sr.to_host() if isinstance(sr, DeviceRatings) else sr
    with open(path, "wb") as fh:
        fh.write(CACHE_MAGIC)
        fh.write(_HEADER.pack(CACHE_VERSION, sr.m, sr.n, sr.nnz))
        for name, disk, _ in _CACHE_LAYOUT:
            fh.write(np.ascontiguousarray(getattr(sr, name), dtype=disk).tobytes())


def load_cache(path) -> SparseRatings:
    """Read a CMFR cache (data.py:317-345): bad magic, version, truncation or
    trailing bytes raise FormatError."""
    with open(path, "rb") as fh:
        blob = fh.read()
    if blob[:4] != CACHE_MAGIC:
        raise FormatError(f"{path}: not a ratings cache (bad magic {blob[:4]!r})")
    if len(blob) < 4 + _HEADER.size:
        raise FormatError(f"{path}: truncated header")
    version, m, n, nnz = _HEADER.unpack_from(blob, 4)
    if version != CACHE_VERSION:
        raise FormatError(f"{path}: unsupported cache version {version}")
    counts = {"row_ptr": m + 1, "col_ptr": n + 1}
    off = 4 + _HEADER.size
    arrays = {}
    for name, disk, mem in _CACHE_LAYOUT:
        k = counts.get(name, nnz)
        nb = k * np.dtype(disk).itemsize
        if off + nb > len(blob):
            raise FormatError(f"{path}: truncated payload")
        arrays[name] = np.frombuffer(blob, dtype=disk, count=k, offset=off).astype(mem)
        off += nb
    if off != len(blob):
        raise FormatError(f"{path}: trailing bytes after payload")
    return SparseRatings(int(m), int(n), int(nnz), **arrays)


# --------------------------------------------------------- split / synthesis

def split_holdout(triples: Triples, test_fraction: float, seed: int):
    """Deterministic disjoint split (data.py:252-267): the reference's PCG64
    permutation, first round(frac*N) positions -> test, both sorted."""
    if not (0.0 < test_fraction < 1.0):
        raise DataError(f"test_fraction must be in (0, 1), got {test_fraction}")
    total = len(triples)
    k = int(round(test_fraction * total))
    perm = np.random.default_rng(seed).permutation(total)
    parts = (np.sort(perm[k:]), np.sort(perm[:k]))
    u, v, r = (np.asarray(a) for a in (triples.user, triples.item, triples.rating))
    return tuple(Triples(u[ix], v[ix], r[ix]) for ix in parts)


def gen_synthetic(m, n, f, density, noise_sigma, seed):
    """Low-rank-plus-noise ratings with the reference's draw sequence
    (data.py:270-302): x_true, theta_true ~ U[-0.5, 0.5) float32, k distinct
    positions by ``choice(m*n, k, replace=False)``, rating = float32 dot
    (+ N(0, sigma) via float64)."""
    if not (0.0 < density <= 1.0):
        raise DataError(f"density must be in (0, 1], got {density}")
    if f < 1:
        raise DataError("f must be >= 1")
    k = int(round(density * m * n))
    if k < 1:
        raise DataError(f"density {density} yields no entries for a {m}x{n} matrix")
    rng = np.random.default_rng(seed)
    x_true = (rng.random((m, f), dtype=np.float32) - np.float32(0.5)).astype(np.float32)
    t_true = (rng.random((n, f), dtype=np.float32) - np.float32(0.5)).astype(np.float32)
    cells = np.sort(rng.choice(m * n, size=k, replace=False))
    users, items = (cells // n).astype(np.int64), (cells % n).astype(np.int64)
    ratings = _host_dot(x_true, t_true, users, items)
    if noise_sigma > 0:
        ratings = (ratings.astype(np.float64) + rng.normal(0.0, noise_sigma, size=k)).astype(np.float32)
    return Triples(users, items, ratings), SyntheticTruth(x_true, t_true, noise_sigma)


def _host_dot(x, t, users, items, chunk=1 << 18):
    # the reference's predict_pairs arithmetic (float32 einsum per chunk); kept on
    # the host so generated inputs are bit-identical to the reference's
    out = np.empty(users.shape[0], dtype=np.float32)
    for lo in range(0, users.shape[0], chunk):
        hi = min(lo + chunk, users.shape[0])
        out[lo:hi] = np.einsum("ij,ij->i", x[users[lo:hi]], t[items[lo:hi]])
    return out


def stream_params(m: int, n: int, nnz: int, noise_sigma: float = 0.1, test_fraction: float = 0.1):
    """Integer Bernoulli thresholds and the float32 noise scale of the streaming
    generator: cells present with p = nnz / (1 - test_fraction) / (m n), held out
    with q = test_fraction (so the expected train count is nnz)."""
    if m < 1 or n < 1 or nnz < 1:
        raise DataError("streaming generator needs m, n, nnz >= 1")
    if not (0.0 <= test_fraction < 1.0):
        raise DataError(f"test_fraction must be in [0, 1), got {test_fraction}")
    p = nnz / (1.0 - test_fraction) / (float(m) * float(n))
    if p > 1.0:
        raise DataError(f"{nnz} ratings do not fit a {m}x{n} matrix")
    thr_cell = min(int(p * 2.0 ** 64), 2 ** 64 - 1)
    thr_test = min(int(test_fraction * 2.0 ** 64), 2 ** 64 - 1)
    scale = float(np.float32(noise_sigma * math.sqrt(3.0)))
    return thr_cell, thr_test, scale


@dataclass
class StreamShard:
    """One rank's generated shards: CSR rows of users [u0, u1) and CSC rows of
    items [v0, v1) (pointers rebased to the shard), the held-out triples of its
    users, and the truth factors the ratings were drawn from."""
    m: int
    n: int
    users: tuple
    items: tuple
    x_view: tuple
    t_view: tuple
    test: Triples
    x_true: torch.Tensor
    t_true: torch.Tensor


def gen_stream_shard(m: int, n: int, f: int, nnz: int, noise_sigma: float = 0.1, test_fraction: float = 0.1,
                     seed: int = 0, users: tuple | None = None, items: tuple | None = None,
                     local_csc: bool = False) -> StreamShard:
    """Streaming synthetic generator (gen.cu): the CSR rows of
    users [u0, u1) and CSC rows of items [v0, v1) of a low-rank-plus-noise
    matrix with ~nnz train ratings, generated on the device in build() order
    from counter-based hashes -- no triples are materialised, no rank sees
    another's shard, and the shards of all ranks tile the global matrix.  The
    model is gen_synthetic's (data.py:270-302: U[-1/2, 1/2) truth, uniformly
    random cells, dot + noise of variance sigma^2) but its draws are not the
    reference's PCG64 stream (Bernoulli cells, Irwin-Hall noise).
    ``local_csc``: the CSC covers ALL items but only this rank's users (ids
    relative to u0) -- the input of the reduce-scatter exchange
    (distributed.ReduceScatterALS) instead of the item range's CSC."""
    u0, u1 = users if users is not None else (0, m)
    v0, v1 = items if items is not None else (0, n)
    thr_cell, thr_test, scale = stream_params(m, n, nnz, noise_sigma, test_fraction)
    dev = nat.device()
    st = nat.stream_ptr()
    X = torch.empty(m, f, dtype=torch.float32, device=dev)
    T = torch.empty(n, f, dtype=torch.float32, device=dev)
    nat.call("cmf_gen_truth", seed, 0, m, f, nat.ptr(X), st)
    nat.call("cmf_gen_truth", seed, 1, n, f, nat.ptr(T), st)

    def side(by_user, lo, hi, mlo=0, mhi=None):
        mhi = (n if by_user else m) if mhi is None else mhi
        nr = hi - lo
        ptr = torch.empty(nr + 1, dtype=torch.int64, device=dev)
        tptr = torch.empty(nr + 1, dtype=torch.int64, device=dev) if by_user else None
        scratch = torch.empty(max(2 * nr, 1), dtype=torch.int64, device=dev)
        nat.call("cmf_gen_count", seed, m, n, thr_cell, thr_test, int(by_user), lo, hi, mlo, mhi, nat.ptr(ptr),
                 nat.ptr(tptr), nat.ptr(scratch), st)
        ntr = int(ptr[-1].item())
        nte = int(tptr[-1].item()) if by_user else 0
        minor = torch.empty(ntr, dtype=torch.int32, device=dev)
        val = torch.empty(ntr, dtype=torch.float32, device=dev)
        tu = torch.empty(nte, dtype=torch.int64, device=dev) if by_user else None
        tv = torch.empty(nte, dtype=torch.int64, device=dev) if by_user else None
        tr = torch.empty(nte, dtype=torch.float32, device=dev) if by_user else None
        nat.call("cmf_gen_fill", seed, m, n, f, thr_cell, thr_test, scale, int(by_user), lo, hi, mlo, mhi,
                 nat.ptr(X), nat.ptr(T), nat.ptr(ptr), nat.ptr(minor), nat.ptr(val), nat.ptr(tptr), nat.ptr(tu),
                 nat.ptr(tv), nat.ptr(tr), st)
        return (ptr, minor, val), (Triples(tu, tv, tr) if by_user else None)

    x_view, test = side(True, u0, u1)
    if local_csc:
        # every item's ratings from this rank's users only, user ids relative to u0
        t_view, _ = side(False, 0, n, u0, u1)
    else:
        t_view, _ = side(False, v0, v1)
    return StreamShard(m, n, (u0, u1), (v0, v1), x_view, t_view, test, X, T)


def gen_synthetic_stream(m: int, n: int, f: int, nnz: int, noise_sigma: float = 0.1, test_fraction: float = 0.1,
                         seed: int = 0):
    """The whole matrix from the streaming generator: (DeviceRatings, test Triples)."""
    sh = gen_stream_shard(m, n, f, nnz, noise_sigma, test_fraction, seed)
    (rp, ci, cv), (cp, ri, rv) = sh.x_view, sh.t_view
    return DeviceRatings(m, n, int(ci.numel()), rp, ci, cv, cp, ri, rv), sh.test


def gen_synthetic_device(m: int, n: int, f: int, nnz: int, noise_sigma: float = 0.1,
                         test_fraction: float = 0.1, seed: int = 0, row_chunk: int | None = None):
    """Fast on-GPU generator for benchmark shapes (Netflix / Yahoo / Hugewiki).

    Same model as ``gen_synthetic`` -- U[-0.5, 0.5) truth factors, uniformly
    random distinct cells, float32 dot + N(0, sigma) -- but cells are drawn
    per row block as independent Bernoulli(p) with p = nnz_total/(m*n), where
    nnz_total = nnz/(1-test_fraction), and a Bernoulli(test_fraction) mask
    makes the holdout.  Train nnz is therefore nnz +- O(sqrt(nnz)).  Not
    bit-identical to the reference generator (which cannot reach these sizes
    on a 62 GB host); returns (DeviceRatings train, Triples test on device).
    """
    dev = nat.device()
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    total = nnz / (1.0 - test_fraction)
    p = total / (float(m) * float(n))
    xt = torch.rand((m, f), generator=g, device=dev) - 0.5
    tt = torch.rand((n, f), generator=g, device=dev) - 0.5
    if row_chunk is None:
        row_chunk = max(1, (1 << 28) // max(n, 1))
    us, vs = [], []
    for r0 in range(0, m, row_chunk):
        r1 = min(m, r0 + row_chunk)
        mask = torch.rand((r1 - r0, n), generator=g, device=dev) < p
        nzr, nzc = torch.nonzero(mask, as_tuple=True)
        us.append(nzr.to(torch.int64) + r0)
        vs.append(nzc.to(torch.int64))
        del mask
    users, items = torch.cat(us), torch.cat(vs)
    del us, vs
    ratings = predict_pairs(xt, tt, users, items)
    ratings = ratings + noise_sigma * torch.randn(ratings.shape, generator=g, device=dev)
    is_test = torch.rand(users.shape, generator=g, device=dev) < test_fraction
    test = Triples(users[is_test], items[is_test], ratings[is_test])
    keep = ~is_test
    train = build_device(Triples(users[keep], items[keep], ratings[keep]), m, n)
    return train, test
