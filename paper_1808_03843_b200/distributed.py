"""Multi-GPU ALS driver: users (CSR rows) and items (CSC rows)
are split into contiguous nnz-balanced ranges, one range per rank (one
process per GPU, torch.distributed over NCCL / NVLink).  Each rank keeps only
its byte-exact slices of the CSR and CSC arrays (pointers rebased), plus full
replicas of X and Theta.  An iteration is

    update-X on my user rows  ->  all-gather X  ->  update-Theta on my item rows
    ->  all-gather Theta

which is the reference's epoch barrier (als.py:132-140) with the exchange
inserted where the other half first reads the updated matrix.  With one rank
there is no collective at all.

Peer-store mode (``attach_replicas``): the ranks map each other's X / Theta
replicas through CUDA IPC (NVLink peer memory), and the fused CG kernel
stores every solved row into all replicas as it finishes it
(cmf_fused_cg_update_peers), so the exchange overlaps the solve and the
all-gather disappears; a stream sync + rank barrier orders the halves.
Non-fused routes (exact, two-step) keep the all-gather.

Shard boundaries: r_s = searchsorted(indptr, s * nnz / k, "left") -- a pure
function of the pointer array, so every rank computes the same plan without
communication, and concatenating the shards reproduces the reference arrays
exactly (tests/test_distributed.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .als import HalfUpdatePlan, resolve_gram_kernel
from .errors import DataError, NumericalError


def shard_bounds(indptr, world: int) -> list[int]:
    """Row boundaries [b_0=0, ..., b_k=nrows] balancing stored ratings."""
    ptr = indptr.cpu().numpy() if isinstance(indptr, torch.Tensor) else np.asarray(indptr)
    nrows = ptr.shape[0] - 1
    nnz = int(ptr[-1])
    bounds = [0]
    for s in range(1, world):
        b = int(np.searchsorted(ptr, s * nnz / world, side="left"))
        bounds.append(min(max(b, bounds[-1]), nrows))
    bounds.append(nrows)
    return bounds


def shard_view(indptr, indices, values, lo: int, hi: int):
    """Rows [lo, hi) as a self-contained view with rebased pointers."""
    p0 = int(indptr[lo])
    p1 = int(indptr[hi])
    ptr = indptr[lo:hi + 1] - p0
    return ptr, indices[p0:p1], values[p0:p1]


@dataclass
class ShardedRatings:
    """One rank's byte-exact slices of the CSR (user rows [xb[r], xb[r+1])) and
    CSC (item rows [tb[r], tb[r+1])) arrays, pointers rebased; m, n, nnz are the
    global sizes.  Built by ``shard_ratings`` without materialising the other
    ranks' rows on this device."""

    m: int
    n: int
    nnz: int
    xb: list
    tb: list
    x_view: tuple
    t_view: tuple


def shard_ratings(triples, m: int, n: int, rank: int, world: int) -> ShardedRatings:
    """Per-rank build: the row/column counts of the host triples
    give the nnz-balanced boundaries (every rank computes the same ones); the
    rank then builds on its device only the triples of its user range (its CSR
    rows) and of its item range (its CSC rows).  Duplicates of a (user, item)
    pair fall in the same shard, so the last-wins de-duplication of
    data.build (data.py:205-249) is shard-local and the concatenated shards
    equal the single-device arrays byte for byte (tests/test_distributed.py).
    The boundaries balance the pre-de-duplication counts, which equal the
    final ones whenever the triples are distinct (the synthetic generator)."""
    from .data import Triples, build_device
    u = np.asarray(triples.user.cpu() if isinstance(triples.user, torch.Tensor) else triples.user)
    v = np.asarray(triples.item.cpu() if isinstance(triples.item, torch.Tensor) else triples.item)
    r = np.asarray(triples.rating.cpu() if isinstance(triples.rating, torch.Tensor) else triples.rating)
    if len(u) and (u.min() < 0 or u.max() >= m or v.min() < 0 or v.max() >= n):
        raise DataError(f"triple out of range for a {m}x{n} matrix")
    row_ptr = np.zeros(m + 1, np.int64)
    np.cumsum(np.bincount(u, minlength=m), out=row_ptr[1:])
    col_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(v, minlength=n), out=col_ptr[1:])
    xb, tb = shard_bounds(row_ptr, world), shard_bounds(col_ptr, world)
    xlo, xhi, tlo, thi = xb[rank], xb[rank + 1], tb[rank], tb[rank + 1]
    if world == 1:
        full = build_device(Triples(u, v, r), m, n)
        return ShardedRatings(m, n, full.nnz, xb, tb,
                              (full.row_ptr, full.col_idx, full.csr_val),
                              (full.col_ptr, full.row_idx, full.csc_val))
    sel = np.flatnonzero((u >= xlo) & (u < xhi))
    part = build_device(Triples(u[sel] - xlo, v[sel], r[sel]), xhi - xlo, n)
    x_view = (part.row_ptr, part.col_idx, part.csr_val)
    nnz_x = part.nnz
    del part
    sel = np.flatnonzero((v >= tlo) & (v < thi))
    part = build_device(Triples(u[sel], v[sel] - tlo, r[sel]), m, thi - tlo)
    t_view = (part.col_ptr, part.row_idx, part.csc_val)
    del part
    # global nnz after de-duplication = sum of every rank's CSR shard
    nnz = nnz_x
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        t = torch.tensor([nnz_x], dtype=torch.int64,
                         device=x_view[0].device if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t)
        nnz = int(t.item())
    return ShardedRatings(m, n, nnz, xb, tb, x_view, t_view)


class RowGather:
    """All-gather of row blocks of a (rows, f) matrix whose rank-s block is
    rows [b_s, b_{s+1}).  Uneven blocks are padded to the largest one for a
    single all_gather_into_tensor, then unpacked in place."""

    def __init__(self, bounds, f, device, dtype=torch.float32):
        self.bounds = bounds
        self.world = len(bounds) - 1
        self.maxrows = max(bounds[i + 1] - bounds[i] for i in range(self.world))
        self.buf = torch.empty((self.world, self.maxrows, f), dtype=dtype, device=device)
        self.equal = all(bounds[i + 1] - bounds[i] == self.maxrows for i in range(self.world))

    def __call__(self, full: torch.Tensor, rank: int, group=None):
        import torch.distributed as dist
        if full.is_cuda and dist.get_backend(group) == "gloo":
            # gloo has no CUDA all-gather: stage through host memory (multi-rank
            # tests on one device; production runs NCCL over NVLink)
            host = full.cpu()
            RowGather(self.bounds, full.shape[1], torch.device("cpu"), full.dtype)(host, rank, group)
            full.copy_(host)
            return
        lo, hi = self.bounds[rank], self.bounds[rank + 1]
        if self.equal and full.is_contiguous():
            dist.all_gather_into_tensor(full[: self.world * self.maxrows].view(-1),
                                        full[lo:hi].reshape(-1), group=group)
            return
        self.buf[rank, : hi - lo].copy_(full[lo:hi])
        dist.all_gather_into_tensor(self.buf.view(-1), self.buf[rank].reshape(-1).clone(),
                                    group=group)
        for s in range(self.world):
            a, b = self.bounds[s], self.bounds[s + 1]
            if s != rank and b > a:
                full[a:b].copy_(self.buf[s, : b - a])


class ShardedALS:
    """Row-sharded ALS iteration over `world` ranks (world == 1: plain device ALS)."""

    def __init__(self, ratings, f: int, lam: float, solver, gram_kernel: str = "auto",
                 rank: int = 0, world: int = 1, weighted_reg: bool = True, group=None):
        self.f, self.lam, self.solver = f, lam, solver
        self.weighted_reg = weighted_reg
        self.rank, self.world, self.group = rank, world, group
        self.gram_kernel = resolve_gram_kernel(gram_kernel, solver, f)
        self.m, self.n = ratings.m, ratings.n
        if isinstance(ratings, ShardedRatings):
            # built per rank (shard_ratings): only this rank's rows are resident
            if len(ratings.xb) != world + 1:
                raise DataError(f"shards were built for {len(ratings.xb) - 1} ranks, not {world}")
            self.xb, self.tb = ratings.xb, ratings.tb
            self.x_view, self.t_view = ratings.x_view, ratings.t_view
            dev = self.x_view[0].device
        else:
            dev = ratings.row_ptr.device
            self.xb = shard_bounds(ratings.row_ptr, world)
            self.tb = shard_bounds(ratings.col_ptr, world)
            self.x_view = shard_view(ratings.row_ptr, ratings.col_idx, ratings.csr_val,
                                     self.xb[rank], self.xb[rank + 1])
            self.t_view = shard_view(ratings.col_ptr, ratings.row_idx, ratings.csc_val,
                                     self.tb[rank], self.tb[rank + 1])
        xs = (self.xb[rank], self.xb[rank + 1])
        ts = (self.tb[rank], self.tb[rank + 1])
        self.x_plan = HalfUpdatePlan(xs[1] - xs[0], f, solver, dev)
        self.t_plan = HalfUpdatePlan(ts[1] - ts[0], f, solver, dev)
        if world > 1:
            self.x_gather = RowGather(self.xb, f, dev)
            self.t_gather = RowGather(self.tb, f, dev)
        self._replicas = None  # (x ptr, theta ptr, peers_x, peers_t, opened storages)

    def attach_replicas(self, x: torch.Tensor, theta: torch.Tensor) -> bool:
        """Map every other rank's copies of x and theta (CUDA IPC) for peer
        stores; collective over the group.  Returns False (all-gather stays)
        when there is a single rank or the route is not the fused kernel."""
        import torch.distributed as dist
        fused = self.gram_kernel == "tc" and self.solver.method == "cg"
        if self.world == 1 or not fused:
            return False
        for t in (x, theta):
            if not (t.is_cuda and t.is_contiguous() and t.dtype == torch.float32):
                raise DataError("replicas must be contiguous float32 CUDA tensors")

        def export(t):
            h = ctypes.create_string_buffer(64)
            off = ctypes.c_int64()
            nat.call("cmf_ipc_export", t.data_ptr(), ctypes.addressof(h), ctypes.addressof(off))
            return h.raw, off.value

        def open_peer(h, off):
            buf = ctypes.create_string_buffer(h, 64)
            ptr = ctypes.c_void_p()
            nat.call("cmf_ipc_open", ctypes.addressof(buf), off, ctypes.addressof(ptr))
            opened.append((ptr.value, off))
            return ptr.value

        mine = (export(x), export(theta))
        everyone = [None] * self.world
        dist.all_gather_object(everyone, mine, group=self.group)
        opened, px, pt = [], [], []
        xlo, tlo = self.xb[self.rank], self.tb[self.rank]
        for r, (hx, ht) in enumerate(everyone):
            if r == self.rank:
                continue
            # my rows land at the same row index of the peer's replica
            px.append(open_peer(*hx) + 4 * xlo * self.f)
            pt.append(open_peer(*ht) + 4 * tlo * self.f)
        dev = x.device
        self._replicas = (x.data_ptr(), theta.data_ptr(),
                          torch.tensor(px, dtype=torch.int64, device=dev),
                          torch.tensor(pt, dtype=torch.int64, device=dev), opened)
        dist.barrier(group=self.group)
        return True

    def local_nnz(self):
        return {"x": int(self.x_view[0][-1]), "t": int(self.t_view[0][-1])}

    def local_rows(self):
        return {"x": self.xb[self.rank + 1] - self.xb[self.rank],
                "t": self.tb[self.rank + 1] - self.tb[self.rank]}

    def detach_replicas(self):
        """Unmap the peers' replicas (after the last iteration that uses them)."""
        if self._replicas is not None:
            torch.cuda.synchronize()
            for ptr, off in self._replicas[4]:
                nat.call("cmf_ipc_close", ptr, off)
            self._replicas = None

    def _half(self, plan, view, fixed, target, lo, record, peers=None):
        ptr, idx, val = view
        # the plan writes rows [0, nrows) of the view; point it at target[lo:]
        plan.launch(ptr, idx, val, fixed, target[lo:], self.lam, self.weighted_reg,
                    self.gram_kernel, record, peers=peers)

    def _peer_barrier(self, record):
        import torch.distributed as dist
        if record is not None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        torch.cuda.current_stream().synchronize()  # my peer stores are complete
        dist.barrier(group=self.group)              # ... and everyone else's
        if record is not None:
            e1.record()
            record.setdefault("peer_barrier", []).append((e0, e1))

    def iteration(self, x: torch.Tensor, theta: torch.Tensor, record: dict | None = None):
        rep = self._replicas
        if rep is not None and (rep[0], rep[1]) == (x.data_ptr(), theta.data_ptr()):
            self._half(self.x_plan, self.x_view, theta, x, self.xb[self.rank], record, peers=rep[2])
            self._peer_barrier(record)
            self._half(self.t_plan, self.t_view, x, theta, self.tb[self.rank], record, peers=rep[3])
            self._peer_barrier(record)
            return
        self._half(self.x_plan, self.x_view, theta, x, self.xb[self.rank], record)
        if self.world > 1:
            self._gather(self.x_gather, x, record)
        self._half(self.t_plan, self.t_view, x, theta, self.tb[self.rank], record)
        if self.world > 1:
            self._gather(self.t_gather, theta, record)

    def _gather(self, g, full, record):
        if record is not None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        g(full, self.rank, self.group)
        if record is not None:
            e1.record()
            record.setdefault("allgather", []).append((e0, e1))

    def check(self):
        """Read the accumulated device flags once (synchronises)."""
        fx, ft = self.x_plan.read_flags(), self.t_plan.read_flags()
        if fx[0] or ft[0]:
            raise NumericalError("Gram entries overflow binary16 range (+-65504); "
                                 "rescale the ratings before using half precision")
        if fx[2] or ft[2]:
            raise DataError("singular system(s) during sharded training")
        return fx[1] + ft[1]


class ReduceScatterALS:
    """Tall-skinny multi-GPU ALS without an X replica (the "better
    exchange for tall-skinny" row).  Rank r owns the user
    rows [ub[r], ub[r+1]) -- its rows of X only -- and the item rows
    [vb[r], vb[r+1]); Theta (n x f, small when m >> n) is replicated.  One
    iteration:

      update-X on my users (fused kernel, fixed = Theta)              no exchange
      pass 1 over my LOCAL CSC (every item x my users): each item's partial
        Gram + bias from my users, fp32, into a partial buffer (n x f x pws)
      reduce-scatter (sum) of the partial buffers: my items' complete accumulators
      pass 2 on my items from the partial alone (empty gather segment, lambda n_v
        with the global n_v)                                          -> Theta rows
      all-gather Theta

    The wire carries (k-1)/k of the partial buffer (Hugewiki, k = 8: ~2 GB per
    rank) instead of (k-1)/k of X (17.5 GB), and no rank holds X.  The partials
    of different ranks are summed in rank order, so results match the replicated
    route up to fp32 summation order (CG route: RMSE parity).  Inputs come from
    data.gen_stream_shard(..., local_csc=True)."""

    def __init__(self, shard, f: int, lam: float, solver, rank: int = 0, world: int = 1, group=None):
        import torch.distributed as dist
        if not (solver.method == "cg" and resolve_gram_kernel("auto", solver, f) == "tc"):
            raise DataError("the reduce-scatter exchange runs the fused CG route (precision='fp16')")
        self.f, self.lam, self.solver = f, lam, solver
        self.gram_kernel = "tc"
        self.rank, self.world, self.group = rank, world, group
        self.m, self.n = shard.m, shard.n
        self.u0, self.u1 = shard.users
        self.x_view, self.c_view = shard.x_view, shard.t_view
        dev = self.x_view[0].device
        n = self.n
        nc = (n + world - 1) // world
        self.nc = nc
        self.vb = [min(s * nc, n) for s in range(world + 1)]
        self.v0, self.v1 = self.vb[rank], self.vb[rank + 1]
        # global per-item counts -> pass-2 pointers of my items (empty segments)
        cnt = torch.diff(self.c_view[0])
        if world > 1:
            cnt = cnt.clone()
            if dist.get_backend(group) == "gloo":
                h = cnt.cpu()
                dist.all_reduce(h, group=group)
                cnt = h.to(dev)
            else:
                dist.all_reduce(cnt, group=group)
        self.n_global = int(cnt.sum().item())
        mine = cnt[self.v0:self.v1]
        self.ptr2 = torch.zeros(mine.numel() + 1, dtype=torch.int64, device=dev)
        torch.cumsum(mine, 0, out=self.ptr2[1:])
        self.seg1 = self.c_view[0][1:].contiguous()  # pass 1: the whole local row
        self.seg2 = self.ptr2[1:].contiguous()        # pass 2: nothing to gather
        pf = int(nat.lib().cmf_fused_cg_partial_floats(1, f))  # floats per item
        self.pf = pf
        self.partial = torch.empty(world * nc * pf, dtype=torch.float32, device=dev)
        self.mine = torch.empty(nc * pf, dtype=torch.float32, device=dev)
        self.x_plan = HalfUpdatePlan(self.u1 - self.u0, f, solver, dev)
        self.c_plan = HalfUpdatePlan(n, f, solver, dev)
        self.t_gather = RowGather(self.vb, f, dev) if world > 1 else None

    def local_rows(self):
        return {"x": self.u1 - self.u0, "t": self.v1 - self.v0}

    def local_nnz(self):
        """Ratings this rank gathers per half: its users' CSR rows and its local CSC."""
        return {"x": int(self.x_view[1].numel()), "t": int(self.c_view[1].numel())}

    def attach_replicas(self, x, theta) -> bool:  # no X replica, no peer stores
        return False

    def detach_replicas(self):
        pass

    def _reduce_scatter(self):
        import torch.distributed as dist
        if self.world == 1:
            self.mine.copy_(self.partial[: self.nc * self.pf])
            return
        if dist.get_backend(self.group) == "gloo":  # ranks sharing a device (tests): via host memory
            h = self.partial.cpu()
            dist.all_reduce(h, group=self.group)
            self.mine.copy_(h[self.rank * self.nc * self.pf:(self.rank + 1) * self.nc * self.pf])
            return
        dist.reduce_scatter_tensor(self.mine, self.partial, group=self.group)

    def iteration(self, x_local, theta, record=None):
        """x_local: this rank's rows of X ((u1-u0) x f), theta: the full replica."""
        s, f = self.solver, self.f
        st = nat.stream_ptr()
        xp, xi, xv = self.x_view
        self.x_plan.launch(xp, xi, xv, theta, x_local, self.lam, True, "tc", record)
        cp, ci, cv = self.c_view
        shadow, _ = self.c_plan._shadow(x_local)
        self.partial.zero_()
        common = (nat.ptr(shadow), self.u1 - self.u0, self.c_plan.w16, f, float(self.lam), 1)
        nat.call("cmf_fused_cg_pass", nat.ptr(cp), nat.ptr(ci), nat.ptr(cv), self.n, int(ci.numel()), *common,
                 nat.ptr(theta), None, 0, nat.ptr(self.seg1), nat.ptr(self.partial), 1, int(s.cg_iters),
                 float(s.cg_tol), nat.ptr(self.c_plan.flags) + 4, nat.ptr(self.c_plan.flags), st)
        self._reduce_scatter()
        nv = self.v1 - self.v0
        if nv:
            nat.call("cmf_fused_cg_pass", nat.ptr(self.ptr2), nat.ptr(ci), nat.ptr(cv), nv, 0, *common,
                     nat.ptr(theta) + 4 * self.v0 * f, None, 0, nat.ptr(self.seg2), nat.ptr(self.mine), 2,
                     int(s.cg_iters), float(s.cg_tol), nat.ptr(self.c_plan.flags) + 4, nat.ptr(self.c_plan.flags),
                     st)
        if self.t_gather is not None:
            self.t_gather(theta, self.rank, self.group)

    def check(self):
        for plan in (self.x_plan, self.c_plan):
            fl = plan.read_flags()
            if fl[0]:
                raise NumericalError("Gram entries overflow binary16 range (+-65504); "
                                     "rescale the ratings before using half precision")
