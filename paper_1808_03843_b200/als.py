"""Explicit-feedback ALS on the B200: the half-iteration and the epoch loop.

Mirrors the reference's als.py (als.py:33-163).  ``update_side`` is the
drop-in boundary (als.py:54-74): same signature, same in-place semantics
(``target`` rows with n_u > 0 are overwritten, ``fixed`` is read-only), same
return value (PhaseTimes, gram_bytes, cg_breakdowns) and errors.

Per half-update the rows are processed in blocks that fit a cached HBM
workspace (all of a Netflix side fits one block): one fused Gram+bias kernel
writes the block's packed systems (fp16 or fp32, 16-byte aligned stride),
then one solve kernel reads them and writes the solutions straight into
``target`` (systems with n_u == 0 are skipped in-kernel, which is the
reference's compaction without the copies).  ``train`` keeps the ratings,
both factor matrices and the test set resident; only per-epoch scalars come
back to the host.
"""

from __future__ import annotations

import os
from dataclasses import asdict, dataclass, field

import numpy as np
import torch

from . import _native as nat
from .data import DeviceRatings, RowView, SparseRatings, Triples
from .errors import DataError, NumericalError
from .factors import init_factors
from .gram import TileConfig, packed_size, roofline_estimate
from .report import EpochRecord, PhaseTimes, TrainReport
from .solvers import SolverConfig, _singular_error, with_accum

WORKSPACE_BYTES = int(float(os.environ.get("CMF_WORKSPACE_GB", "16")) * (1 << 30))


@dataclass
class AlsConfig:
    f: int = 100
    lam: float = 0.05
    epochs: int = 10
    solver: SolverConfig = field(default_factory=SolverConfig)
    init_scale: float = 0.1
    seed: int = 0
    target_rmse: float | None = None
    weighted_reg: bool = True
    tiles: TileConfig = field(default_factory=TileConfig)
    gram_kernel: str = "auto"

    def __post_init__(self):
        if self.f < 1:
            raise DataError("f must be >= 1")
        if self.lam < 0:
            raise DataError("lambda must be >= 0")
        if self.epochs < 1:
            raise DataError("epochs must be >= 1")


def aligned_stride(f: int) -> int:
    """Packed row stride rounded to 8 elements (16-byte rows in fp16)."""
    return (packed_size(f) + 7) // 8 * 8


TC_MAX_F = 120  # tensor-core paths: roundup8(f) feature rows + 2 rating rows within M = 128
SPLIT_SCALE = 64.0  # split-fp16 shadow scale: lo stays normal for |theta| >= 2^-9


def resolve_gram_kernel(kernel: str | None, solver: SolverConfig, f: int | None = None) -> str:
    """Kernel choice for update_side/train.

    "auto": the CG route with binary16 Hermitian storage (precision="fp16",
    the paper's approximate route) runs fused on the tensor cores ("tc": Gram
    in TMEM, repacked to binary16 there, CG matvecs on the tensor core, A never
    stored) when f <= 120.  precision="fp32" keeps fp32 storage: the
    split-precision tensor-core Gram ("tc_split": hi/lo fp16 operands, three
    MMAs, fp32-faithful) writes fp32 packed systems that the fp32 CG (or the
    Cholesky) reads -- the same route the exact solver takes, since the 1e-4
    factor bar rules out a single fp16/TF32 pass.  accum="fp64"
    also leaves the fused kernel (its vectors are fp32): "tc_unfused" for
    fp16 storage.  Larger f falls back to the SIMT FMA Gram.
    "tc_unfused" is the paper's two-step scheme on the tensor cores: packed
    fp16/fp32 A_u written to HBM, then the batched CG kernel reads it.
    An explicit "tc" with precision="fp32" or accum="fp64" is refused
    (DataError): the fused kernel computes in binary16/fp32 only.
    """
    solver = with_accum(solver, "fp32")
    if kernel in (None, "auto"):
        kernel = os.environ.get("CMF_TRAIN_GRAM_KERNEL", "auto")
    small = f is None or f <= TC_MAX_F
    if kernel == "auto":
        if not small:
            return "fma"
        if solver.method == "cg" and solver.precision == "fp16":
            return "tc" if solver.accum == "fp32" else "tc_unfused"
        return "tc_split"
    if kernel not in nat.GRAM_KERNELS:
        raise DataError(f"unknown gram kernel {kernel!r}")
    if kernel == "tc" and solver.method == "cg" and (solver.precision != "fp16" or solver.accum != "fp32"):
        raise DataError("the fused tensor-core CG kernel stores A_u in binary16 and runs fp32 vectors; "
                        "use precision='fp16', accum='fp32' (or gram_kernel='tc_unfused' / 'tc_split')")
    if kernel in ("tc", "tc_unfused") and solver.method == "exact":
        raise DataError("the single-pass fp16 tensor-core Gram cannot feed the exact solver; "
                        "use gram_kernel='tc_split', 'fma' or 'bitwise'")
    if kernel == "tc_split" and solver.precision != "fp32":
        raise DataError("the split-precision Gram stores fp32")
    if kernel.startswith("tc") and f is not None and f > TC_MAX_F:
        raise DataError(f"tensor-core Gram supports f <= {TC_MAX_F}")
    return kernel


class _Workspace:
    """Per-device scratch for the packed systems of one row block."""

    def __init__(self):
        self.bufs = {}

    def get(self, dev, nbytes: int, key: str = "systems") -> torch.Tensor:
        key = (dev.index, key)
        t = self.bufs.get(key)
        if t is None or t.numel() < nbytes:
            self.bufs.pop(key, None)
            t = torch.empty(nbytes, dtype=torch.uint8, device=dev)
            self.bufs[key] = t
        return t


_WS = _Workspace()


def release_workspace():
    _WS.bufs.clear()


def _view_dev(view: RowView, dev):
    return (nat.to_dev(view.indptr, torch.int64, dev), nat.to_dev(view.indices, torch.int32, dev),
            nat.to_dev(view.values, torch.float32, dev))


class HalfUpdatePlan:
    """Device buffers for repeated half-updates of one view: the packed-system
    workspace (16-byte aligned stride), b, n_u and a 4-int flag block
    (overflow, CG breakdowns, singular systems).  Launching through a plan
    never synchronises; ``check`` reads the flags once."""

    def __init__(self, nrows: int, f: int, solver: SolverConfig, dev,
                 workspace_bytes: int | None = None):
        solver = with_accum(solver, "fp32")
        self.f, self.solver, self.nrows, self.dev = f, solver, nrows, dev
        self.half = solver.precision == "fp16"
        self.esize = 2 if self.half else 4
        self.stride = aligned_stride(f)
        self.row_bytes = self.stride * self.esize + f * 4 + 8
        budget = WORKSPACE_BYTES if workspace_bytes is None else int(workspace_bytes)
        self.rows_blk = max(1, min(nrows, budget // self.row_bytes)) if nrows else 1
        self.a_ws = self.b_ws = self.nu_ws = None  # allocated on first two-step launch
        self.flags = torch.zeros(4, dtype=torch.int32, device=dev)
        self.w16 = nat.tc_width(f)
        self.shadow = None  # binary16 copy of the fixed factors (tensor-core Gram)
        self._shadow_lo = None

    def _workspace(self):
        if self.a_ws is None:
            rb, f = self.rows_blk, self.f
            ws = _WS.get(self.dev, rb * self.row_bytes)
            a = ws[: rb * self.stride * self.esize]
            self.a_ws = a.view(torch.float16 if self.half else torch.float32).view(rb, self.stride)
            off = rb * self.stride * self.esize
            self.b_ws = ws[off: off + rb * f * 4].view(torch.float32).view(rb, f)
            off += rb * f * 4
            self.nu_ws = ws[off: off + rb * 8].view(torch.int64)

    def _shadow(self, fx, split: bool = False):
        """binary16 shadow of the fixed factors (hi, or hi + lo for the split Gram)."""
        need = (fx.shape[0] + 1) * self.w16 * (2 if split else 1)  # + the zero padding row
        if self.shadow is None or self.shadow.numel() < need:
            self.shadow = torch.empty(need, dtype=torch.float16, device=fx.device)
        if split:
            half = (fx.shape[0] + 1) * self.w16
            nat.call("cmf_factors_to_half_split", nat.ptr(fx), fx.shape[0], self.f,
                     nat.ptr(self.shadow), nat.ptr(self.shadow) + 2 * half, self.w16, SPLIT_SCALE,
                     nat.ptr(self.flags), nat.stream_ptr())
            return self.shadow, nat.ptr(self.shadow) + 2 * half
        nat.call("cmf_factors_to_half", nat.ptr(fx), fx.shape[0], self.f, nat.ptr(self.shadow),
                 self.w16, nat.ptr(self.flags), nat.stream_ptr())
        return self.shadow, None

    def launch(self, indptr, indices, values, fx, tg, lam, weighted_reg, kernel, record=None,
               row0: int = 0, nrows: int | None = None, reuse_shadow: bool = False,
               nnz: int | None = None, peers=None, implicit=None):
        """Gram(+bias) -> solve for rows [row0, row0+nrows) of the view, block by
        block, solutions written into tg (rows indexed like the view).  ``nnz``:
        ratings in those rows (default: all of the view's), which picks the
        fused kernel's CTA shape.  ``peers``: device int64 tensor of replica
        pointers (offset like ``tg``) that the fused kernel also stores each
        solved row into (multi-GPU, distributed.ShardedALS).  ``implicit``:
        (alpha, gram_full) -- the implicit-feedback system (implicit.py:63-84)
        on the fused route: per-rating operand weights alpha*r, confidences
        1 + alpha*r, base F^T F (device fp32, f rows of stride roundup4(f)),
        plain lambda; rows without ratings are left to the caller."""
        f, solver = self.f, self.solver
        nrows = self.nrows if nrows is None else nrows
        st = nat.stream_ptr()
        tc = kernel.startswith("tc")
        if record is not None and tc:
            es0 = torch.cuda.Event(enable_timing=True)
            es0.record()
        if tc and reuse_shadow and self.shadow is not None:  # same fixed factors as the last call
            shadow, lo = self.shadow, self._shadow_lo
        else:
            shadow, lo = self._shadow(fx, split=kernel == "tc_split") if tc else (None, None)
            self._shadow_lo = lo
        if record is not None and tc:
            es1 = torch.cuda.Event(enable_timing=True)
            es1.record()
            record.setdefault("shadow16", []).append((es0, es1))
        if kernel == "tc" and solver.method == "cg":
            # fused: Gram in TMEM -> CG in registers -> x, one launch, no workspace
            if record is not None:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
            nnz = int(values.numel()) if nnz is None else int(nnz)
            common = (nat.ptr(indptr) + 8 * row0, nat.ptr(indices), nat.ptr(values), nrows, nnz,
                      nat.ptr(shadow), fx.shape[0], self.w16, f, float(lam), int(bool(weighted_reg)),
                      nat.ptr(tg) + 4 * row0 * f)
            tail = (int(solver.cg_iters), float(solver.cg_tol), nat.ptr(self.flags) + 4,
                    nat.ptr(self.flags), st)
            if peers is not None and peers.numel() and row0:
                raise DataError("peer stores take whole views (row0 == 0)")
            npeers = int(peers.numel()) if peers is not None else 0
            # long rows over a fixed side larger than L2: the kernel runs two passes
            # and parks each row's partial Gram in this workspace (~1 GB for the
            # Netflix item side); other views never touch it
            ws, wsb = None, 0
            if nnz >= 1024 * max(nrows, 1) and fx.shape[0] * self.w16 * 2 > (48 << 20):
                wsb = int(nat.lib().cmf_fused_cg_workspace_bytes(nrows, f))
                ws = _WS.get(self.dev, wsb, key="fused2p")
            if implicit is not None:
                alpha, gram_full = implicit
                nat.call("cmf_fused_cg_update_implicit", *common[:9], float(alpha), float(lam),
                         nat.ptr(gram_full), common[11], nat.ptr(peers) if npeers else None, npeers,
                         tail[0], tail[1], tail[2], tail[3], nat.ptr(ws), wsb, tail[4])
            else:
                nat.call("cmf_fused_cg_update_ws", *common, nat.ptr(peers) if npeers else None, npeers,
                         tail[0], tail[1], tail[2], tail[3], nat.ptr(ws), wsb, tail[4])
            if ws is not None and f <= 104:
                nat.LAUNCHES[0] += 2  # two passes: the segment split + the second fused launch
            if record is not None:
                e1.record()
                record.setdefault("fused_tc_cg", []).append((e0, e1))
            return
        self._workspace()
        for r0 in range(row0, row0 + nrows, self.rows_blk):
            nb = min(self.rows_blk, row0 + nrows - r0)
            if record is not None:
                e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                e0.record()
            if tc and lo is not None:
                # split-precision (fp32) Gram: long rows over a fixed side whose hi + lo
                # shadow exceeds L2 run in passes over fixed-side id ranges (the
                # segment bounds live in a small workspace; see cmf_gram_assemble_tc_ws)
                nnz_b = (int(values.numel()) if nnz is None else int(nnz)) * nb // max(nrows, 1)
                wsb = int(nat.lib().cmf_gram_tc_workspace_bytes(nb, nnz_b, fx.shape[0], f, 1))
                ws = _WS.get(self.dev, wsb, key="gram_passes") if wsb else None
                nat.call("cmf_gram_assemble_tc_ws", nat.ptr(indptr) + 8 * r0, nat.ptr(indices),
                         nat.ptr(values), nb, nnz_b, nat.ptr(shadow), lo, fx.shape[0], SPLIT_SCALE, self.w16, f,
                         float(lam), int(bool(weighted_reg)), nat.PREC[solver.precision],
                         nat.ptr(self.a_ws), self.stride, nat.ptr(self.b_ws),
                         nat.ptr(self.nu_ws), nat.ptr(self.flags), nat.ptr(ws), wsb, st)
                if wsb:  # P passes + P - 1 segment splits
                    nat.LAUNCHES[0] += 2 * (wsb // (8 * nb))
            elif tc:
                nat.call("cmf_gram_assemble_tc", nat.ptr(indptr) + 8 * r0, nat.ptr(indices),
                         nat.ptr(values), nb, nat.ptr(shadow), lo, fx.shape[0], SPLIT_SCALE, self.w16, f,
                         float(lam),
                         int(bool(weighted_reg)), None, nat.PREC[solver.precision],
                         nat.ptr(self.a_ws), self.stride, nat.ptr(self.b_ws),
                         nat.ptr(self.nu_ws), nat.ptr(self.flags), st)
            else:
                nat.call("cmf_gram_assemble", nat.ptr(indptr) + 8 * r0, nat.ptr(indices), None,
                         nat.ptr(values), nb, nat.ptr(fx), fx.shape[0], f, float(lam),
                         int(bool(weighted_reg)), None, nat.PREC[solver.precision],
                         nat.GRAM_KERNELS[kernel], nat.ptr(self.a_ws), self.stride,
                         nat.ptr(self.b_ws), nat.ptr(self.nu_ws), nat.ptr(self.flags), st)
            if record is not None:
                e1.record()
            tgt = nat.ptr(tg) + 4 * r0 * f
            if solver.method == "cg":
                nat.call("cmf_batch_cg", nat.ptr(self.a_ws), nat.PREC[solver.precision],
                         self.stride, nat.ptr(self.b_ws), tgt, None, float(solver.cg_tol),
                         nat.ptr(self.nu_ws), nb, f, int(solver.cg_iters),
                         nat.ACCUM[solver.accum], tgt, None, None, nat.ptr(self.flags) + 4, st)
            else:
                nat.call("cmf_batch_cholesky", nat.ptr(self.a_ws), self.stride,
                         nat.ptr(self.b_ws), nat.ptr(self.nu_ws), nb, f,
                         nat.ACCUM[solver.accum], tgt, None, nat.ptr(self.flags) + 8, st)
            if record is not None:
                e2.record()
                record.setdefault("gram_" + ("tc" if tc else kernel), []).append((e0, e1))
                record.setdefault("solve_" + solver.method, []).append((e1, e2))

    def read_flags(self):
        fl = self.flags.cpu().tolist()  # synchronises
        self.flags.zero_()
        return fl


def resolve_events(record: dict) -> dict:
    """{name: [(start, end) events]} -> {name: [ms, ...]} (synchronises)."""
    out = {}
    for name, pairs in record.items():
        out[name] = [a.elapsed_time(b) for a, b in pairs]
    return out


def update_side(view: RowView, fixed, target, lam: float, solver: SolverConfig,
                tiles: TileConfig | None = None, weighted_reg: bool = True, *,
                gram_kernel: str | None = None, workspace_bytes: int | None = None):
    """One half-update; writes the solutions into ``target`` in place."""
    if target.shape[0] != view.nrows or fixed.shape[1] != target.shape[1]:
        raise DataError("factor matrices do not match the ratings view")
    if view.ncols != fixed.shape[0]:
        raise DataError(f"feature matrix has {fixed.shape[0]} rows, ratings expect {view.ncols}")
    if tiles is not None and not isinstance(tiles, TileConfig):
        raise DataError("tiles must be a TileConfig")
    kernel = resolve_gram_kernel(gram_kernel, solver, int(fixed.shape[1]))
    host = not nat.is_device(target)
    dev = nat.device()
    if (host and kernel == "tc" and solver.method == "cg"
            and _all_pinned(view.indptr, view.indices, view.values, fixed, target)
            and int(view.nrows) >= STREAM_MIN_ROWS):
        return _update_side_streamed(view, fixed, target, lam, solver, weighted_reg, dev)
    indptr, indices, values = _view_dev(view, dev)
    fx = nat.to_dev(fixed, torch.float32, dev)
    tg = nat.to_dev(target, torch.float32, dev) if host else target
    if not (tg.is_contiguous() and tg.dtype == torch.float32):
        raise DataError("device target must be a contiguous float32 tensor")
    nrows, f = int(view.nrows), int(fx.shape[1])
    plan = HalfUpdatePlan(nrows, f, solver, dev, workspace_bytes)
    rec = {}
    plan.launch(indptr, indices, values, fx, tg, lam, weighted_reg, kernel, rec)
    fl = plan.read_flags()
    if fl[0]:
        raise NumericalError(_OVERFLOW_MSG)
    if fl[2]:
        raise _locate_singular(indptr, indices, values, nrows, fx, f, lam, weighted_reg,
                               kernel, solver)
    times = PhaseTimes()
    for name, ms in resolve_events(rec).items():
        if name.startswith("gram") or name == "shadow16":
            times.accumulate += sum(ms) / 1e3
        elif name.startswith("fused"):
            # one kernel does both; report it under accumulate (the Gram dominates)
            times.accumulate += sum(ms) / 1e3
        else:
            times.solve += sum(ms) / 1e3
    if host:
        if isinstance(target, torch.Tensor):
            target.copy_(tg)
        else:
            target[...] = nat.to_host(tg)
    return times, nrows * packed_size(f) * plan.esize, int(fl[1])


_OVERFLOW_MSG = ("Gram entries overflow binary16 range (+-65504); "
                 "rescale the ratings before using half precision")

STREAM_CHUNKS = int(os.environ.get("CMF_STREAM_CHUNKS", "8"))
STREAM_MIN_ROWS = 4096


def _all_pinned(*ts) -> bool:
    return all(isinstance(t, torch.Tensor) and t.device.type == "cpu" and t.is_pinned() and t.is_contiguous()
               for t in ts)


def _update_side_streamed(view: RowView, fixed, target, lam, solver, weighted_reg, dev):
    """update_side for pinned host buffers on the fused CG route, with the PCIe
    transfers overlapped: the fixed factors and indptr go first, then the rows
    are cut into STREAM_CHUNKS nnz-balanced chunks; chunk k's indices / ratings
    / warm start are copied on a copy stream while the fused kernel solves chunk
    k-1, and each solved chunk of ``target`` is copied back on a third stream.
    Same results as the unchunked call (each row's system is independent)."""
    f = int(fixed.shape[1])
    nrows = int(view.nrows)
    comp = torch.cuda.current_stream(dev)
    h2d = torch.cuda.Stream(dev)
    d2h = torch.cuda.Stream(dev)
    indptr_h = view.indptr.to(torch.int64) if view.indptr.dtype != torch.int64 else view.indptr
    ptr_np = indptr_h.numpy()
    nnz = int(ptr_np[-1])
    k = max(1, min(STREAM_CHUNKS, nrows // 1024))
    cuts = np.searchsorted(ptr_np, np.linspace(0, nnz, k + 1)[1:-1], side="left")
    bounds = np.unique(np.concatenate([[0], cuts, [nrows]]))
    indptr = torch.empty(nrows + 1, dtype=torch.int64, device=dev)
    indices = torch.empty(nnz, dtype=torch.int32, device=dev)
    values = torch.empty(nnz, dtype=torch.float32, device=dev)
    fx = torch.empty(fixed.shape, dtype=torch.float32, device=dev)
    tg = torch.empty(target.shape, dtype=torch.float32, device=dev)
    plan = HalfUpdatePlan(nrows, f, solver, dev)
    # the buffers above were allocated on the compute stream: a block the caching
    # allocator recycled may still be read by a kernel queued there
    h2d.wait_stream(comp)
    with torch.cuda.stream(h2d):
        fx.copy_(fixed, non_blocking=True)
        indptr.copy_(indptr_h, non_blocking=True)
        ev_base = torch.cuda.Event()
        ev_base.record(h2d)
        evs = []
        for r0, r1 in zip(bounds[:-1], bounds[1:]):
            p0, p1 = int(ptr_np[r0]), int(ptr_np[r1])
            indices[p0:p1].copy_(view.indices[p0:p1], non_blocking=True)
            values[p0:p1].copy_(view.values[p0:p1], non_blocking=True)
            tg[r0:r1].copy_(target[r0:r1], non_blocking=True)
            e = torch.cuda.Event()
            e.record(h2d)
            evs.append(e)
    comp.wait_event(ev_base)
    rec = {}
    for ci, (r0, r1) in enumerate(zip(bounds[:-1], bounds[1:])):
        comp.wait_event(evs[ci])
        plan.launch(indptr, indices, values, fx, tg, lam, weighted_reg, "tc", rec,
                    row0=int(r0), nrows=int(r1 - r0), reuse_shadow=ci > 0,
                    nnz=int(ptr_np[r1] - ptr_np[r0]))
        done = torch.cuda.Event()
        done.record(comp)
        d2h.wait_event(done)
        with torch.cuda.stream(d2h):
            target[r0:r1].copy_(tg[r0:r1], non_blocking=True)
    # keep the device buffers alive until the copies that use them have run
    for t in (indptr, indices, values, fx, tg):
        t.record_stream(h2d)
        t.record_stream(d2h)
    d2h.synchronize()
    fl = plan.read_flags()
    if fl[0]:
        raise NumericalError(_OVERFLOW_MSG)
    times = PhaseTimes()
    for name, ms in resolve_events(rec).items():
        times.accumulate += sum(ms) / 1e3
    return times, nrows * packed_size(f) * plan.esize, int(fl[1])


def _locate_singular(indptr, indices, values, nrows, fx, f, lam, weighted_reg, kernel, solver):
    """Recompute the side with per-system info to name the failing rows, numbered
    among rows with n_u > 0 as the reference's compacted batch does (als.py:69-71)."""
    dev = fx.device
    solver = with_accum(solver, "fp32")
    P = packed_size(f)
    a = torch.empty((nrows, P), dtype=torch.float32, device=dev)
    b = torch.empty((nrows, f), dtype=torch.float32, device=dev)
    nu = torch.empty(nrows, dtype=torch.int64, device=dev)
    # the SIMT Gram names the rows for every route (the tensor-core kernels have
    # their own entry point; which rows are singular does not depend on it)
    simt = kernel if kernel in ("bitwise", "fma") else "fma"
    nat.call("cmf_gram_assemble", nat.ptr(indptr), nat.ptr(indices), None, nat.ptr(values), nrows,
             nat.ptr(fx), fx.shape[0], f, float(lam), int(bool(weighted_reg)), None, 0,
             nat.GRAM_KERNELS[simt], nat.ptr(a), P, nat.ptr(b), nat.ptr(nu), None,
             nat.stream_ptr())
    out = torch.empty_like(b)
    info = torch.zeros(nrows, dtype=torch.int32, device=dev)
    nat.call("cmf_batch_cholesky", nat.ptr(a), P, nat.ptr(b), nat.ptr(nu), nrows, f,
             nat.ACCUM[solver.accum], nat.ptr(out), nat.ptr(info), None, nat.stream_ptr())
    sel = torch.nonzero(nu > 0).flatten()
    bad = torch.nonzero(info[sel]).flatten()
    return _singular_error(bad.cpu().tolist())


# ------------------------------------------------------------------ evaluation

def _ratings_dev(r):
    return r if isinstance(r, DeviceRatings) else r.to_device()


def _reduce_buf(dev):
    return torch.empty(nat.REDUCE_SLOTS + 1, dtype=torch.float64, device=dev)


def objective(x, theta, ratings, lam: float, weighted: bool = True) -> float:
    """Weighted-lambda training objective in float64 (als.py:77-97), on the GPU."""
    dev = nat.device()
    r = _ratings_dev(ratings)
    xd, td = nat.to_dev(x, torch.float32, dev), nat.to_dev(theta, torch.float32, dev)
    f = int(xd.shape[1])
    out = _reduce_buf(dev)
    res = torch.empty(3, dtype=torch.float64, device=dev)
    st = nat.stream_ptr()
    nat.call("cmf_sq_error_csr", nat.ptr(r.row_ptr), nat.ptr(r.col_idx), nat.ptr(r.csr_val),
             r.m, nat.ptr(xd), nat.ptr(td), f, nat.ptr(out), st)
    res[0] = out[0]
    nat.call("cmf_weighted_sqnorm", nat.ptr(r.row_ptr) if weighted else None, nat.ptr(xd), r.m, f,
             nat.ptr(out), st)
    res[1] = out[0]
    nat.call("cmf_weighted_sqnorm", nat.ptr(r.col_ptr) if weighted else None, nat.ptr(td), r.n, f,
             nat.ptr(out), st)
    res[2] = out[0]
    data, rx, rt = res.cpu().tolist()
    return data + lam * (rx + rt)


def rmse(x, theta, test: Triples) -> float:
    """Test RMSE without clamping (als.py:100-107), on the GPU."""
    if len(test) == 0:
        raise DataError("cannot evaluate RMSE on an empty test set")
    dev = nat.device()
    xd, td = nat.to_dev(x, torch.float32, dev), nat.to_dev(theta, torch.float32, dev)
    u = nat.to_dev(test.user, torch.int64, dev)
    v = nat.to_dev(test.item, torch.int64, dev)
    r = nat.to_dev(test.rating, torch.float32, dev)
    out = _reduce_buf(dev)
    nat.call("cmf_sq_error", nat.ptr(u), nat.ptr(v), 1, nat.ptr(r), u.shape[0], nat.ptr(xd),
             nat.ptr(td), int(xd.shape[1]), nat.ptr(out), nat.stream_ptr())
    return float(np.sqrt(out[0].item() / u.shape[0]))


# ------------------------------------------------------------------- training

def train(train_ratings, test, cfg: AlsConfig):
    """ALS for cfg.epochs or until test RMSE <= cfg.target_rmse (als.py:110-157).

    Host SparseRatings in -> numpy factors out; DeviceRatings in -> CUDA tensors
    out.  Returns (X, Theta, TrainReport).
    """
    host = isinstance(train_ratings, SparseRatings)
    dev = nat.device()
    r = _ratings_dev(train_ratings)
    m, n = r.m, r.n
    x = nat.to_dev(init_factors(m, cfg.f, cfg.init_scale, [cfg.seed, 0]), torch.float32, dev)
    theta = nat.to_dev(init_factors(n, cfg.f, cfg.init_scale, [cfg.seed, 1]), torch.float32, dev)
    test_d = test.to_device() if test is not None and len(test) else None
    nu_rows = torch.diff(r.row_ptr)
    nu_cols = torch.diff(r.col_ptr)
    config = asdict(cfg)
    config["engine"] = "als"
    report = TrainReport(engine="als", config=config,
                         cold_rows=int((nu_rows == 0).sum().item()),
                         cold_cols=int((nu_cols == 0).sum().item()),
                         flops=roofline_estimate(m, n, max(r.nnz, 1), cfg.f,
                                                 f_s=cfg.solver.cg_iters))
    csr, csc = r.csr_view(), r.csc_view()
    stop = "epochs"
    for epoch in range(cfg.epochs):
        times = PhaseTimes()
        tx, bytes_x, brk_x = update_side(csr, theta, x, cfg.lam, cfg.solver, cfg.tiles,
                                         cfg.weighted_reg, gram_kernel=cfg.gram_kernel)
        times += tx
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        obj_mid = objective(x, theta, r, cfg.lam, cfg.weighted_reg)
        e1.record()
        tt, bytes_t, brk_t = update_side(csc, x, theta, cfg.lam, cfg.solver, cfg.tiles,
                                         cfg.weighted_reg, gram_kernel=cfg.gram_kernel)
        times += tt
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2.record()
        obj = objective(x, theta, r, cfg.lam, cfg.weighted_reg)
        test_rmse = rmse(x, theta, test_d) if test_d is not None else None
        e3.record()
        e3.synchronize()
        times.eval += (e0.elapsed_time(e1) + e2.elapsed_time(e3)) / 1e3
        report.gram_bytes_x, report.gram_bytes_theta = bytes_x, bytes_t
        report.add_epoch(EpochRecord.from_phases(epoch, obj, times, objective_mid=obj_mid,
                                                 rmse=test_rmse, cg_breakdowns=brk_x + brk_t))
        if cfg.target_rmse is not None and test_rmse is not None and test_rmse <= cfg.target_rmse:
            stop = "target_rmse"
            break
    report.stop_reason = stop
    if host:
        return nat.to_host(x), nat.to_host(theta), report
    return x, theta, report
