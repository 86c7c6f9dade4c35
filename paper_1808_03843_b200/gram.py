"""Per-row normal-equation assembly (K1 Gram + K2 bias) on the B200.

Mirrors the reference's gram.py (gram.py:39-381): same types, packed layout,
names and errors.  ``assemble_side`` launches ONE fused kernel per call
(cmf_gram_assemble) that gathers each row's factor rows, accumulates the
packed lower triangle, adds the regulariser, stores fp32 or fp16 (RNE) and
accumulates the right-hand side in float64.

Gram kernels (``kernel=``):
  "bitwise" -- float32 mul-then-add in CSR order: bit-identical to the
               reference's numba loop.  Default for ``assemble_side``.
  "fma"     -- fused multiply-add (one rounding per update), 2x fewer issue
               slots; the default inside ``update_side``/``train``.
  "tc"      -- tcgen05 tensor-core path (fp16 operands, fp32 TMEM
               accumulation) for the CG route.

Inputs may be numpy arrays (results come back as numpy, like the reference)
or CUDA tensors (results stay on the device).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .data import RowView, SparseRatings
from .errors import DataError, NumericalError
from .report import PhaseTimes

DEFAULT_KERNEL = os.environ.get("CMF_GRAM_KERNEL", "bitwise")


@dataclass
class TileConfig:
    """The reference's tiling knobs (gram.py:39-51).  Validated and recorded;
    the GPU kernel's register tiling is fixed by f, and -- exactly as in the
    reference -- results do not depend on these values."""

    tile: int = 8
    batch: int = 32

    def __post_init__(self):
        if self.tile < 1:
            raise DataError("tile must be >= 1")
        if self.batch < 1:
            raise DataError("batch must be >= 1")


def _is_half(a) -> bool:
    return a.dtype in (np.float16, torch.float16)


def _nbytes(a) -> int:
    return int(a.numel() * a.element_size()) if isinstance(a, torch.Tensor) else int(a.nbytes)


@dataclass
class GramSystem:
    f: int
    a_lower: object
    b: object = None
    n_u: int = 0

    @property
    def precision(self) -> str:
        return "fp16" if _is_half(self.a_lower) else "fp32"

    @property
    def is_empty(self) -> bool:
        return self.n_u == 0

    def full(self) -> np.ndarray:
        a = self.a_lower.cpu().numpy() if isinstance(self.a_lower, torch.Tensor) else self.a_lower
        return unpack_lower(a, self.f)


@dataclass
class GramBatch:
    f: int
    a_lower: object  # (N, P) float32 / float16
    b: object        # (N, f) float32
    n_u: object      # (N,) int64

    def __len__(self):
        return int(self.a_lower.shape[0])

    def __getitem__(self, i: int) -> GramSystem:
        return GramSystem(self.f, self.a_lower[i], self.b[i], int(self.n_u[i]))

    @property
    def precision(self) -> str:
        return "fp16" if _is_half(self.a_lower) else "fp32"

    @property
    def a_nbytes(self) -> int:
        return _nbytes(self.a_lower)

    @classmethod
    def stack(cls, systems) -> "GramBatch":
        systems = list(systems)
        if not systems:
            raise DataError("cannot stack an empty sequence of systems")
        f = systems[0].f
        if any(s.f != f for s in systems):
            raise DataError("all systems in a batch must share f")
        if isinstance(systems[0].a_lower, torch.Tensor):
            return cls(f, torch.stack([s.a_lower for s in systems]),
                       torch.stack([s.b for s in systems]),
                       torch.tensor([s.n_u for s in systems], dtype=torch.int64,
                                    device=systems[0].a_lower.device))
        return cls(f, np.stack([s.a_lower for s in systems]), np.stack([s.b for s in systems]),
                   np.asarray([s.n_u for s in systems], dtype=np.int64))


def packed_size(f: int) -> int:
    return f * (f + 1) // 2


def pack_lower(full) -> np.ndarray:
    """Row-major packed lower triangle (index i*(i+1)/2 + j), float32."""
    full = np.asarray(full)
    rows, cols = np.tril_indices(full.shape[0])
    return np.ascontiguousarray(full[rows, cols], dtype=np.float32)


def unpack_lower(packed, f: int) -> np.ndarray:
    """Symmetric float32 matrix from packed lower storage."""
    rows, cols = np.tril_indices(f)
    out = np.zeros((f, f), dtype=np.float32)
    vals = np.asarray(packed).astype(np.float32)
    out[rows, cols] = vals
    out[cols, rows] = vals
    return out


def pack_half(a_lower):
    """float32 -> binary16, round to nearest even, on the GPU (cmf_pack_half).
    A finite entry that overflows raises NumericalError (gram.py:132-146)."""
    host = not nat.is_device(a_lower)
    src = nat.to_dev(a_lower, torch.float32)
    out = torch.empty(src.shape, dtype=torch.float16, device=src.device)
    flag = torch.zeros(1, dtype=torch.int32, device=src.device)
    nat.call("cmf_pack_half", nat.ptr(src), nat.ptr(out), src.numel(), nat.ptr(flag),
             nat.stream_ptr())
    if int(flag.item()):
        raise NumericalError("Gram entries overflow binary16 range (+-65504); "
                             "rescale the ratings before using half precision")
    return nat.to_host(out) if host else out


def _view_on_device(view: RowView):
    dev = nat.device()
    return (nat.to_dev(view.indptr, torch.int64, dev), nat.to_dev(view.indices, torch.int32, dev),
            nat.to_dev(view.values, torch.float32, dev))


def assemble_side(view: RowView, theta, lam: float, cfg: TileConfig | None = None,
                  precision: str = "fp32", weighted_reg: bool = True, a_weights=None,
                  b_weights=None, base_packed=None, *, kernel: str | None = None):
    """Every row's (A_u, b_u) for one half-update (gram.py:236-314).

    Returns (GramBatch, PhaseTimes); ``accumulate`` holds the fused kernel's
    device time (gather + Gram + store + bias run as one kernel).
    """
    if cfg is None:
        cfg = TileConfig()
    if precision not in ("fp32", "fp16"):
        raise DataError(f"unknown precision {precision!r}")
    kernel = kernel or DEFAULT_KERNEL
    if kernel not in nat.GRAM_KERNELS:
        raise DataError(f"unknown gram kernel {kernel!r}")
    f = int(theta.shape[1])
    if view.ncols != theta.shape[0]:
        raise DataError(f"feature matrix has {theta.shape[0]} rows, ratings expect {view.ncols}")
    P = packed_size(f)
    host = not nat.is_device(theta)
    dev = nat.device()
    indptr, indices, values = _view_on_device(view)
    th = nat.to_dev(theta, torch.float32, dev)
    base = None
    if base_packed is not None:
        base = nat.to_dev(base_packed, torch.float32, dev).reshape(-1)
        if base.shape[0] != P:
            raise DataError("base matrix does not match the factor dimension")
    aw = None if a_weights is None else nat.to_dev(a_weights, torch.float32, dev)
    bw = values if b_weights is None else nat.to_dev(b_weights, torch.float32, dev)
    nrows = int(view.nrows)
    dt = torch.float16 if precision == "fp16" else torch.float32
    b_out = torch.empty((nrows, f), dtype=torch.float32, device=dev)
    nu = torch.empty(nrows, dtype=torch.int64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    if kernel.startswith("tc"):
        if aw is not None:
            raise DataError("the tensor-core Gram kernel does not take a_weights")
        split = kernel == "tc_split"
        if split and precision != "fp32":
            raise DataError("the split-precision Gram stores fp32")
        stride = (P + 7) // 8 * 8  # 16-byte rows
        a_full = torch.empty((nrows, stride), dtype=dt, device=dev)
        w16 = nat.tc_width(f)
        # (+1 row: the all-zero row the gather reads for padding positions)
        shadow = torch.empty((2 if split else 1, th.shape[0] + 1, w16), dtype=torch.float16, device=dev)
        scale = 64.0
        if split:
            nat.call("cmf_factors_to_half_split", nat.ptr(th), th.shape[0], f, nat.ptr(shadow[0]),
                     nat.ptr(shadow[1]), w16, scale, nat.ptr(flag), nat.stream_ptr())
        else:
            nat.call("cmf_factors_to_half", nat.ptr(th), th.shape[0], f, nat.ptr(shadow[0]), w16,
                     nat.ptr(flag), nat.stream_ptr())
        nat.call("cmf_gram_assemble_tc", nat.ptr(indptr), nat.ptr(indices), nat.ptr(bw), nrows,
                 nat.ptr(shadow[0]), nat.ptr(shadow[1]) if split else None, th.shape[0], scale, w16, f,
                 float(lam), int(bool(weighted_reg)), nat.ptr(base),
                 nat.PREC[precision], nat.ptr(a_full), stride, nat.ptr(b_out), nat.ptr(nu),
                 nat.ptr(flag), nat.stream_ptr())
        a_out = a_full[:, :P]
    else:
        a_out = torch.empty((nrows, P), dtype=dt, device=dev)
        nat.call("cmf_gram_assemble", nat.ptr(indptr), nat.ptr(indices), nat.ptr(aw),
                 nat.ptr(bw), nrows, nat.ptr(th), th.shape[0], f, float(lam),
                 int(bool(weighted_reg)), nat.ptr(base), nat.PREC[precision],
                 nat.GRAM_KERNELS[kernel], nat.ptr(a_out), P, nat.ptr(b_out), nat.ptr(nu),
                 nat.ptr(flag), nat.stream_ptr())
    ev1.record()
    if int(flag.item()):
        raise NumericalError("Gram entries overflow binary16 range (+-65504); "
                             "rescale the ratings before using half precision")
    times = PhaseTimes(accumulate=ev0.elapsed_time(ev1) / 1e3)
    if host:
        return GramBatch(f, nat.to_host(a_out), nat.to_host(b_out), nat.to_host(nu)), times
    return GramBatch(f, a_out, b_out, nu), times


def _one_row(ratings: SparseRatings, u: int) -> RowView:
    view = ratings.csr_view()
    lo, hi = int(view.indptr[u]), int(view.indptr[u + 1])
    return RowView(np.array([0, hi - lo], dtype=np.int64), view.indices[lo:hi],
                   view.values[lo:hi], 1, view.ncols)


def get_hermitian(ratings: SparseRatings, u: int, theta, lam: float,
                  cfg: TileConfig | None = None, precision: str = "fp32",
                  weighted_reg: bool = True) -> GramSystem:
    """A_u for one CSR row (gram.py:317-331); ``b`` left unset."""
    batch, _ = assemble_side(_one_row(ratings, u), theta, lam, cfg=cfg, precision=precision,
                             weighted_reg=weighted_reg)
    sys_ = batch[0]
    sys_.b = None
    return sys_


def get_bias(ratings: SparseRatings, u: int, theta) -> np.ndarray:
    """b_u = sum_v r_uv theta_v (float64 accumulation -> float32), K2 alone."""
    if theta.shape[0] != ratings.n:
        raise DataError(f"feature matrix has {theta.shape[0]} rows, ratings expect {ratings.n}")
    view = _one_row(ratings, u)
    dev = nat.device()
    indptr, indices, values = _view_on_device(view)
    th = nat.to_dev(theta, torch.float32, dev)
    f = int(th.shape[1])
    out = torch.zeros((1, f), dtype=torch.float32, device=dev)
    nat.call("cmf_spmm_bias", nat.ptr(indptr), nat.ptr(indices), nat.ptr(values), 1, nat.ptr(th),
             th.shape[0], f, nat.ptr(out), nat.stream_ptr())
    return nat.to_host(out)[0]


def roofline_estimate(m: int, n: int, nnz: int, f: int, f_s: int = 6) -> dict:
    """The reference's flop/byte conventions (gram.py:347-381), FMA = 2 flops."""
    if min(m, n, nnz, f) <= 0:
        raise DataError("all roofline inputs must be positive")
    if f_s < 1:
        raise DataError("f_s must be >= 1")
    P = packed_size(f)
    systems = m + n
    return {
        "hermitian_flops": 2 * nnz * P,
        "hermitian_bytes": 4 * nnz * f + 4 * m * (P + f) + 8 * nnz,
        "solve_flops_exact": systems * f ** 3,
        "solve_flops_cg": systems * f_s * (2 * f * f + 10 * f),
        "sgd_flops": 12 * nnz * f,
        "sgd_bytes": 4 * nnz * (4 * f + 3),
        "hermitian_cm_ratio": float(f),
        "sgd_cm_ratio": 1.0,
    }
