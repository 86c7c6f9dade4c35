"""Worker-pool control: the reference's set_workers / get_workers names
(parallel.py:11-27, exported at cmf/__init__.py:23).

The reference sizes a numba thread pool that its row-parallel kernels draw
from.  Here every row-parallel kernel runs on the GPU, with its parallelism
fixed by the launch grid (one persistent CTA per SM, or a grid sized to the
batch); no host thread pool computes anything on the hot path.  The knob is
kept so that callers of the reference API (and its tests) run unchanged: it
validates and records the request, clamped to the host's CPU count as the
reference clamps to NUMBA_NUM_THREADS, and results never depend on it --
which the reference also promises ("bitwise independent of the worker
count").
"""

from __future__ import annotations

import os

_WORKERS = os.cpu_count() or 1


def set_workers(n: int) -> int:
    """Record a worker count (clamped to the host CPU count); returns it.
    ValueError for n < 1, as the reference."""
    global _WORKERS
    if n < 1:
        raise ValueError("worker count must be >= 1")
    _WORKERS = min(int(n), os.cpu_count() or 1)
    return _WORKERS


def get_workers() -> int:
    """The recorded worker count."""
    return _WORKERS
