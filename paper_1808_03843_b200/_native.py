"""ctypes binding of libcmf_b200.so (include/cmf_b200.h) plus the host-side
plumbing every public function shares: moving numpy inputs to the device,
passing torch CUDA tensors as raw pointers with the current stream, and
mapping C status codes to the reference's exception tree (errors.py).

There is no CPU fallback: if the library or a CUDA device is missing, every
compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np
import torch

from .errors import CmfError, DataError, NumericalError, SingularSystemError

_PKG = os.path.dirname(os.path.abspath(__file__))
# CMF_LIB_PATH: load another build of the library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("CMF_LIB_PATH") or os.path.join(_PKG, "libcmf_b200.so")

CMF_OK, CMF_EINVAL, CMF_EOVERFLOW, CMF_ESINGULAR, CMF_ECUDA = 0, 1, 2, 3, 4
PREC = {"fp32": 0, "fp16": 1}
GRAM_KERNELS = {"bitwise": 0, "fma": 1, "tc": 2, "tc_unfused": 2, "tc_split": 2}
ACCUM = {"fp32": 0, "fp64": 1}

_vp, _i32, _i64, _f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double

_SIGNATURES = {
    "cmf_last_error": (ctypes.c_char_p, []),
    "cmf_version": (ctypes.c_int, []),
    "cmf_device_info": (ctypes.c_int, [_vp, _vp, _vp]),
    "cmf_gram_assemble": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _vp, _i64, _i32, _f64, _i32,
                                         _vp, _i32, _i32, _vp, _i64, _vp, _vp, _vp, _vp]),
    "cmf_gram_assemble_tc": (ctypes.c_int, [_vp, _vp, _vp, _i64, _vp, _vp, _i64, ctypes.c_float, _i32, _i32,
                                            _f64, _i32, _vp, _i32, _vp, _i64, _vp, _vp, _vp, _vp]),
    "cmf_gram_assemble_tc_ws": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _vp, _vp, _i64, ctypes.c_float, _i32,
                                               _i32, _f64, _i32, _i32, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _vp]),
    "cmf_gram_tc_workspace_bytes": (ctypes.c_int64, [_i64, _i64, _i64, _i32, _i32]),
    "cmf_factors_to_half_split": (ctypes.c_int, [_vp, _i64, _i32, _vp, _vp, _i32, ctypes.c_float,
                                                 _vp, _vp]),
    "cmf_tc_width": (ctypes.c_int, [_i32]),
    "cmf_debug_trace": (ctypes.c_int, [_vp]),
    "cmf_ipc_export": (ctypes.c_int, [_vp, _vp, _vp]),
    "cmf_ipc_open": (ctypes.c_int, [_vp, _i64, _vp]),
    "cmf_ipc_close": (ctypes.c_int, [_vp, _i64]),
    "cmf_fused_cg_update": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _i32, _i32, _f64, _i32, _vp,
                                           _i32, _f64, _vp, _vp, _vp]),
    "cmf_fused_cg_update_peers": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _i32, _i32, _f64, _i32, _vp,
                                                 _vp, _i32, _i32, _f64, _vp, _vp, _vp]),
    "cmf_fused_cg_update_ws": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _i32, _i32, _f64, _i32,
                                              _vp, _vp, _i32, _i32, _f64, _vp, _vp, _vp, _i64, _vp]),
    "cmf_fused_cg_workspace_bytes": (ctypes.c_int64, [_i64, _i32]),
    "cmf_fused_base_ld": (ctypes.c_int32, [_i32]),
    "cmf_fused_cg_pass": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _i32, _i32, _f64, _i32, _vp, _vp, _i32,
                                         _vp, _vp, _i32, _i32, _f64, _vp, _vp, _vp]),
    "cmf_fused_cg_partial_floats": (ctypes.c_int64, [_i64, _i32]),
    "cmf_fused_cg_update_implicit": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _i32, _i32, _f64, _f64,
                                                    _vp, _vp, _vp, _i32, _i32, _f64, _vp, _vp, _vp, _i64, _vp]),
    "cmf_factors_to_half": (ctypes.c_int, [_vp, _i64, _i32, _vp, _i32, _vp, _vp]),
    "cmf_spmm_bias": (ctypes.c_int, [_vp, _vp, _vp, _i64, _vp, _i64, _i32, _vp, _vp]),
    "cmf_batch_cg": (ctypes.c_int, [_vp, _i32, _i64, _vp, _vp, _vp, _f64, _vp, _i64, _i32, _i32,
                                    _i32, _vp, _vp, _vp, _vp, _vp]),
    "cmf_batch_cholesky": (ctypes.c_int, [_vp, _i64, _vp, _vp, _i64, _i32, _i32, _vp, _vp, _vp,
                                          _vp]),
    "cmf_half_update": (ctypes.c_int, [_vp, _vp, _vp, _i64, _vp, _i64, _vp, _i32, _f64, _i32,
                                       _i32, _i32, _i32, _i32, _f64, _i32, _vp, _i64, _vp, _vp,
                                       _i64, _vp, _vp, _vp]),
    "cmf_pack_half": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp]),
    "cmf_sq_error": (ctypes.c_int, [_vp, _vp, _i32, _vp, _i64, _vp, _vp, _i32, _vp, _vp]),
    "cmf_sq_error_csr": (ctypes.c_int, [_vp, _vp, _vp, _i64, _vp, _vp, _i32, _vp, _vp]),
    "cmf_weighted_sqnorm": (ctypes.c_int, [_vp, _vp, _i64, _i32, _vp, _vp]),
    "cmf_predict_pairs": (ctypes.c_int, [_vp, _vp, _i32, _i64, _vp, _vp, _i32, _vp, _vp]),
    "cmf_build": (ctypes.c_int, [_vp, _vp, _i32, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64,
                                 _vp, _vp, _vp]),
    "cmf_build_workspace_bytes": (ctypes.c_int64, [_i64]),
    "cmf_dense_gram_workspace_bytes": (ctypes.c_int64, [_i64, _i32, _i32]),
    "cmf_dense_gram": (ctypes.c_int, [_vp, _i64, _i32, _i32, _vp, _vp, _i64, _vp]),
    "cmf_implicit_loss_csr": (ctypes.c_int, [_vp, _vp, _vp, _i64, _vp, _vp, _i32, _f64, _vp, _vp]),
    "cmf_group_workspace_bytes": (ctypes.c_int64, [_i64]),
    "cmf_group_rows": (ctypes.c_int, [_vp, _vp, _i32, _i64, _i64, _vp, _vp, _vp, _i64, _vp]),
    "cmf_mpr_count": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp, _i64, _i32, _vp, _vp]),
    "cmf_gen_truth": (ctypes.c_int, [ctypes.c_uint64, _i32, _i64, _i32, _vp, _vp]),
    "cmf_gen_count": (ctypes.c_int, [ctypes.c_uint64, _i64, _i64, ctypes.c_uint64, ctypes.c_uint64, _i32, _i64,
                                     _i64, _i64, _i64, _vp, _vp, _vp, _vp]),
    "cmf_gen_fill": (ctypes.c_int, [ctypes.c_uint64, _i64, _i64, _i32, ctypes.c_uint64, ctypes.c_uint64,
                                    ctypes.c_float, _i32, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                    _vp, _vp, _vp]),
}
EXPORTED = tuple(_SIGNATURES)
REDUCE_SLOTS = 1024  # eval.cu: doubles an eval `out` buffer must hold

_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load libcmf_b200.so and declare every exported signature (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise CmfError(f"native library missing: {path} (run __graft_entry__.build())")
            L = ctypes.CDLL(path)
            for name, (res, args) in _SIGNATURES.items():
                # an older build (A/B timing via CMF_LIB_PATH) may lack newer entry
                # points; they fail when called (tests/test_abi_host.py checks that
                # the current build exports every one)
                if not hasattr(L, name):
                    continue
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def lib():
    if _lib is None:
        load_library()
    if not torch.cuda.is_available():
        raise CmfError("paper_1808_03843_b200 needs a CUDA device (B200, sm_100a); "
                       "there is no CPU fallback")
    return _lib


def check(rc: int, what: str = ""):
    if rc == CMF_OK:
        return
    msg = (_lib.cmf_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == CMF_EINVAL:
        raise DataError(text)
    if rc == CMF_EOVERFLOW:
        raise NumericalError(text)
    if rc == CMF_ESINGULAR:
        raise SingularSystemError(text)
    raise CmfError(text)


# Kernel-launching entry points called since the counter was last reset (the
# benchmark's "gpu_launches" claim counts launches of OUR kernels).
_LAUNCH_COST = {"cmf_factors_to_half_split": 1, "cmf_fused_cg_update": 1, "cmf_fused_cg_update_peers": 1, "cmf_fused_cg_update_ws": 1, "cmf_fused_cg_update_implicit": 1, "cmf_fused_cg_pass": 1, "cmf_dense_gram": 2, "cmf_implicit_loss_csr": 2, "cmf_group_rows": 6, "cmf_mpr_count": 1, "cmf_gen_truth": 1, "cmf_gen_count": 3, "cmf_gen_fill": 1, "cmf_gram_assemble": 1, "cmf_gram_assemble_tc": 1, "cmf_gram_assemble_tc_ws": 1, "cmf_factors_to_half": 1, "cmf_spmm_bias": 1, "cmf_batch_cg": 1,
                "cmf_batch_cholesky": 1, "cmf_pack_half": 1, "cmf_sq_error": 2,
                "cmf_sq_error_csr": 2, "cmf_weighted_sqnorm": 2, "cmf_predict_pairs": 1}
LAUNCHES = [0]


def call(name: str, *args):
    fn = getattr(lib(), name)
    check(fn(*args), name)
    LAUNCHES[0] += _LAUNCH_COST.get(name, 0)


# ---------------------------------------------------------------- tensors

def tc_width(f: int) -> int:
    """Row width (halves) of the binary16 factor shadow the tensor-core Gram reads
    (= cmf_tc_width: f rounded up to 8, so every row is 16-byte aligned for TMA)."""
    return ((f + 7) // 8) * 8


def device() -> torch.device:
    lib()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


_dummies = {}


def ptr(t) -> int | None:
    """Raw device address; None stays NULL (the ABI's "absent" marker).  An
    empty tensor has data_ptr() == 0, which the ABI would read as "absent", so
    it is given a valid (never dereferenced) 16-byte scratch address instead."""
    if t is None:
        return None
    p = t.data_ptr()
    if p == 0 and t.numel() == 0:
        key = t.device
        if key not in _dummies:
            _dummies[key] = torch.zeros(4, dtype=torch.float32, device=key)
        p = _dummies[key].data_ptr()
    return p


def is_device(a) -> bool:
    return isinstance(a, torch.Tensor) and a.is_cuda


def to_dev(a, dtype: torch.dtype, dev=None) -> torch.Tensor:
    """numpy / torch -> contiguous CUDA tensor of `dtype` (no copy when it already is)."""
    dev = dev or device()
    if isinstance(a, torch.Tensor):
        if a.device.type == "cpu" and a.is_pinned():
            # pinned host buffers (the e2e path): async DMA, no staging copy
            return a.contiguous().to(dev, non_blocking=True).to(dtype)
        t = a.to(device=dev, dtype=dtype)
        return t.contiguous()
    arr = np.ascontiguousarray(a)
    t = torch.from_numpy(arr)
    if t.dtype != dtype:
        t = t.to(dtype)
    if arr.nbytes >= (1 << 20):
        t = t.pin_memory()
        return t.to(dev, non_blocking=True)
    return t.to(dev)


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()
