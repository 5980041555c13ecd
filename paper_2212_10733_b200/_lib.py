"""ctypes binding of the C ABI in include/mlk_b200.h.

There is no fallback: if ``libmlk_b200.so`` is missing or no sm_100 device
is present, every call raises :class:`BackendError`.  Device buffers are
torch CUDA tensors (plumbing only); all compute happens in the library.
"""

from __future__ import annotations

import ctypes
import os
import functools
from pathlib import Path

import torch

from .errors import (BackendError, ConfigError, DimensionError, FormatError,
                     SizeMismatchError)

LIB_PATH = Path(os.environ.get("MLK_B200_LIB") or
               Path(__file__).resolve().parent / "libmlk_b200.so")

F_SELECTED, F_NONFINITE, F_RECHECK = 1, 2, 4
F_EXC_NEWTON, F_EXC_OVERFLOW, F_EXC_GATE = 8, 16, 32
F_EXCEPTION = F_NONFINITE | F_EXC_NEWTON | F_EXC_OVERFLOW | F_EXC_GATE


class MlkShard(ctypes.Structure):
    _fields_ = [("base", ctypes.c_int64), ("plane_stride", ctypes.c_int64),
                ("block", ctypes.c_int32), ("n_img", ctypes.c_int32),
                ("img_off", ctypes.c_int32), ("small_blas", ctypes.c_int32),
                ("mean", ctypes.c_double), ("std", ctypes.c_double), ("eb", ctypes.c_double),
                ("lossless", ctypes.c_int32), ("w_off", ctypes.c_int32),
                ("j0", ctypes.c_int32), ("pad", ctypes.c_int32)]


class MlkGrid(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int32), ("cols", ctypes.c_int32), ("D", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("mass", ctypes.c_double),
                ("vol", ctypes.c_void_p), ("vpar", ctypes.c_void_p), ("vperp2", ctypes.c_void_p),
                ("hmvol", ctypes.c_void_p), ("ash", ctypes.c_void_p),
                ("tree_cols", ctypes.c_void_p), ("s0", ctypes.c_double),
                ("s1", ctypes.c_double), ("s2", ctypes.c_double), ("sep", ctypes.c_int32),
                ("pad2", ctypes.c_int32), ("vcls", ctypes.c_double * 4)]


class MlkNewton(ctypes.Structure):
    _fields_ = [("step", ctypes.c_double), ("max_iter", ctypes.c_int32),
                ("retry", ctypes.c_int32), ("tol", ctypes.c_double), ("floor", ctypes.c_double),
                ("retry_step", ctypes.c_double), ("retry_max_iter", ctypes.c_int32),
                ("lam_f32", ctypes.c_int32), ("tau", ctypes.c_double)]


class MlkReportSeg(ctypes.Structure):
    _fields_ = [("flags", ctypes.c_void_p), ("status", ctypes.c_void_p),
                ("stats", ctypes.c_void_p), ("qoi", ctypes.c_void_p), ("fqoi", ctypes.c_void_p),
                ("fsse", ctypes.c_void_p), ("ferr", ctypes.c_void_p), ("order", ctypes.c_void_p),
                ("n", ctypes.c_int64)]


REPORT_NVALS = 20

assert ctypes.sizeof(MlkShard) == 72
assert ctypes.sizeof(MlkGrid) == 136

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_D = ctypes.c_double

# name -> argtypes (all return int status)
_SIGS = {
    "mlk_device_check": [],
    "mlk_newton_solve_batch": [_P, _P, _P, _I64, _I32, _D, _I32, _D, _P, _P, _P, _P],
    "mlk_zigzag_map": [_P, _P, _I64, _P],
    "mlk_zigzag_unmap": [_P, _P, _I64, _P],
    "mlk_varint_encode_batch": [_P, _P, _I32, _P, _P, _P, _P],
    "mlk_varint_decode_batch": [_P, _P, _P, _I32, _P, _P, _P, _P, _P],
    "mlk_pack_indices": [_P, _I64, _I32, _P, _P, _P],
    "mlk_unpack_indices": [_P, _I64, _I32, _P, _P],
    "mlk_zlib_compress6": [_P, _P, _P, _I32, _P, _P, _I64, _P, _P, _I32, _I64, _P],
    "mlk_zlib_compress6_warp": [_P, _P, _P, _I32, _I32, _I32, _P, _P, _I64, _P, _I32, _P, _I64,
                                _P, _P],
    "mlk_zlib_compress6_warp_dyn": [_P, _P, _P, _I32, _I32, _I32, _P, _P, _I64, _P, _I32, _P,
                                    _I64, _P, _P, _P],
    "mlk_gather_segments": [_P, _P, _P, _I32, _P, _P, _P],
    "mlk_zlib_decompress": [_P, _P, _P, _I32, _P, _P, _I64, _P, _P],
    "mlk_stage1": [_P, _P, _I32, _I32, _P, _P, _I32, _P, _P, _P, _P],
    "mlk_kmeans": [_P, _P, _P, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P],
    "mlk_kmeans_prof": [_P, _P],
    "mlk_synth_planes": [_P, _I64, _I64, _I32, _P, _D, _D, _P, _P],
    "mlk_select": [_P, _P, _P, _I32, _I32, _P, _P, _I32, _I32, _P, _D, _P, _P, _P, _P, _P],
    "mlk_recheck": [_P, _P, _P, _I32, _I32, _P, _P, _I32, _P, _I32, _P, _D, _P, _P, _P],
    "mlk_compact": [_P, _P, _P, _I32, _D, _P, _P, _P, _P, _P, _P],
    "mlk_parse_residual_section": [_P, _I64, _I32, _I32, _I32, _I64, _I32, _P, _P, _P, _P, _P,
                                   _P, _P],
    "mlk_is_pinned": [_P],
    "mlk_host_register": [_P, _I64],
    "mlk_search_tree": [_P, _P, _P, _P, _P, _P, _P, _I32, _I32, _I32, _P, _P],
    "mlk_host_unregister": [_P],
    "mlk_host_exception_entries": [_P, _P, _P, _P, _I64, _I32],
    "mlk_probe": [_P, _P, _P, _I32, _P, _P, _I32, _P, _I32, _P, _P, _P, _P, _I32, _P, _D, _P,
                  _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P],
    "mlk_probe_bins": [_P, _P, _I32, _P, _P, _I32, _P, _I32, _P, _P, _P, _I32, _P, _P, _P,
                       _P, _P],
    "mlk_project": [_P, _P, _P, _P, _I32, _I32, _P, _P, _I32, _P, _I32, _P, _P, _P, _P, _P,
                    _P, _P, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _I32, _P, _P],
    "mlk_split_flags": [_P, _I32, ctypes.c_uint32, _P, _P, _P, _P],
    "mlk_list_flags": [_P, _P, _I32, ctypes.c_uint32, _P, _P, _P],
    "mlk_pack_residuals": [_P, _P, _P, _P, _P, _P, _P, _P, _I32, _I32, _I32, _P, _P],
    "mlk_pack_lambdas": [_P, _P, _P, _I32, _I32, _P, _I32, _P, _P],
    "mlk_pack_exceptions": [_P, _P, _I32, _P, _P, _P, _I32, _I32, _P, _P],
    "mlk_compare": [_P, _P, _I32, _P, _P, _P, _P, _P, _P, _P],
    "mlk_report": [_P, _I32, _P, _I64, _P, _P, _P],
    "mlk_pq_nearest": [_P, _I64, _I32, _P, _I32, _P, _P],
    "mlk_pq_lookup": [_P, _I64, _I32, _P, _I32, _P, _P, _P],
    "mlk_quantize_codes": [_P, _I64, _D, _P, _P, _P],
    "mlk_dequantize": [_P, _I64, _D, _I32, _P, _P],
    "mlk_quantize_roundtrip": [_P, _P, _I64, _D, _P, _P],
    "mlk_apply_lambda_rows": [_P, _I64, _I32, _P, _P, _I64, _D, _P, _P],
    "mlk_ae_decode": [_P, _I64, _I32, _P, _I32, _D, _D, _P, _P, _P],
    "mlk_ae_train": [_P, _P, _P, _P, _I32, _I32, _I32, _I32, _D, _D, _D, _D, _D, _D, _P, _I32, _P, _P, _P],
    "mlk_ae_train_config": [_P, _P],
    "mlk_decode": [_P, _I32, _I32, _P, _P, _I32, _P, _I32, _P, _P, _P, _P, _P, _P, _P, _P,
                   _D, _P, _P, _P],
}

_ERRORS = {-1: DimensionError, -2: ConfigError, -3: FormatError, -4: SizeMismatchError,
           -5: ValueError, -6: BackendError}


@functools.lru_cache(maxsize=None)
def host_lib() -> ctypes.CDLL:
    """The library with its signatures set, for its HOST-only entry points
    (search trees, archive parsing): loads without a GPU."""
    if not LIB_PATH.exists():
        raise BackendError(f"{LIB_PATH.name} not built; run __graft_entry__.build()")
    so = ctypes.CDLL(str(LIB_PATH))
    for name, argtypes in _SIGS.items():
        fn = getattr(so, name, None)
        if fn is None:
            continue
        fn.argtypes = argtypes
        fn.restype = ctypes.c_int
    so.mlk_version.restype = ctypes.c_char_p
    return so


@functools.lru_cache(maxsize=None)
def lib() -> ctypes.CDLL:
    if not torch.cuda.is_available():
        raise BackendError("no CUDA device: the B200 path has no CPU fallback")
    so = host_lib()
    torch.cuda.init()
    if so.mlk_device_check() != 0:
        raise BackendError("current CUDA device is not sm_100 (B200)")
    return so


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_handle() -> int:
    """cudaStream_t of the current stream (the raw accessor skips the device
    resolution torch.cuda.current_stream() does on every call)."""
    if _raw_stream is not None:
        return _raw_stream(torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        if t.numel() and not t.is_cuda:
            raise BackendError("device pointer expected")
        return t.data_ptr()
    return t


LAUNCHES = 0  # kernels launched through call() (bench.py's gpu_launches)
# entry points that launch more than one kernel per call (DEFLATE: the LZ77
# parse, then trees + bit stream)
_KERNELS_PER_CALL = {"mlk_zlib_compress6_warp_dyn": 2, "mlk_zlib_compress6_warp": 2}
_FNS = {}


def call(name: str, *args, msg: str = "", stream: int | None = None) -> None:
    """Launch `name` on the current stream (or the raw cudaStream_t `stream`)."""
    global LAUNCHES
    LAUNCHES += _KERNELS_PER_CALL.get(name, 1)
    fn = _FNS.get(name)
    if fn is None:
        fn = _FNS[name] = getattr(lib(), name)
    conv = [(a.data_ptr() if a.is_cuda or not a.numel() else ptr(a))
            if isinstance(a, torch.Tensor) else a for a in args]
    rc = fn(*conv, stream_handle() if stream is None else stream)
    if rc != 0:
        raise _ERRORS.get(rc, BackendError)(f"{name} failed ({rc}) {msg}".strip())


def exported_symbols():
    """Names of every entry point include/mlk_b200.h declares."""
    return list(_SIGS) + ["mlk_version"]
