"""ctypes bindings for oracle/ckernels.c -- TEST INFRASTRUCTURE ONLY."""

from __future__ import annotations

import ctypes
import functools

import numpy as np

from oracle import build as _build

_i64 = ctypes.c_int64
_dbl = ctypes.c_double
_int = ctypes.c_int
_vp = ctypes.c_void_p


@functools.lru_cache(maxsize=None)
def lib():
    so = ctypes.CDLL(str(_build.build()))
    so.oracle_project_batch.argtypes = [_vp, _i64, _i64, _vp, _vp, _vp, _dbl, _vp, _dbl,
                                        _dbl, _int, _dbl, _int, _dbl, _int, _vp, _vp, _vp, _vp]
    so.oracle_project_batch.restype = None
    so.oracle_newton.argtypes = [_vp, _vp, _vp, _i64, _dbl, _int, _dbl, _vp, _vp]
    so.oracle_newton.restype = _int
    so.oracle_varint_encode.argtypes = [_vp, _i64, _vp]
    so.oracle_varint_encode.restype = _i64
    so.oracle_varint_decode.argtypes = [_vp, _i64, _i64, _vp]
    so.oracle_varint_decode.restype = _i64
    so.oracle_pack_indices.argtypes = [_vp, _i64, _int, _vp]
    so.oracle_pack_indices.restype = _int
    so.oracle_unpack_indices.argtypes = [_vp, _i64, _int, _vp]
    so.oracle_unpack_indices.restype = None
    so.oracle_encode.argtypes = [_vp, _i64, _i64, _vp, _int, _dbl, _dbl, _vp, _vp]
    so.oracle_encode.restype = None
    so.oracle_decode.argtypes = [_vp, _i64, _int, _vp, _i64, _vp, _dbl, _dbl, _vp]
    so.oracle_decode.restype = None
    return so


def _p(a):
    return a.ctypes.data_as(_vp)


def newton_solve(f_plus, a, b, step, max_iter, tol):
    fp = np.ascontiguousarray(f_plus, dtype=np.float64)
    av = np.ascontiguousarray(a, dtype=np.float64)
    bv = np.ascontiguousarray(b, dtype=np.float64)
    lam = np.zeros(4)
    it = np.zeros(1, dtype=np.int32)
    st = lib().oracle_newton(_p(fp), _p(av), _p(bv), fp.size, float(step), int(max_iter),
                             float(tol), _p(lam), _p(it))
    return lam, int(st), int(it[0])


def project_batch(flat, vol, vpar, vperp, mass, qois, floor, step, max_iter, tol,
                  retry=False, retry_step=0.01, retry_max_iter=400):
    flat = np.ascontiguousarray(flat, dtype=np.float64)
    n, d = flat.shape
    q = np.ascontiguousarray(qois, dtype=np.float64)
    lams = np.zeros((n, 4))
    status = np.zeros(n, dtype=np.int32)
    iters = np.zeros(n, dtype=np.int32)
    work = np.empty(5 * d)
    cells = [np.ascontiguousarray(x, dtype=np.float64) for x in (vol, vpar, vperp)]
    lib().oracle_project_batch(_p(flat), n, d, _p(cells[0]), _p(cells[1]), _p(cells[2]),
                               float(mass), _p(q), float(floor), float(step), int(max_iter),
                               float(tol), int(bool(retry)), float(retry_step),
                               int(retry_max_iter), _p(lams), _p(status), _p(iters), _p(work))
    return lams, status, iters


def varint_encode(values) -> bytes:
    v = np.ascontiguousarray(values, dtype=np.uint64)
    out = np.empty(max(1, 10 * v.size), dtype=np.uint8)
    k = lib().oracle_varint_encode(_p(v), v.size, _p(out))
    return out[:k].tobytes()


def varint_decode(buf: bytes, count: int):
    arr = np.frombuffer(buf, dtype=np.uint8).copy() if len(buf) else np.zeros(1, np.uint8)
    out = np.zeros(count, dtype=np.uint64)
    k = lib().oracle_varint_decode(_p(arr), len(buf), count, _p(out))
    if k == -1:
        raise ValueError("varint stream truncated")
    if k == -2:
        raise ValueError("varint value exceeds 64 bits")
    return out, int(k)


def pack_indices(idx, bits: int) -> bytes:
    v = np.ascontiguousarray(idx, dtype=np.uint16)
    out = np.zeros((v.size * bits + 7) // 8 or 1, dtype=np.uint8)
    if lib().oracle_pack_indices(_p(v), v.size, int(bits), _p(out)) != 0:
        raise ValueError("index does not fit the configured bit width")
    return out[:(v.size * bits + 7) // 8].tobytes()


def unpack_indices(buf: bytes, count: int, bits: int):
    arr = np.frombuffer(buf, dtype=np.uint8).copy()
    if arr.size * 8 < count * bits:
        raise ValueError("packed index stream too short")
    out = np.empty(count, dtype=np.uint16)
    if count:
        lib().oracle_unpack_indices(_p(arr), count, int(bits), _p(out))
    return out


def encode(flat, w32, mean, std):
    flat = np.ascontiguousarray(flat, dtype=np.float64)
    n, d = flat.shape
    w = np.ascontiguousarray(w32, dtype=np.float32)
    out = np.empty((n, w.shape[0]))
    work = np.empty(d)
    lib().oracle_encode(_p(flat), n, d, _p(w), w.shape[0], float(mean), float(std), _p(out), _p(work))
    return out


def decode(lat, w32, mean, std, tree_cols):
    lat = np.ascontiguousarray(lat, dtype=np.float64)
    w = np.ascontiguousarray(w32, dtype=np.float32)
    d = w.shape[1]
    tc = np.ascontiguousarray(tree_cols, dtype=np.uint8)
    out = np.empty((lat.shape[0], d))
    lib().oracle_decode(_p(lat), lat.shape[0], w.shape[0], _p(w), d, _p(tc), float(mean),
                        float(std), _p(out))
    return out
