"""The reference's operator API (mlk/kernels.py:20-32) on the B200.

Same names, signatures, return types and error behaviour as
``mlk._ckernels`` / ``mlk._pykernels``; each call runs the batched device
kernel of include/mlk_b200.h on one stream (inputs copied in, results
copied out).  These per-call entry points exist for API parity and tests;
the pipeline uses the fused stage kernels.
"""

from __future__ import annotations

import numpy as np
import torch

from ._lib import call

BACKEND = "sm_100a"
NEWTON_CONVERGED, NEWTON_MAX_ITER, NEWTON_DEGENERATE = 0, 1, 2

__all__ = ["BACKEND", "NEWTON_CONVERGED", "NEWTON_MAX_ITER", "NEWTON_DEGENERATE",
           "newton_solve", "zigzag_map", "zigzag_unmap", "varint_encode", "varint_decode",
           "pack_indices", "unpack_indices"]


def _dev():
    return torch.device("cuda", torch.cuda.current_device())


def _to(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).to(_dev(), dtype=dtype)


def newton_solve(f_plus, a, b, step, max_iter, tol):
    """Damped dual Newton (_ckernels.pyx:62-137) -> (lam, status, iterations)."""
    fp = np.ascontiguousarray(f_plus, dtype=np.float64).reshape(-1)
    d = fp.size
    av = np.ascontiguousarray(a, dtype=np.float64).reshape(4, d)
    bv = np.ascontiguousarray(b, dtype=np.float64).reshape(4)
    lam = torch.empty(4, dtype=torch.float64, device=_dev())
    st = torch.empty(1, dtype=torch.int32, device=_dev())
    it = torch.empty(1, dtype=torch.int32, device=_dev())
    call("mlk_newton_solve_batch", _to(fp, torch.float64), _to(av, torch.float64),
         _to(bv, torch.float64), 1, d, float(step), int(max_iter), float(tol), lam, st, it)
    return lam.cpu().numpy(), int(st.item()), int(it.item())


def zigzag_map(values):
    q = np.ascontiguousarray(values, dtype=np.int64).reshape(-1)
    if q.size == 0:
        return np.zeros(0, dtype=np.uint64)
    z = torch.empty(q.size, dtype=torch.int64, device=_dev())
    call("mlk_zigzag_map", _to(q, torch.int64), z, q.size)
    return z.cpu().numpy().view(np.uint64)


def zigzag_unmap(codes):
    z = np.ascontiguousarray(codes, dtype=np.uint64).reshape(-1)
    if z.size == 0:
        return np.zeros(0, dtype=np.int64)
    q = torch.empty(z.size, dtype=torch.int64, device=_dev())
    call("mlk_zigzag_unmap", _to(z.view(np.int64), torch.int64), q, z.size)
    return q.cpu().numpy()


def varint_encode(values) -> bytes:
    v = np.ascontiguousarray(values, dtype=np.uint64).reshape(-1)
    if v.size == 0:
        return b""
    dev = _dev()
    out = torch.empty(10 * v.size, dtype=torch.uint8, device=dev)
    ln = torch.empty(1, dtype=torch.int64, device=dev)
    call("mlk_varint_encode_batch", _to(v.view(np.int64), torch.int64),
         torch.tensor([0, v.size], dtype=torch.int64, device=dev), 1, out,
         torch.zeros(1, dtype=torch.int64, device=dev), ln)
    return out[:int(ln.item())].cpu().numpy().tobytes()


def varint_decode(buf, count):
    if count == 0:
        return np.zeros(0, dtype=np.uint64), 0
    raw = np.frombuffer(bytes(buf), dtype=np.uint8)
    dev = _dev()
    vals = torch.zeros(count, dtype=torch.int64, device=dev)
    used = torch.empty(1, dtype=torch.int64, device=dev)
    call("mlk_varint_decode_batch", _to(raw if raw.size else np.zeros(1, np.uint8), torch.uint8),
         torch.zeros(1, dtype=torch.int64, device=dev),
         torch.tensor([raw.size], dtype=torch.int64, device=dev), 1,
         torch.tensor([count], dtype=torch.int64, device=dev), vals,
         torch.zeros(1, dtype=torch.int64, device=dev), used)
    n = int(used.item())
    if n == -1:
        raise ValueError("varint stream truncated")
    if n == -2:
        raise ValueError("varint value exceeds 64 bits")
    return vals.cpu().numpy().view(np.uint64), n


def pack_indices(indices, bits):
    if not 1 <= bits <= 16:
        raise ValueError(f"bits must be in [1, 16], got {bits}")
    idx = np.ascontiguousarray(indices, dtype=np.uint16).reshape(-1)
    if idx.size == 0:
        return b""
    dev = _dev()
    nbytes = (idx.size * bits + 7) // 8
    out = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    call("mlk_pack_indices", _to(idx.view(np.int16), torch.int16), idx.size, bits, out, bad)
    if int(bad.item()):
        raise ValueError("index does not fit the configured bit width")
    return out.cpu().numpy().tobytes()


def unpack_indices(buf, count, bits):
    if not 1 <= bits <= 16:
        raise ValueError(f"bits must be in [1, 16], got {bits}")
    if count == 0:
        return np.zeros(0, dtype=np.uint16)
    raw = np.frombuffer(bytes(buf), dtype=np.uint8)
    if raw.size * 8 < count * bits:
        raise ValueError("packed index stream too short")
    out = torch.empty(count, dtype=torch.int16, device=_dev())
    call("mlk_unpack_indices", _to(raw, torch.uint8), count, bits, out)
    return out.cpu().numpy().view(np.uint16)
