"""The device DEFLATE restatement (csrc/zlib6.h) reproduces zlib.compress(x, 6)
byte-for-byte.  Host build of the same header (no GPU needed)."""

from __future__ import annotations

import ctypes
import functools
import subprocess
import zlib
from pathlib import Path

import numpy as np
import pytest

HERE = Path(__file__).resolve().parent
SRC = HERE / "native" / "z6_host.cpp"
HDR = HERE.parent / "paper_2212_10733_b200" / "csrc" / "zlib6.h"
OUT = HERE / "native" / "_build" / "libz6host.so"


@functools.lru_cache(maxsize=None)
def z6():
    if not OUT.exists() or OUT.stat().st_mtime < max(SRC.stat().st_mtime, HDR.stat().st_mtime):
        OUT.parent.mkdir(exist_ok=True)
        subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", str(OUT), str(SRC)],
                       check=True)
    lib = ctypes.CDLL(str(OUT))
    lib.z6_compress.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p,
                                ctypes.c_longlong]
    lib.z6_compress.restype = ctypes.c_longlong
    return lib


def deflate6(data: bytes) -> bytes:
    buf = ctypes.create_string_buffer(len(data) + len(data) // 8 + 64)
    src = ctypes.create_string_buffer(data, max(1, len(data)))
    n = z6().z6_compress(src, len(data), buf, len(buf))
    assert n >= 0, n
    return buf.raw[:n]


def _varints(q):
    z = ((q.astype(np.int64) << 1) ^ (q.astype(np.int64) >> 63)).astype(np.uint64)
    out = bytearray()
    for x in z.tolist():
        while x >= 0x80:
            out.append((x & 0x7F) | 0x80)
            x >>= 7
        out.append(x)
    return bytes(out)


CORPORA = {
    "empty": [b""],
    "tiny": [b"a", b"ab", b"abc", b"abcd", b"aaaa", b"\0" * 5],
    "zeros": [b"\0" * n for n in (10, 100, 258, 259, 1000, 1521, 15210)],
    "text": [(b"the quick brown fox jumps over the lazy dog " * 40)[:n] for n in (50, 300, 1700)],
}


@pytest.mark.parametrize("name", list(CORPORA))
def test_fixed_corpora(name):
    for data in CORPORA[name]:
        assert deflate6(data) == zlib.compress(data, 6), (name, len(data))


def test_random_small_alphabets():
    rng = np.random.default_rng(7)
    for t in range(300):
        n = int(rng.integers(1, 6000))
        k = int(rng.choice([2, 3, 5, 8, 17, 64, 256]))
        data = rng.integers(0, k, n, dtype=np.uint8).tobytes()
        assert deflate6(data) == zlib.compress(data, 6), (t, n, k)


def test_residual_like_varints():
    """Streams shaped like the pipeline's: zigzag varints of smooth + noisy q."""
    rng = np.random.default_rng(11)
    for t in range(200):
        scale = 10 ** rng.uniform(-1, 5)
        base = np.cumsum(rng.standard_normal(1521)) * rng.uniform(0, 2)
        q = np.rint(base + rng.standard_normal(1521) * scale).astype(np.int64)
        if t % 7 == 0:
            q[rng.uniform(size=1521) < 0.8] = 0
        data = _varints(q)
        assert deflate6(data) == zlib.compress(data, 6), t


def test_lossless_like_streams():
    rng = np.random.default_rng(3)
    for t in range(40):
        r = rng.standard_normal(1521) * 10 ** rng.uniform(-3, 12)
        bits = np.ascontiguousarray(r).view(np.uint64)
        out = bytearray()
        for x in bits.tolist():
            while x >= 0x80:
                out.append((x & 0x7F) | 0x80)
                x >>= 7
            out.append(x)
        data = bytes(out)
        assert deflate6(data) == zlib.compress(data, 6), t


def test_golden_payloads():
    """Payload bytes the reference itself produced (tests/golden/units.npz)."""
    from tests import golden_util as G
    meta, a = G.load("units")
    for t in range(len(meta["payload_ebs"])):
        p = a[f"pl{t}_p"].tobytes()
        raw = zlib.decompress(p[13:])
        assert deflate6(raw) == p[13:], t


def inflate(data: bytes, cap: int) -> bytes:
    lib = z6()
    lib.z6_inflate.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p,
                               ctypes.c_longlong]
    lib.z6_inflate.restype = ctypes.c_longlong
    out = ctypes.create_string_buffer(max(1, cap))
    src = ctypes.create_string_buffer(data, max(1, len(data)))
    n = lib.z6_inflate(src, len(data), out, cap)
    if n < 0:
        raise ValueError(f"inflate error {n}")
    return out.raw[:n]


def test_inflate_roundtrip_all_levels():
    rng = np.random.default_rng(5)
    for t in range(200):
        n = int(rng.integers(0, 5000))
        k = int(rng.choice([2, 7, 40, 256]))
        data = rng.integers(0, k, n, dtype=np.uint8).tobytes()
        for level in (0, 1, 6, 9):
            comp = zlib.compress(data, level)
            assert inflate(comp, n + 16) == data, (t, level)


def test_inflate_rejects_corruption():
    comp = bytearray(zlib.compress(b"hello world " * 50, 6))
    with pytest.raises(ValueError):
        inflate(bytes(comp[:-1]), 1000)
    comp[-1] ^= 1
    with pytest.raises(ValueError):
        inflate(bytes(comp), 1000)
    with pytest.raises(ValueError):
        inflate(b"\x78\x9c" + b"\xff" * 10, 1000)
