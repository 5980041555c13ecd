"""Host <-> device staging for the public API (compress / decompress).

The end-to-end path moves the whole timestep over PCIe: 1.6 GB of f0 in,
the archive (~1/7 of that) out.  Pageable copies run at a fraction of the
link rate and a fresh `bytes` object costs a page fault per 4 KiB, so:

  * uploads go through a persistent pinned staging buffer, filled in 64 MiB
    chunks by a thread pool (numpy copies release the GIL) with each chunk's
    async H2D issued on a copy stream as soon as it lands -- host copy and
    PCIe transfer overlap;
  * downloads land in a persistent pinned buffer with one async copy; the
    archive `bytes` is allocated uninitialised and filled by the same pool.
"""

from __future__ import annotations

import collections
import ctypes
import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

__all__ = ["upload_planes", "upload_pieces", "upload_bytes", "download_bytes", "download_view",
           "download_array", "download_pinned_array", "download_into", "download_ranges",
           "download_to_file", "mapped_file", "release_maps", "pinned", "pinned_empty",
           "ArchiveWriter"]

CHUNK = 64 << 20
UP_CHUNK = 2 << 20    # upload_pieces copy granularity
UP_DEPTH = 2          # upload_pieces copies queued on the copy engine at once
DOWN_CHUNK = 16 << 20 # ArchiveWriter D2H granularity
PREFAULT = os.environ.get("MLK_PREFAULT", "1") != "0"
_POOL = None
_PINNED = {}
_COPY_STREAMS = {}
_LAST_UPLOAD = {}


def _pool():
    global _POOL
    if _POOL is None:
        _POOL = ThreadPoolExecutor(max_workers=max(2, min(16, os.cpu_count() or 2)),
                                   thread_name_prefix="mlk-hostio")
    return _POOL


def pinned(name: str, nbytes: int) -> torch.Tensor:
    """Grow-only pinned uint8 buffer by name."""
    b = _PINNED.get(name)
    if b is None or b.numel() < nbytes:
        b = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, pin_memory=True)
        _PINNED[name] = b
    return b


def _copy_stream(dev):
    s = _COPY_STREAMS.get(dev.index)
    if s is None:
        s = _COPY_STREAMS[dev.index] = torch.cuda.Stream(device=dev)
    return s


def _is_pinned(arr: np.ndarray) -> bool:
    if not arr.flags.c_contiguous or arr.nbytes == 0:
        return False
    from ._lib import lib
    return bool(lib().mlk_is_pinned(ctypes.c_void_p(arr.ctypes.data)))


def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """A numpy array in page-locked host memory (torch's caching host
    allocator).  Filling the timestep's f0 into such a buffer lets compress()
    DMA it straight to the GPU."""
    nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
    host = torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)
    return host.numpy()[:nbytes].view(dtype).reshape(shape)


def device_planes_buffer(data: np.ndarray, dev, node_range=None, pad_elems: int = 2):
    """The (uninitialised) device buffer upload_planes fills, tail pad zeroed."""
    P, N = data.shape[:2]
    lo, hi = node_range or (0, N)
    n = P * (hi - lo) * int(np.prod(data.shape[2:]))
    buf = torch.empty(n + pad_elems, dtype=torch.float64, device=dev)
    if pad_elems:
        buf[n:].zero_()
    return buf


def upload_planes(data: np.ndarray, dev, node_range=None, pad_elems: int = 2,
                  plane_events: bool = False, into: torch.Tensor | None = None):
    """data[:, lo:hi] of a (P, N, ...) float64 array -> flat device buffer
    (+pad_elems zeros of tail padding), on the current stream's timeline.

    plane_events=True returns (buf, [event per plane]) and leaves the ordering
    to the caller: the current stream must wait on plane p's event before it
    reads plane p (compress_device runs stage 1 plane by plane as they land).
    into: a buffer from device_planes_buffer to fill instead of a new one."""
    P, N = data.shape[:2]
    lo, hi = node_range or (0, N)
    per_node = int(np.prod(data.shape[2:])) * data.itemsize
    slab = (hi - lo) * per_node
    total = P * slab
    buf = into if into is not None else device_planes_buffer(data, dev, node_range, pad_elems)
    events = []
    if total == 0:
        return (buf, events) if plane_events else buf
    cs = _copy_stream(dev)
    cs.wait_stream(torch.cuda.current_stream(dev))  # buf allocation is ordered first
    dst = buf.view(torch.uint8)
    if _is_pinned(data):
        # the caller's array is page-locked: DMA each plane slab directly
        src = torch.from_numpy(data.reshape(P, -1).view(np.uint8))
        with torch.cuda.stream(cs):
            for p in range(P):
                dst[p * slab:(p + 1) * slab].copy_(src[p, lo * per_node:hi * per_node],
                                                   non_blocking=True)
                if plane_events:
                    e = torch.cuda.Event()
                    e.record(cs)
                    events.append(e)
        ev = torch.cuda.Event()
        ev.record(cs)
    else:
        stage = pinned(f"up{dev.index}", total)
        last = _LAST_UPLOAD.get(dev.index)
        if last is not None:
            last.synchronize()  # the previous upload has left the staging buffer
        st_np = stage.numpy()
        # (plane, byte range within the slab) pieces of <= CHUNK bytes
        pieces = []
        for p in range(P):
            for a in range(0, slab, CHUNK):
                pieces.append((p, a, min(slab, a + CHUNK)))
        src2d = data.reshape(P, N * per_node // data.itemsize)

        def fill(piece):
            p, a, b = piece
            row = src2d[p].view(np.uint8)[lo * per_node:hi * per_node]
            st_np[p * slab + a:p * slab + b] = row[a:b]
            return piece

        with torch.cuda.stream(cs):
            for p, a, b in _pool().map(fill, pieces):
                o = p * slab
                dst[o + a:o + b].copy_(stage[o + a:o + b], non_blocking=True)
                if plane_events and b == slab:
                    e = torch.cuda.Event()
                    e.record(cs)
                    events.append(e)
        ev = torch.cuda.Event()
        ev.record(cs)
        _LAST_UPLOAD[dev.index] = ev
    buf.record_stream(cs)
    if plane_events:
        return buf, events
    torch.cuda.current_stream(dev).wait_event(ev)
    return buf

class PieceUpload:
    """Handle of upload_pieces: wait(g) orders the current stream after group
    g's copies (blocking the host only until they have been issued)."""

    def __init__(self, buf, n_groups):
        self.buf = buf
        self.issued = [threading.Event() for _ in range(n_groups)]
        self.events = [None] * n_groups
        self.error = None
        self.thread = None

    def wait(self, g):
        self.issued[g].wait()
        if self.error is not None:
            raise self.error
        torch.cuda.current_stream(self.buf.device).wait_event(self.events[g])

    def join(self):
        if self.thread is not None:
            self.thread.join()
        if self.error is not None:
            raise self.error


class UploadDone(PieceUpload):
    """PieceUpload of a buffer whose copies are already ordered on the
    current stream (upload_planes)."""

    def __init__(self, buf):
        super().__init__(buf, 1)
        self.issued[0].set()

    def wait(self, g):
        pass


def upload_pieces(data: np.ndarray, dev, groups, pad_elems: int = 2) -> PieceUpload:
    """(P, N, ...) float64 host array -> flat device buffer of the same layout
    (+pad_elems zeros), copied group by group: `groups` is a list of lists of
    (plane, node_lo, node_hi) pieces.  A background thread issues the copies
    in order on the copy stream (DMA straight from page-locked caller memory,
    otherwise through the pinned staging buffer filled by the pool), so the
    caller can start on group 0 while later groups are still in flight."""
    P, N = data.shape[:2]
    per_node = int(np.prod(data.shape[2:])) * data.itemsize
    total = P * N * per_node
    buf = torch.empty(total // data.itemsize + pad_elems, dtype=torch.float64, device=dev)
    if pad_elems:
        buf[total // data.itemsize:].zero_()
    h = PieceUpload(buf, len(groups))
    cs = _copy_stream(dev)
    cs.wait_stream(torch.cuda.current_stream(dev))  # buf allocation is ordered first
    buf.record_stream(cs)
    flat = data.reshape(P, N * per_node // data.itemsize)
    pinned_src = _is_pinned(data)
    if not pinned_src:
        stage = pinned(f"up{dev.index}", total)
        last = _LAST_UPLOAD.get(dev.index)
        if last is not None:
            last.synchronize()  # the previous upload has left the staging buffer
        st_np = stage.numpy()
    dst = buf.view(torch.uint8)

    def spans(group):
        out = []
        for p, lo, hi in group:
            a0, a1 = (p * N + lo) * per_node, (p * N + hi) * per_node
            out += [(p, lo * per_node + a - a0, min(a1, a + UP_CHUNK) - a0 + lo * per_node, a)
                    for a in range(a0, a1, UP_CHUNK)]
        return out

    def fill(sp):
        p, b0, b1, a = sp
        st_np[a:a + b1 - b0] = flat[p].view(np.uint8)[b0:b1]
        return sp

    def run():
        try:
            torch.cuda.set_device(dev)
            inflight = collections.deque()
            with torch.cuda.stream(cs):
                for g, group in enumerate(groups):
                    sps = spans(group)
                    it = iter(sps) if pinned_src else _pool().map(fill, sps)
                    for p, b0, b1, a in it:
                        # the copy engine serves copies in issue order: keep only
                        # UP_DEPTH chunks queued so the compute stream's small
                        # D2H reads do not wait behind the whole upload
                        if len(inflight) >= UP_DEPTH:
                            inflight.popleft().synchronize()
                        src = (torch.from_numpy(flat[p].view(np.uint8)[b0:b1]) if pinned_src
                               else stage[a:a + b1 - b0])
                        dst[a:a + b1 - b0].copy_(src, non_blocking=True)
                        e = torch.cuda.Event()
                        e.record(cs)
                        inflight.append(e)
                    ev = torch.cuda.Event()
                    ev.record(cs)
                    h.events[g] = ev
                    h.issued[g].set()
                if not pinned_src:
                    _LAST_UPLOAD[dev.index] = h.events[-1]
        except BaseException as e:  # surfaced by wait()
            h.error = e
            for x in h.issued:
                x.set()

    h.thread = threading.Thread(target=run, daemon=True, name="mlk-upload")
    h.thread.start()
    return h


class ArchiveWriter:
    """Builds the archive `bytes` while the device is still working: each
    shard group's blobs are copied D2H on their own stream as soon as they are
    packed and copied into the (uninitialised, upper-bound sized) bytes object
    by the pool; pages ahead of the write position are pre-faulted in the
    background; finish() writes the preamble + offset index and shrinks the
    object to its length (realloc of an mmap'd block: no copy)."""

    _HINT = {}

    def __init__(self, dev, cap: int, head_len: int):
        self.dev = dev
        self.cap = cap
        self.head_len = head_len
        self.obj = _new_bytes(None, cap)
        self.addr = _bytes_buffer(self.obj)
        self.view = np.ctypeslib.as_array((ctypes.c_uint8 * cap).from_address(self.addr))
        _advise_huge(self.view)
        self.pos = head_len
        self.d2h_bytes = 0
        self.jobs = []
        self.d2h = _d2h_stream(dev)
        self.n_groups = 0
        hint = min(cap, self._HINT.get(dev.index, 0)) if PREFAULT else 0
        self._prefault(head_len, hint)

    def _prefault(self, lo, hi):
        """Touch one byte per page of [lo, hi) in the pool (first-touch faults
        off the critical path; the bytes are overwritten later)."""
        step = 4096
        spans = [(a, min(hi, a + CHUNK)) for a in range(lo, hi, CHUNK)]
        v = self.view

        def touch(sp):
            v[sp[0]:sp[1]:step] = 0

        self.prefault_jobs = [_pool().submit(touch, sp) for sp in spans]
        self.jobs += self.prefault_jobs

    def prefaulted(self):
        """Block until the pre-faulting is done (page faults take the address
        space lock, which the driver's host-side calls contend for)."""
        for j in self.prefault_jobs:
            j.result()

    def add(self, src: torch.Tensor, nbytes: int):
        """Append the first nbytes of a device uint8 tensor (enqueued after the
        current stream's work)."""
        if nbytes == 0:
            return
        if self.pos + nbytes > self.cap:
            raise MemoryError("archive larger than its bound")
        stage = pinned(f"arc{self.dev.index}_{self.n_groups}", nbytes)
        self.n_groups += 1
        self.d2h.wait_stream(torch.cuda.current_stream(self.dev))
        st_np = stage.numpy()
        body = self.view[self.pos:self.pos + nbytes]

        def cp(job):
            ev, a, b = job
            ev.synchronize()
            body[a:b] = st_np[a:b]

        # chunked D2H: each chunk is copied into the bytes object as it lands
        with torch.cuda.stream(self.d2h):
            for a in range(0, nbytes, DOWN_CHUNK):
                b = min(nbytes, a + DOWN_CHUNK)
                stage[a:b].copy_(src[a:b], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.d2h)
                self.jobs.append(_pool().submit(cp, (ev, a, b)))
        src.record_stream(self.d2h)
        self.pos += nbytes
        self.d2h_bytes += nbytes

    def add_with_host_rows(self, src: torch.Tensor, nbytes: int, holes, fill):
        """add() for a buffer whose byte ranges `holes` [(offset, length)] are
        written from host memory by fill(view, offset, length) jobs instead
        of being copied back from the device."""
        if not holes:
            return self.add(src, nbytes)
        base = self.pos
        if base + nbytes > self.cap:
            raise MemoryError("archive larger than its bound")
        holes = sorted((int(o), int(n)) for o, n in holes if n > 0)
        stage = pinned(f"arc{self.dev.index}_{self.n_groups}", nbytes)
        self.n_groups += 1
        self.d2h.wait_stream(torch.cuda.current_stream(self.dev))
        st_np = stage.numpy()
        body = self.view[base:base + nbytes]

        def cp(job):
            ev, a, b = job
            ev.synchronize()
            body[a:b] = st_np[a:b]

        spans, pos = [], 0
        for o, n in holes:
            if o > pos:
                spans.append((pos, o))
            pos = o + n
        if pos < nbytes:
            spans.append((pos, nbytes))
        with torch.cuda.stream(self.d2h):
            for lo, hi in spans:
                for a in range(lo, hi, DOWN_CHUNK):
                    b = min(hi, a + DOWN_CHUNK)
                    stage[a:b].copy_(src[a:b], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(self.d2h)
                    self.jobs.append(_pool().submit(cp, (ev, a, b)))
                self.d2h_bytes += hi - lo
        src.record_stream(self.d2h)
        for o, n in holes:
            self.jobs += fill(body, o, n)
        self.pos += nbytes

    def drain(self):
        """Wait for every pool job writing into the archive object (error
        paths: the object must outlive them)."""
        for j in self.jobs:
            try:
                j.result()
            except Exception:
                pass

    def finish(self, head: bytes) -> bytes:
        if len(head) != self.head_len:
            raise ValueError("archive head length changed")
        err = None
        for j in self.jobs:  # every job finishes before an error propagates
            try:
                j.result()
            except Exception as e:  # noqa: BLE001
                err = err or e
        if err is not None:
            raise err
        self.view[:len(head)] = np.frombuffer(head, dtype=np.uint8)
        n = self.pos
        self._HINT[self.dev.index] = n
        self.view = None
        ref = ctypes.py_object(self.obj)
        self.obj = None
        if n != self.cap and _resize_bytes(ctypes.byref(ref), n) != 0:
            raise MemoryError("could not shrink the archive")
        return ref.value


_D2H_STREAMS = {}


def _d2h_stream(dev):
    s = _D2H_STREAMS.get(dev.index)
    if s is None:
        s = _D2H_STREAMS[dev.index] = torch.cuda.Stream(device=dev)
    return s


_MADV_HUGEPAGE = 14
_libc = None


def _advise_huge(arr: np.ndarray):
    """Ask for transparent huge pages on a fresh large array (fewer faults)."""
    global _libc
    try:
        if _libc is None:
            _libc = ctypes.CDLL(None, use_errno=True)
        a = arr.ctypes.data
        lo = (a + (2 << 20) - 1) & ~((2 << 20) - 1)
        hi = (a + arr.nbytes) & ~((2 << 20) - 1)
        if hi > lo:
            _libc.madvise(ctypes.c_void_p(lo), ctypes.c_size_t(hi - lo), _MADV_HUGEPAGE)
    except Exception:
        pass


# The archive is returned as `bytes` (the reference API's type) without an
# extra host copy: the documented C-API pattern for building a bytes object in
# place -- PyBytes_FromStringAndSize(NULL, n) gives an uninitialised object
# whose buffer (PyBytes_AsString) may be written until the object is shared,
# and _PyBytes_Resize may shrink such a brand-new object.  Nothing else sees
# the object before it is complete.
_new_bytes = ctypes.pythonapi.PyBytes_FromStringAndSize
_new_bytes.restype = ctypes.py_object
_new_bytes.argtypes = [ctypes.c_void_p, ctypes.c_ssize_t]
_resize_bytes = ctypes.pythonapi._PyBytes_Resize
_resize_bytes.restype = ctypes.c_int
_resize_bytes.argtypes = [ctypes.POINTER(ctypes.py_object), ctypes.c_ssize_t]
_bytes_as_string = ctypes.pythonapi.PyBytes_AsString
_bytes_as_string.restype = ctypes.c_void_p
_bytes_as_string.argtypes = [ctypes.py_object]


def _bytes_buffer(obj: bytes) -> int:
    """Address of a brand-new bytes object's buffer (PyBytes_AsString)."""
    addr = _bytes_as_string(obj)
    if not addr:
        raise MemoryError("PyBytes_AsString failed")
    return addr


def download_bytes(src: torch.Tensor, nbytes: int, prefix: bytes = b"") -> bytes:
    """prefix + the first nbytes of a device uint8 tensor, as one bytes object."""
    dev = src.device
    stage = pinned(f"down{dev.index}", nbytes)
    if nbytes:
        stage[:nbytes].copy_(src[:nbytes], non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
    total = len(prefix) + nbytes
    out = _new_bytes(None, total)  # uninitialised; filled before anyone sees it
    view = np.ctypeslib.as_array((ctypes.c_uint8 * total).from_address(_bytes_buffer(out)))
    _advise_huge(view)
    view[:len(prefix)] = np.frombuffer(prefix, dtype=np.uint8)
    body = view[len(prefix):]
    st_np = stage.numpy()
    spans = [(a, min(nbytes, a + CHUNK)) for a in range(0, nbytes, CHUNK)]

    def cp(span):
        a, b = span
        body[a:b] = st_np[a:b]

    list(_pool().map(cp, spans))
    return out


def download_view(src: torch.Tensor, nbytes: int) -> np.ndarray:
    """The first nbytes of a device uint8 tensor in the pinned download buffer
    (a view: valid until the next download on this device)."""
    stage = pinned(f"down{src.device.index}", nbytes)
    if nbytes:
        stage[:nbytes].copy_(src[:nbytes], non_blocking=True)
        torch.cuda.current_stream(src.device).synchronize()
    return stage.numpy()[:nbytes]


def download_ranges(src: torch.Tensor, nbytes: int, ranges) -> np.ndarray:
    """download_view of a device uint8 tensor restricted to `ranges` [(a, b),
    ...]: only those bytes are copied (to the same offsets of the pinned
    view; the rest of it is stale)."""
    stage = pinned(f"down{src.device.index}", nbytes)
    for a, b in ranges:
        if b > a:
            stage[a:b].copy_(src[a:b], non_blocking=True)
    torch.cuda.current_stream(src.device).synchronize()
    return stage.numpy()[:nbytes]


def upload_bytes(raw, dev, ranges=None) -> torch.Tensor:
    """A bytes-like object -> device uint8 tensor of the same length (pinned
    staging, chunked).  ranges: [(start, end), ...] -- only those bytes are
    copied (each to its own offset); the rest of the tensor is left
    uninitialised (a rank decoding part of an archive skips the other
    ranks' exception images)."""
    src = np.frombuffer(raw, dtype=np.uint8)
    n = src.size
    buf = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    if n == 0:
        return buf
    stage = pinned(f"upb{dev.index}", n)
    last = _LAST_UPLOAD.get(("b", dev.index))
    if last is not None:
        last.synchronize()
    st_np = stage.numpy()
    spans = [(a, min(e, a + CHUNK)) for s0, e in (ranges or [(0, n)])
             for a in range(s0, e, CHUNK)]

    def fill(span):
        a, b = span
        st_np[a:b] = src[a:b]
        return span

    cs = _copy_stream(dev)
    cs.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(cs):
        for a, b in _pool().map(fill, spans):
            buf[a:b].copy_(stage[a:b], non_blocking=True)
    ev = torch.cuda.Event()
    ev.record(cs)
    _LAST_UPLOAD[("b", dev.index)] = ev
    torch.cuda.current_stream(dev).wait_event(ev)
    buf.record_stream(cs)
    return buf


def download_array(src: torch.Tensor, shape, dtype=np.float64) -> np.ndarray:
    """Device tensor -> a fresh numpy array: chunked async D2H into pinned
    memory overlapped with thread-parallel copies into the result."""
    dev = src.device
    out = np.empty(shape, dtype=dtype)
    nbytes = out.nbytes
    if nbytes == 0:
        return out
    _advise_huge(out)
    flat = out.reshape(-1).view(np.uint8)
    s8 = src.reshape(-1).view(torch.uint8)[:nbytes]
    stage = pinned(f"dla{dev.index}", nbytes)
    st_np = stage.numpy()
    cs = _copy_stream(dev)
    cs.wait_stream(torch.cuda.current_stream(dev))
    spans = [(a, min(nbytes, a + CHUNK)) for a in range(0, nbytes, CHUNK)]
    events = []
    with torch.cuda.stream(cs):
        for a, b in spans:
            stage[a:b].copy_(s8[a:b], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
            events.append(ev)

    def cp(k):
        a, b = spans[k]
        events[k].synchronize()
        flat[a:b] = st_np[a:b]

    list(_pool().map(cp, range(len(spans))))
    return out


_MAPS = {}   # (st_dev, st_ino, size) -> mmap
_REGS = {}   # (map key, page-aligned start, end) -> registered address


def mapped_file(fd: int, total: int) -> np.ndarray:
    """A shared, writable uint8 view of the first `total` bytes of an open
    file, cached per (device, inode, size): a file rewritten step after step
    keeps its page-table entries, so filling it costs a memcpy, not a page
    fault per 4 KiB (the mapping pins the inode, so the key cannot be reused
    by another file while it is cached)."""
    import mmap
    st = os.fstat(fd)
    key = (st.st_dev, st.st_ino, total)
    m = _MAPS.get(key)
    if m is None:
        for k in [k for k in _MAPS if k[:2] == key[:2]]:
            _drop_map(k)
        flags = mmap.MAP_SHARED | getattr(mmap, "MAP_POPULATE", 0)
        m = _MAPS[key] = mmap.mmap(fd, total, flags, mmap.PROT_WRITE | mmap.PROT_READ)
    return np.frombuffer(m, dtype=np.uint8)


def _drop_map(key):
    from ._lib import lib
    for rk in [rk for rk in _REGS if rk[0] == key]:
        lib().mlk_host_unregister(ctypes.c_void_p(_REGS.pop(rk)))
    del _MAPS[key]  # unmapped once no view of it is left


def release_maps() -> None:
    """Unregister and drop every cached mapped_file mapping (call after
    deleting the files)."""
    for k in list(_MAPS):
        _drop_map(k)


def download_to_file(src: torch.Tensor, nbytes: int, fd: int, total: int, offset: int) -> None:
    """The first nbytes of a device tensor into bytes [offset, offset + nbytes)
    of an open file of size `total`, by DMA straight into its shared mapping:
    the page range is page-locked once (cudaHostRegister, cached with the
    mapping) and every later call is one device-to-host copy."""
    if nbytes == 0:
        return
    from ._lib import lib
    view = mapped_file(fd, total)
    st = os.fstat(fd)
    key = (st.st_dev, st.st_ino, total)
    base = view.ctypes.data
    page = os.sysconf("SC_PAGE_SIZE")
    lo = (base + offset) // page * page
    hi = -(-(base + offset + nbytes) // page) * page
    hi = min(hi, -(-(base + total) // page) * page)
    rk = (key, lo, hi)
    if rk not in _REGS:
        if lib().mlk_host_register(ctypes.c_void_p(lo), hi - lo) != 0:
            del view
            download_into(src, nbytes, mapped_file(fd, total)[offset:offset + nbytes])
            return
        _REGS[rk] = lo
    dst = torch.from_numpy(view[offset:offset + nbytes])
    dst.copy_(src.reshape(-1).view(torch.uint8)[:nbytes], non_blocking=True)
    torch.cuda.current_stream(src.device).synchronize()
    del dst, view


def download_into(src: torch.Tensor, nbytes: int, dst: np.ndarray) -> None:
    """The first nbytes of a device tensor into a writable host uint8 array
    (e.g. a mapped_file view): chunked async D2H into pinned memory, each
    chunk copied out by a pool thread as soon as it lands."""
    if nbytes == 0:
        return
    dev = src.device
    s8 = src.reshape(-1).view(torch.uint8)[:nbytes]
    stage = pinned(f"dli{dev.index}", nbytes)
    st_np = stage.numpy()
    cs = _copy_stream(dev)
    cs.wait_stream(torch.cuda.current_stream(dev))
    spans = [(a, min(nbytes, a + DOWN_CHUNK)) for a in range(0, nbytes, DOWN_CHUNK)]
    events = []
    with torch.cuda.stream(cs):
        for a, b in spans:
            stage[a:b].copy_(s8[a:b], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
            events.append(ev)

    def put(k):
        a, b = spans[k]
        events[k].synchronize()
        dst[a:b] = st_np[a:b]

    list(_pool().map(put, range(len(spans))))


def download_pinned_array(src: torch.Tensor, shape, dtype=np.float64) -> np.ndarray:
    """Device tensor -> numpy array backed by page-locked memory from torch's
    caching host allocator: one DMA at full PCIe rate, no staging copy and
    no page faults (freed results are recycled for the next call)."""
    nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
    host = torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)
    if nbytes:
        host[:nbytes].copy_(src.reshape(-1).view(torch.uint8)[:nbytes], non_blocking=True)
        torch.cuda.current_stream(src.device).synchronize()
    return host.numpy()[:nbytes].view(dtype).reshape(shape)
