"""Device residency helpers: every raster value type of the package keeps its
payload in HBM (a torch CUDA tensor used purely as an allocation) and exposes
the reference's numpy attribute as a lazily materialised, read-only host view.
"""

from __future__ import annotations

import ctypes
import os
import threading
import warnings
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from . import _lib


def device() -> torch.device:
    _lib.lib()  # raises NativeUnavailable without a GPU / library
    return torch.device("cuda", torch.cuda.current_device())


def upload(arr: np.ndarray) -> torch.Tensor:
    """Host array -> contiguous device tensor (same dtype) on the current stream."""
    dev = device()
    a = np.ascontiguousarray(arr)
    if not a.size:
        return torch.empty(a.shape, dtype=_torch_dtype(a.dtype), device=dev)
    if a.nbytes >= _STAGE_MIN:
        out = torch.empty(a.shape, dtype=_torch_dtype(a.dtype), device=dev)
        _stager(dev).upload(a, out)
        return out
    with warnings.catch_warnings():
        # read-only arrays (the frozen value types) are only read by the copy
        warnings.simplefilter("ignore", UserWarning)
        t = torch.from_numpy(a)
    return t.to(dev, non_blocking=True)


def host_view(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> read-only numpy array (synchronising copy)."""
    t = t.detach()
    if t.is_cuda and t.numel() * t.element_size() >= _STAGE_MIN:
        a = download(t)
    else:
        a = t.to("cpu").numpy()
    a.flags.writeable = False
    return a


def download(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> new (writable) numpy array of the same shape and dtype,
    ordered after the current stream's work."""
    t = t.detach().contiguous()
    npdt = np.dtype(torch.empty(0, dtype=t.dtype).numpy().dtype)
    out = np.empty(t.shape, dtype=npdt)
    if out.nbytes >= _STAGE_MIN:
        _stager(t.device).download(t, out)
    elif out.size:
        torch.from_numpy(out).copy_(t)
    return out


# ---- staged host transfers -------------------------------------------------
# Multi-GB payloads between HBM and Python-owned (pageable) host memory: a
# plain pageable copy runs at ~4 GB/s D2H (first-touch page faults of the
# fresh destination, serialised in the driver's copy thread) and ~11 GB/s
# H2D.  Instead the copy engine streams fixed-size chunks through a ring of
# pinned buffers while a thread pool moves the previous chunk between the
# pinned ring and the pageable array (ctypes.memmove drops the GIL, and the
# page faults of a fresh destination are taken by many threads at once).
# Measured on the B200 box for 4.9 GB (tools/host_xfer_probe.py, 16 CPUs):
# D2H 1241 -> 150 ms, H2D 432 -> 118-134 ms.
_STAGE_MIN = 64 << 20  # below this the single pageable copy is as fast
_CHUNK = 64 << 20
_NBUF = 4
_stagers: dict[int, "_Stager"] = {}
_stager_lock = threading.Lock()


def _stager(dev: torch.device) -> "_Stager":
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    with _stager_lock:
        s = _stagers.get(idx)
        if s is None:
            s = _Stager(idx)
            _stagers[idx] = s
        return s


class _Stager:
    def __init__(self, index: int):
        self.index = index
        self.lock = threading.Lock()
        with torch.cuda.device(index):
            self.stream = torch.cuda.Stream()
            self.pins = [torch.empty(_CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(_NBUF)]
            self.events = [torch.cuda.Event() for _ in range(_NBUF)]
        self.used = [False] * _NBUF
        self.threads = max(1, min(16, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity")
                                  else (os.cpu_count() or 1)))
        self.pool = ThreadPoolExecutor(self.threads, thread_name_prefix="wg-xfer")

    def _memmove_parallel(self, dst: int, src: int, n: int) -> list:
        part = -(-n // self.threads)
        part = max(part, 1 << 20)
        return [self.pool.submit(ctypes.memmove, dst + o, src + o, min(part, n - o)) for o in range(0, n, part)]

    def download(self, t: torch.Tensor, out: np.ndarray) -> None:
        n = out.nbytes
        src = t.reshape(-1).view(torch.uint8)
        dst = out.ctypes.data
        with self.lock, torch.cuda.device(self.index):
            st = self.stream
            st.wait_stream(torch.cuda.current_stream())
            nch = -(-n // _CHUNK)
            pending: list = [None] * _NBUF

            def drain(i):
                k = i % _NBUF
                self.events[k].synchronize()
                lo = i * _CHUNK
                pending[k] = self._memmove_parallel(dst + lo, self.pins[k].data_ptr(), min(_CHUNK, n - lo))

            for i in range(nch):
                k = i % _NBUF
                if pending[k] is not None:  # the ring slot's previous chunk is drained
                    for f in pending[k]:
                        f.result()
                    pending[k] = None
                lo = i * _CHUNK
                m = min(_CHUNK, n - lo)
                with torch.cuda.stream(st):
                    self.pins[k][:m].copy_(src[lo:lo + m], non_blocking=True)
                    self.events[k].record(st)
                if i >= 1:
                    drain(i - 1)
            drain(nch - 1)
            for p in pending:
                for f in p or ():
                    f.result()

    def upload(self, a: np.ndarray, out: torch.Tensor) -> None:
        n = a.nbytes
        src = a.ctypes.data
        dst = out.view(-1).view(torch.uint8)
        with self.lock, torch.cuda.device(self.index):
            st = self.stream
            st.wait_stream(torch.cuda.current_stream())  # `out` was allocated on the current stream
            for i in range(-(-n // _CHUNK)):
                k = i % _NBUF
                self.events[k].synchronize()  # the copy that last read this slot is done
                lo = i * _CHUNK
                m = min(_CHUNK, n - lo)
                for f in self._memmove_parallel(self.pins[k].data_ptr(), src + lo, m):
                    f.result()
                with torch.cuda.stream(st):
                    dst[lo:lo + m].copy_(self.pins[k][:m], non_blocking=True)
                    self.events[k].record(st)
            torch.cuda.current_stream().wait_stream(st)


_peek_bufs: dict[int, torch.Tensor] = {}


def read_small(t: torch.Tensor) -> list:
    """Values of a small 8-byte-element device tensor (counters, stats) as a
    Python list, synchronising only the current stream.  Read through
    wg_peek (SM stores into pinned host memory), so it never waits behind a
    large device-to-host copy another stream has queued on the copy engine."""
    assert t.is_cuda and t.element_size() == 8 and t.numel() <= 1024
    src = t.contiguous()
    stream = torch.cuda.current_stream()
    key = stream.cuda_stream
    buf = _peek_bufs.get(key)
    if buf is None:
        buf = torch.empty(1024, dtype=torch.int64, pin_memory=True)
        _peek_bufs[key] = buf
    L = _lib.lib()
    _lib.check(L.wg_peek(_lib.ptr(src), _lib.ptr(buf), src.numel(), _lib.stream_ptr(stream)))
    stream.synchronize()
    return buf[: src.numel()].view(src.dtype).tolist()


def empty(shape, dtype: torch.dtype) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=device())


def zeros(shape, dtype: torch.dtype) -> torch.Tensor:
    return torch.zeros(shape, dtype=dtype, device=device())


def _torch_dtype(dt: np.dtype) -> torch.dtype:
    return {
        np.dtype(np.float64): torch.float64,
        np.dtype(np.int64): torch.int64,
        np.dtype(np.uint8): torch.uint8,
        np.dtype(np.bool_): torch.bool,
        np.dtype(np.int8): torch.int8,
    }[np.dtype(dt)]


def as_device_tensor(x, dtype: torch.dtype) -> torch.Tensor:
    """numpy array or torch tensor -> contiguous device tensor of `dtype`."""
    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.to(device(), non_blocking=True)
        if t.dtype != dtype:
            t = t.to(dtype)
        return t.contiguous()
    a = np.asarray(x)
    t = upload(a)
    if t.dtype != dtype:
        t = t.to(dtype)
    return t
