"""Device residency helpers: every raster value type of the package keeps its
payload in HBM (a torch CUDA tensor used purely as an allocation) and exposes
the reference's numpy attribute as a lazily materialised, read-only host view.
"""

from __future__ import annotations

import warnings

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
    with warnings.catch_warnings():
        # read-only arrays (the frozen value types) are only read by the copy
        warnings.simplefilter("ignore", UserWarning)
        t = torch.from_numpy(a)
    return t.to(dev, non_blocking=True)


def host_view(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> read-only numpy array (synchronising copy)."""
    a = t.detach().to("cpu").numpy()
    a.flags.writeable = False
    return a


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
