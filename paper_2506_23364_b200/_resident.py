"""Base class for the immutable raster value types (NormalField, SlopeField,
ReleaseMask, RunoutRaster, OverlayTexture): each named payload lives in HBM
as a torch CUDA tensor and is exposed under the reference's attribute name as
a lazily materialised read-only numpy array.
"""

from __future__ import annotations

from dataclasses import FrozenInstanceError

import numpy as np
import torch

from . import _device


class Resident:
    _payload: tuple[str, ...] = ()
    _dtypes: dict[str, tuple[np.dtype, torch.dtype]] = {}

    def __init__(self, **arrays):
        object.__setattr__(self, "_h", {})
        object.__setattr__(self, "_d", {})
        for name in self._payload:
            x = arrays[name]
            npdt, tdt = self._dtypes[name]
            if isinstance(x, torch.Tensor):
                t = x.detach()
                if t.dtype != tdt:
                    t = t.to(tdt)
                if t.is_cuda:
                    self._d[name] = t.contiguous()
                else:
                    a = t.contiguous().numpy()
                    a.flags.writeable = False
                    self._h[name] = a
            else:
                a = np.ascontiguousarray(np.asarray(x, dtype=npdt))
                a.flags.writeable = False
                self._h[name] = a
        object.__setattr__(self, "_frozen", True)

    def __setattr__(self, name, value):
        raise FrozenInstanceError(f"cannot assign to field '{name}'")

    def __getattr__(self, name):
        # reference attribute names resolve to the host view
        payload = type(self)._payload
        if name in payload:
            h = self._h.get(name)
            if h is None:
                h = _device.host_view(self._d[name])
                self._h[name] = h
            return h
        raise AttributeError(f"{type(self).__name__!s} has no attribute {name!r}")

    def dev(self, name: str) -> torch.Tensor:
        """Device tensor of a payload (uploaded on first use if host-built)."""
        t = self._d.get(name)
        if t is None:
            t = _device.upload(self._h[name])
            self._d[name] = t
        return t

    def shape_of(self, name: str) -> tuple[int, ...]:
        t = self._d.get(name)
        return tuple(t.shape) if t is not None else tuple(self._h[name].shape)

    def on_device(self, name: str) -> bool:
        return name in self._d
