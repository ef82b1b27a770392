"""ctypes binding of the wgb200 C ABI (include/wgb200.h).

This is the only way the package reaches its compute kernels.  There is no
CPU fallback: every op that needs the library calls :func:`lib`, which raises
:class:`NativeUnavailable` when the shared library is missing or no CUDA
device is visible.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from pathlib import Path

import torch

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "_lib" / "libwgb200.so"
CSRC = _PKG / "csrc"

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None

c_i64 = ctypes.c_int64
c_u64 = ctypes.c_uint64
c_dbl = ctypes.c_double
c_int = ctypes.c_int
c_ptr = ctypes.c_void_p
c_size = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/wgb200.h one to one
SIGNATURES: dict[str, tuple] = {
    "wg_last_error": (ctypes.c_char_p, []),
    "wg_version": (ctypes.c_char_p, []),
    "wg_launch_count": (c_u64, []),
    "wg_device_sms": (c_int, [ctypes.POINTER(c_int)]),
    "wg_peek": (c_int, [c_ptr, c_ptr, c_i64, c_ptr]),
    "wg_grid_scan": (c_int, [c_ptr, c_i64, c_dbl, c_ptr, c_ptr]),
    "wg_copy2d_f64": (c_int, [c_ptr, c_i64, c_ptr, c_i64, c_i64, c_i64, c_ptr]),
    "wg_normals": (c_int, [c_ptr, c_i64, c_i64, c_dbl, c_dbl, c_ptr, c_ptr, c_ptr]),
    "wg_steepness": (c_int, [c_ptr, c_i64, c_ptr, c_ptr]),
    "wg_hillshade": (c_int, [c_ptr, c_i64, c_dbl, c_dbl, c_dbl, c_ptr, c_ptr]),
    "wg_hillshade_rgba": (c_int, [c_ptr, c_i64, c_dbl, c_dbl, c_dbl, c_ptr, c_ptr]),
    "wg_release_mask": (c_int, [c_ptr, c_i64, c_i64, c_dbl, c_dbl, c_i64, c_ptr, c_ptr, c_ptr]),
    "wg_lattice_release_mask": (c_int, [c_ptr, c_i64, c_i64, c_dbl, c_dbl, c_dbl, c_dbl, c_i64, c_i64, c_i64, c_ptr,
                                        c_ptr, c_ptr]),
    "wg_compact_scratch_bytes": (c_size, [c_i64]),
    "wg_mask_compact": (c_int, [c_ptr, c_i64, c_ptr, c_ptr, c_ptr, c_ptr]),
    "wg_avalanche_scratch_bytes": (c_size, [c_i64, c_i64, c_i64]),
    "wg_run_avalanche": (
        c_int,
        [c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl,
         c_i64, c_ptr, c_i64, c_u64, c_ptr, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_int, c_int, c_int, c_int, c_ptr,
         c_ptr],
    ),
    "wg_absmax": (c_int, [c_ptr, c_i64, c_ptr, c_ptr]),
    "wg_sorted_offsets": (c_int, [c_ptr, c_i64, c_ptr, c_i64, c_ptr, c_ptr]),
    "wg_tiles_pack": (c_int, [c_ptr, c_ptr, c_i64, c_i64, c_int, c_ptr, c_ptr, c_i64, c_i64, c_ptr, c_ptr, c_ptr]),
    "wg_tiles_accumulate": (c_int, [c_ptr, c_ptr, c_i64, c_i64, c_int, c_ptr, c_i64, c_ptr, c_ptr]),
    "wg_tiles_zero": (c_int, [c_ptr, c_ptr, c_i64, c_i64, c_int, c_ptr, c_i64, c_ptr]),
    "wg_build_quad": (c_int, [c_ptr, c_i64, c_i64, c_ptr, c_ptr]),
    "wg_build_pair": (c_int, [c_ptr, c_i64, c_i64, c_ptr, c_ptr]),
    "wg_trace_particle": (
        c_int,
        [c_ptr, c_i64, c_i64, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_i64,
         c_dbl, c_dbl, c_dbl, c_u64, c_ptr, c_i64, c_ptr, c_ptr],
    ),
    "wg_particle_records": (
        c_int,
        [c_ptr, c_i64, c_i64, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_i64,
         c_ptr, c_i64, c_u64, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr],
    ),
    "wg_trig_eval": (c_int, [c_ptr, c_i64, c_ptr, c_ptr, c_ptr]),
    "wg_div_eval": (c_int, [c_ptr, c_ptr, c_i64, c_ptr, c_ptr]),
    "wg_sqrt_eval": (c_int, [c_ptr, c_i64, c_ptr, c_ptr, c_ptr]),
    "wg_acos_eval": (c_int, [c_ptr, c_i64, c_ptr, c_ptr, c_ptr]),
    "wg_runout_stats": (c_int, [c_ptr, c_ptr, c_i64, c_ptr, c_ptr]),
    "wg_snow": (c_int, [c_ptr, c_ptr, c_i64, c_dbl, c_dbl, c_dbl, c_dbl, c_int, c_dbl, c_ptr, c_ptr]),
    "wg_colorize": (c_int, [c_ptr, c_i64, c_dbl, c_ptr, c_ptr, c_int, c_int, c_ptr, c_ptr]),
    "wg_max_f64": (c_int, [c_ptr, c_i64, c_ptr, c_ptr, c_ptr]),
    "wg_mipmap_scratch_bytes": (c_size, [c_i64, c_i64]),
    "wg_mipmap": (c_int, [c_ptr, c_i64, c_i64, c_ptr, c_ptr, c_ptr]),
    "wg_digest": (c_int, [c_ptr, c_i64, c_ptr, c_ptr]),
    "wg_digest2d": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr]),
    "wg_synth_combine": (c_int, [c_ptr, c_ptr, c_ptr, c_int, c_i64, c_i64, c_ptr, c_ptr]),
    "wg_sub_scalar": (c_int, [c_ptr, c_i64, c_dbl, c_ptr]),
    "wg_png_capacity": (c_i64, [c_i64, c_i64]),
    "wg_png_scratch_bytes": (c_size, [c_i64, c_i64, c_i64]),
    "wg_png_tiles": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_ptr]),
    "wg_png_encode": (c_int, [c_ptr, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_ptr]),
    "wg_ascii_read_scratch_bytes": (c_size, [c_i64, c_i64]),
    "wg_ascii_read": (c_int, [c_ptr, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_ptr]),
    "wg_ascii_format_scratch_bytes": (c_size, [c_i64]),
    "wg_ascii_format_capacity": (c_i64, [c_i64]),
    "wg_ascii_format": (c_int, [c_ptr, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_ptr]),
}

WG_OK, WG_ECUDA, WG_EARG, WG_ELIMIT = 0, 1, 2, 3


class NativeUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is missing; there is no fallback."""


class NativeError(RuntimeError):
    """A wgb200 entry point returned a CUDA failure."""


def build(force: bool = False) -> Path:
    """Compile libwgb200.so in-tree for sm_100a (nvcc via csrc/Makefile)."""
    if force or not LIB_PATH.exists():
        cmd = ["make", "-C", str(CSRC), "-j", str(min(8, os.cpu_count() or 1))]
        subprocess.run(cmd, check=True, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    return LIB_PATH


def load(path: Path | None = None) -> ctypes.CDLL:
    """Load the shared library (no device required) and bind every symbol."""
    global _lib
    with _lock:
        if _lib is None:
            p = Path(path or LIB_PATH)
            if not p.exists():
                raise NativeUnavailable(
                    f"{p} is missing: build it with paper_2506_23364_b200._lib.build() "
                    "(nvcc, sm_100a); there is no CPU fallback"
                )
            h = ctypes.CDLL(str(p))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            _lib = h
        return _lib


def lib() -> ctypes.CDLL:
    """The library, for a compute call: requires a visible CUDA device."""
    if not torch.cuda.is_available():
        raise NativeUnavailable(
            "no CUDA device visible: paper_2506_23364_b200 computes only on the GPU (no CPU fallback)"
        )
    return load()


def check(rc: int, exc_for_arg: type[Exception] = ValueError) -> None:
    if rc == WG_OK:
        return
    msg = (load().wg_last_error() or b"").decode(errors="replace")
    if rc == WG_EARG:
        raise exc_for_arg(msg)
    raise NativeError(f"wgb200 error {rc}: {msg}")


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    return int(t.data_ptr())


def launch_count() -> int:
    return int(load().wg_launch_count())
