"""ctypes binding of the C ABI in ``include/fvsrn_b200.h`` (libfvsrn_b200.so).

This is the only place the Python host API touches native code.  The library is
built in-tree by ``make`` / ``__graft_entry__.build()``; if it is missing the
import fails loudly -- there is no CPU fallback on the product path.
"""

from __future__ import annotations

import ctypes as C
import math
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(os.environ.get("FVSRN_LIB") or
                Path(__file__).resolve().parent / "libfvsrn_b200.so")   # FVSRN_LIB: A/B builds

FVSRN_OK, FVSRN_EINVAL, FVSRN_ECAPACITY, FVSRN_ECUDA, FVSRN_ENOMEM = range(5)
ACT_CODES = {"relu": 0, "sigmoid": 1, "softplus": 2, "snake": 3, "snake_alt": 4}
HEAD_CODES = {"density": 0, "color": 1}
DIR_CODES = {"pos": 0, "dirP": 1, "dirF": 2}
TIME_CODES = {"none": 0, "direct": 1, "fourier": 2, "both": 3}
FOURIER_CODES = {"off": 0, "nerf": 1, "random": 2}
GRID_F32, GRID_U8 = 0, 1

_f = C.POINTER(C.c_float)
_d = C.POINTER(C.c_double)
_pf = C.POINTER(_f)


class ModelDesc(C.Structure):
    _fields_ = [
        ("layers", C.c_int32), ("hidden", C.c_int32), ("d_in", C.c_int32), ("d_out", C.c_int32),
        ("activation", C.c_int32), ("head", C.c_int32), ("direction_mode", C.c_int32),
        ("fourier_mode", C.c_int32), ("fourier_m", C.c_int32), ("fourier_d_in", C.c_int32),
        ("b_matrix", _f),
        ("time_mode", C.c_int32), ("time_fourier_count", C.c_int32),
        ("time_b", _f),
        ("has_time_range", C.c_int32), ("time_range", C.c_double * 2),
        ("grid_resolution", C.c_int32), ("grid_channels", C.c_int32),
        ("n_grids", C.c_int32),
        ("keyframe_times", _d),
        ("temporal", C.c_int32),
        ("grid_precision", C.c_int32),
        ("grids", _pf),
        ("grid_codes", C.POINTER(C.POINTER(C.c_uint8))),
        ("grid_mins", _pf),
        ("grid_maxs", _pf),
        ("weights", _pf),
        ("biases", _pf),
    ]


class TFDesc(C.Structure):
    _fields_ = [("n", C.c_int32), ("xs", _f), ("rgbs", _f), ("sigmas", _f)]


class CameraDesc(C.Structure):
    _fields_ = [
        ("eye", C.c_double * 3), ("target", C.c_double * 3), ("up", C.c_double * 3),
        ("fov_y", C.c_double), ("width", C.c_int32), ("height", C.c_int32),
        ("has_basis", C.c_int32), ("b_forward", C.c_double * 3), ("b_right", C.c_double * 3),
        ("b_up", C.c_double * 3), ("half_w", C.c_double), ("half_h", C.c_double),
    ]


class SettingsDesc(C.Structure):
    _fields_ = [
        ("stepsize", C.c_double), ("max_steps", C.c_int32), ("background", C.c_double * 3),
        ("early_term_alpha", C.c_double), ("eps_blend", C.c_double),
    ]


class ShardDesc(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("compact", C.c_int32)]


EXPORTS = {
    # name: (restype, argtypes)
    "fvsrn_last_error": (C.c_char_p, []),
    "fvsrn_set_dvr_kernel": (C.c_int32, [C.c_int32]),
    "fvsrn_set_grid_sampler": (C.c_int32, [C.c_int32]),
    "fvsrn_mlp_forward_backward": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                               C.c_void_p]),
    "fvsrn_layer_grads": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                      C.c_void_p, C.c_int32, C.c_void_p]),
    "fvsrn_grid_sample_backward": (C.c_int32, [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64,
                                               C.c_void_p, C.c_void_p]),
    "fvsrn_model_grads": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p]),
    "fvsrn_train_world_grads": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_int64,
                                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_void_p]),
    "fvsrn_train_screen_forward": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                               C.POINTER(SettingsDesc)] + [C.c_void_p] * 7),
    "fvsrn_train_screen_backward": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                                C.c_double] + [C.c_void_p] * 8 + [C.c_int64] +
                                               [C.c_void_p] * 5),
    "fvsrn_f32_eval": (C.c_int32, [C.c_void_p] * 6 + [C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]),
    "fvsrn_adam_step": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                    C.c_double, C.c_double, C.c_double, C.c_double, C.c_int32,
                                    C.c_void_p, C.c_void_p]),
    "fvsrn_kernel_timer": (C.c_int32, [C.c_int32]),
    "fvsrn_ipc_export": (C.c_int32, [C.c_void_p, C.c_char_p, C.POINTER(C.c_uint64)]),
    "fvsrn_ipc_open": (C.c_int32, [C.c_char_p, C.c_uint64, C.c_int32, C.POINTER(C.c_void_p)]),
    "fvsrn_ipc_close": (C.c_int32, [C.c_void_p]),
    "fvsrn_kernel_timer_read": (C.c_int32, [C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                            C.POINTER(C.c_int64)]),
    "fvsrn_kernel_timer_info": (C.c_int32, [C.c_char_p, C.c_int32]),
    "fvsrn_version": (C.c_char_p, []),
    "fvsrn_device_count": (C.c_int32, []),
    "fvsrn_model_create": (C.c_int32, [C.POINTER(ModelDesc), C.c_int32, C.POINTER(C.c_void_p)]),
    "fvsrn_model_destroy": (C.c_int32, [C.c_void_p]),
    "fvsrn_model_sampler": (C.c_int32, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_float)]),
    "fvsrn_model_info": (C.c_int32, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                     C.POINTER(C.c_int32)]),
    "fvsrn_render": (C.c_int32, [C.c_void_p, C.POINTER(TFDesc), C.POINTER(CameraDesc),
                                 C.POINTER(SettingsDesc), C.c_double, _f,
                                 C.POINTER(C.c_uint64)]),
    "fvsrn_render_rgba8": (C.c_int32, [C.c_void_p, C.POINTER(TFDesc), C.POINTER(CameraDesc),
                                       C.POINTER(SettingsDesc), C.c_double, C.c_void_p,
                                       C.POINTER(C.c_uint64)]),
    "fvsrn_render_device": (C.c_int32, [C.c_void_p, C.POINTER(TFDesc), C.POINTER(CameraDesc),
                                        C.POINTER(SettingsDesc), C.c_double, C.POINTER(ShardDesc),
                                        C.c_void_p, C.c_void_p, C.c_void_p]),
    "fvsrn_tiles_to_frame_device": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                                C.c_void_p, C.c_void_p]),
    "fvsrn_render_rays": (C.c_int32, [C.c_void_p, C.POINTER(TFDesc), _d, _d, C.c_int64,
                                      C.POINTER(SettingsDesc), C.c_double, _f,
                                      C.POINTER(C.c_uint64)]),
    "fvsrn_eval_density": (C.c_int32, [C.c_void_p, _d, C.c_int64, C.c_double, _f]),
    "fvsrn_eval_color": (C.c_int32, [C.c_void_p, _d, _d, C.c_int64, C.c_double, _f]),
    "fvsrn_decode_density": (C.c_int32, [C.c_void_p, C.c_int32, C.c_double, _f]),
    "fvsrn_decode_density_device": (C.c_int32, [C.c_void_p, C.c_int32, C.c_double, C.c_int64,
                                                C.c_int64, C.c_void_p, C.c_void_p]),
    "fvsrn_fused_eval": (C.c_int32, [C.c_void_p, _f, C.c_int64, _f]),
    "fvsrn_volume_create": (C.c_int32, [_f, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                        C.POINTER(C.c_void_p)]),
    "fvsrn_volume_destroy": (C.c_int32, [C.c_void_p]),
    "fvsrn_volume_render": (C.c_int32, [C.c_void_p, C.POINTER(TFDesc), C.POINTER(CameraDesc),
                                        C.POINTER(SettingsDesc), _f, C.POINTER(C.c_uint64)]),
    "fvsrn_volume_render_device": (C.c_int32, [C.c_void_p, C.POINTER(TFDesc), C.POINTER(CameraDesc),
                                               C.POINTER(SettingsDesc), C.POINTER(ShardDesc),
                                               C.c_void_p, C.c_void_p]),
    "fvsrn_volume_render_rays": (C.c_int32, [C.c_void_p, C.POINTER(TFDesc), _d, _d, C.c_int64,
                                             C.POINTER(SettingsDesc), _f, C.POINTER(C.c_uint64)]),
    "fvsrn_render_multi": (C.c_int32, [C.POINTER(C.c_void_p), C.c_int32, C.POINTER(TFDesc),
                                       C.POINTER(CameraDesc), C.POINTER(SettingsDesc), C.c_double,
                                       _f, C.POINTER(C.c_uint64)]),
    "fvsrn_decode_density_multi": (C.c_int32, [C.POINTER(C.c_void_p), C.c_int32, C.c_int32,
                                               C.c_double, _f]),
    "fvsrn_host_alloc": (C.c_int32, [C.c_uint64, C.POINTER(C.c_void_p)]),
    "fvsrn_host_free": (C.c_int32, [C.c_void_p]),
}

class TrainDesc(C.Structure):
    """fvsrn_train_desc"""
    _fields_ = [("layers", C.c_int32), ("hidden", C.c_int32), ("d_in", C.c_int32),
                ("d_out", C.c_int32), ("activation", C.c_int32), ("head", C.c_int32),
                ("fourier_m", C.c_int32), ("d_b_matrix", C.c_void_p),
                ("grid_resolution", C.c_int32), ("grid_channels", C.c_int32),
                ("n_keyframes", C.c_int32), ("keyframe_times", C.POINTER(C.c_double)),
                ("time_mode", C.c_int32), ("time_fourier_count", C.c_int32),
                ("time_b", C.POINTER(C.c_float)), ("time_t0", C.c_double), ("time_t1", C.c_double),
                ("raw_width", C.c_int32), ("fourier_in", C.c_int32)]


_LIB = None


def lib():
    """Load (once) and return the native library; raises if it was not built."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA library first "
                "(`make` or `python -c 'import __graft_entry__ as g; g.build()'`). "
                "The fV-SRN B200 path has no CPU fallback.")
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in EXPORTS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = handle
    return _LIB


class CapacityError(ValueError):
    """Network does not fit (fused.py:30-31 counterpart)."""


def check(rc: int) -> None:
    if rc == FVSRN_OK:
        return
    msg = lib().fvsrn_last_error().decode(errors="replace")
    if rc == FVSRN_EINVAL:
        raise ValueError(msg)
    if rc == FVSRN_ECAPACITY:
        raise CapacityError(msg)
    raise RuntimeError(f"fvsrn_b200 native error {rc}: {msg}")


def fptr(a: np.ndarray):
    return a.ctypes.data_as(_f)


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_d)


def t_arg(t) -> float:
    return math.nan if t is None else float(t)


class _PinnedOwner:
    """Frees a fvsrn_host_alloc block when the last numpy view of it dies."""

    def __init__(self, ptr: int):
        self.ptr = ptr

    def __del__(self):
        try:
            lib().fvsrn_host_free(C.c_void_p(self.ptr))
        except Exception:  # pragma: no cover - interpreter shutdown
            pass


def pinned_empty(shape, dtype=np.float32) -> np.ndarray:
    """numpy array in page-locked host memory (full-bandwidth device->host reads)."""
    dtype = np.dtype(dtype)
    nbytes = max(1, int(np.prod(shape)) * dtype.itemsize)
    p = C.c_void_p()
    check(lib().fvsrn_host_alloc(nbytes, C.byref(p)))
    buf = (C.c_char * nbytes).from_address(p.value)
    buf._owner = _PinnedOwner(p.value)     # lives exactly as long as the buffer object
    return np.frombuffer(buf, dtype=np.uint8, count=nbytes).view(dtype)[:int(np.prod(shape))].reshape(shape)


class _PooledOwner:
    """Returns a pooled page-locked block to ``_POOL`` when the last numpy view of it dies."""

    def __init__(self, ptr: int, nbytes: int):
        self.ptr, self.nbytes = ptr, nbytes

    def __del__(self):
        try:
            _POOL.give(self.ptr, self.nbytes)
        except Exception:  # pragma: no cover - interpreter shutdown
            pass


class _PinnedPool:
    """Page-locked (portable, mapped) host blocks recycled by size for the arrays the stock
    API returns (``render_image(src, cam, settings)`` without ``out=``): the render kernels
    store each finished pixel straight into the returned frame over PCIe instead of a
    pageable device->host copy after the march.  A block goes back to the pool when the
    caller drops the last view of it.  At most ``CAP`` bytes are handed out at once
    (beyond that arrays are ordinary pageable memory) and ``IDLE`` bytes kept idle."""

    CAP = 4 << 30
    IDLE = 1 << 30

    def __init__(self):
        import threading

        self.lock = threading.Lock()
        self.free: dict[int, list[int]] = {}
        self.out_bytes = 0
        self.idle_bytes = 0

    def take(self, nbytes: int):
        with self.lock:
            lst = self.free.get(nbytes)
            if lst:
                self.idle_bytes -= nbytes
                self.out_bytes += nbytes
                return lst.pop()
            if self.out_bytes + nbytes > self.CAP:
                return None
            self.out_bytes += nbytes
        p = C.c_void_p()
        if lib().fvsrn_host_alloc(nbytes, C.byref(p)) != FVSRN_OK:
            with self.lock:
                self.out_bytes -= nbytes
            return None
        return p.value

    def give(self, ptr: int, nbytes: int):
        with self.lock:
            self.out_bytes -= nbytes
            if self.idle_bytes + nbytes <= self.IDLE:
                self.free.setdefault(nbytes, []).append(ptr)
                self.idle_bytes += nbytes
                return
        lib().fvsrn_host_free(C.c_void_p(ptr))


_POOL = _PinnedPool()


def pooled_empty(shape, dtype=np.float32) -> np.ndarray:
    """Like ``pinned_empty`` but from the recycling pool (pageable ``np.empty`` when the
    pool's cap is reached)."""
    dtype = np.dtype(dtype)
    count = int(np.prod(shape))
    nbytes = max(1, count * dtype.itemsize)
    ptr = _POOL.take(nbytes)
    if ptr is None:
        return np.empty(shape, dtype=dtype)
    buf = (C.c_char * nbytes).from_address(ptr)
    buf._owner = _PooledOwner(ptr, nbytes)
    return np.frombuffer(buf, dtype=np.uint8, count=nbytes).view(dtype)[:count].reshape(shape)


def current_device() -> int:
    env = os.environ.get("FVSRN_DEVICE")
    if env is not None:
        return int(env)
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # pragma: no cover
        pass
    return 0
