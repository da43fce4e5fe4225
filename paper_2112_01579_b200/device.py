"""Device-resident fV-SRN model: one ``fvsrn_model_t`` per (model, GPU).

Upload happens once (weights packed into fp16 mma B-fragments, grids to fp16
(R,R,R,F_pad), u8 checkpoints dequantised with the reference formula); every
render / eval call after that only ships per-frame constants (camera basis,
TF, time) -- the ownership contract of SURVEY 8(b).
"""

from __future__ import annotations

import ctypes as C
import math
import threading

import numpy as np

from . import _lib as L


def camera_basis(cam):
    """render.py:78-86 evaluated with numpy (bit-identical per-frame basis)."""
    eye = np.asarray(cam.eye, dtype=np.float64)
    fwd = np.asarray(cam.target, dtype=np.float64) - eye
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(cam.up, dtype=np.float64))
    right = right / np.linalg.norm(right)
    up = np.cross(right, fwd)
    half_h = np.tan(cam.fov_y / 2.0)
    half_w = half_h * cam.width / cam.height
    return fwd, right, up, float(half_w), float(half_h)


_CAM_CACHE: dict = {}
_TF_CACHE: dict = {}
_CACHE_MAX = 64
_desc_lock = threading.Lock()


def _cache_put(cache: dict, key, value):
    """Insert with FIFO eviction; the descriptor caches are shared by every thread that
    renders (service workers), so eviction and insertion happen under one lock."""
    with _desc_lock:
        while len(cache) >= _CACHE_MAX:
            cache.pop(next(iter(cache)), None)
        cache[key] = value
    return value


def _words(a) -> np.ndarray:
    a = np.ascontiguousarray(a)
    return a.reshape(-1).view(np.uint8)


def grid_fingerprint(grids, sampled: bool = False) -> tuple:
    """Cheap content fingerprint of latent grids: the XOR of all 64-bit words plus the
    byte length (0.1 ms for a 2 MiB f32 grid), or with ``sampled`` a CRC of every
    4099th value (microseconds; used per frame by ModelSource)."""
    import zlib

    out = []
    for g in grids:
        v = np.ascontiguousarray(g.values if hasattr(g, "values") else g, dtype=np.float32).reshape(-1)
        if sampled:
            out.append((v.size, zlib.crc32(v[::4099].tobytes())))
        else:
            head = v[: v.size - v.size % 2]
            out.append((v.size, int(np.bitwise_xor.reduce(head.view(np.uint64))) if head.size else 0,
                        float(v[-1]) if v.size % 2 else 0.0))
    return tuple(out)


def param_fingerprint(model, sampled_grids: bool = False) -> tuple:
    """What the device copy of ``model`` was built from: array identities, an exact CRC of
    every weight and bias (<= 90 KB) and a grid fingerprint.  device_model() compares it
    on every call so in-place edits (adam_step, trainers, direct writes) are picked up;
    the reference re-reads the arrays on every call."""
    import zlib

    p = model.params
    crc = 0
    for a in (*p.weights, *p.biases):
        crc = zlib.crc32(np.ascontiguousarray(a, dtype=np.float32), crc)
    ids = tuple(id(a) for a in model.trainable_arrays())
    return ids, crc, grid_fingerprint(model.grids, sampled_grids)


def camera_desc(cam) -> L.CameraDesc:
    """Descriptor with the numpy-evaluated basis; cached per camera value (the basis
    costs ~50 us of numpy per frame, more than the C entry's whole host path)."""
    key = (tuple(map(float, cam.eye)), tuple(map(float, cam.target)), tuple(map(float, cam.up)),
           float(cam.fov_y), int(cam.width), int(cam.height))
    d = _CAM_CACHE.get(key)
    return d if d is not None else _cache_put(_CAM_CACHE, key, _camera_desc(cam))


def _camera_desc(cam) -> L.CameraDesc:
    d = L.CameraDesc()
    d.eye[:] = [float(v) for v in cam.eye]
    d.target[:] = [float(v) for v in cam.target]
    d.up[:] = [float(v) for v in cam.up]
    d.fov_y = float(cam.fov_y)
    d.width, d.height = int(cam.width), int(cam.height)
    fwd, right, up, hw, hh = camera_basis(cam)
    d.has_basis = 1
    d.b_forward[:] = fwd.tolist()
    d.b_right[:] = right.tolist()
    d.b_up[:] = up.tolist()
    d.half_w, d.half_h = hw, hh
    return d


class _TF:
    """Keeps the TF arrays alive while the descriptor is in use."""

    def __init__(self, tf):
        self.xs = np.ascontiguousarray(tf.xs, dtype=np.float32)
        self.rgbs = np.ascontiguousarray(tf.rgbs, dtype=np.float32)
        self.sigmas = np.ascontiguousarray(tf.sigmas, dtype=np.float32)
        self.desc = L.TFDesc(len(self.xs), L.fptr(self.xs), L.fptr(self.rgbs), L.fptr(self.sigmas))


def tf_desc(tf):
    """TF descriptor.  Reused per TF object when its arrays are already float32 and
    contiguous: the descriptor then points at the caller's arrays, so in-place edits
    are still seen (the C entry reads the TF on every call)."""
    if tf is None:
        return None
    hit = _TF_CACHE.get(id(tf))
    if hit is not None and hit[0] is tf and hit[1].xs is tf.xs and hit[1].rgbs is tf.rgbs \
            and hit[1].sigmas is tf.sigmas:
        return hit[1]
    d = _TF(tf)
    if d.xs is tf.xs and d.rgbs is tf.rgbs and d.sigmas is tf.sigmas:
        _cache_put(_TF_CACHE, id(tf), (tf, d))
    return d


def settings_desc(s) -> L.SettingsDesc:
    d = L.SettingsDesc()
    d.stepsize = float(s.stepsize)
    d.max_steps = int(s.max_steps)
    d.background[:] = [float(v) for v in s.background]
    d.early_term_alpha = float(s.early_term_alpha)
    d.eps_blend = float(s.eps_blend)
    return d


class DeviceModel:
    """Owns one native model handle; immutable after creation, thread-safe to use."""

    def __init__(self, model, device: int | None = None):
        lib = L.lib()
        cfg = model.config
        self.device = L.current_device() if device is None else int(device)
        self.head = cfg.head
        self.temporal = cfg.is_temporal
        self.d_in = cfg.input_width
        self.direction_mode = cfg.direction_mode
        keep = []   # arrays that must outlive the create call

        def f32(a):
            a = np.ascontiguousarray(a, dtype=np.float32)
            keep.append(a)
            return a

        d = L.ModelDesc()
        d.layers, d.hidden = cfg.layers, cfg.hidden
        d.d_in, d.d_out = cfg.input_width, cfg.output_width
        d.activation = L.ACT_CODES[model.params.activation]
        d.head = L.HEAD_CODES[cfg.head]
        d.direction_mode = L.DIR_CODES[cfg.direction_mode]
        enc = model.spatial_encoder
        d.fourier_mode = L.FOURIER_CODES[enc.mode if enc.m > 0 else "off"]
        d.fourier_m = enc.m
        d.fourier_d_in = enc.d_in
        d.b_matrix = L.fptr(f32(enc.b_matrix)) if enc.m > 0 else None
        d.time_mode = L.TIME_CODES[cfg.time_mode]
        d.time_fourier_count = cfg.time_fourier_count
        if model.time_encoder is not None:
            d.time_b = L.fptr(f32(model.time_encoder.b_matrix[:, 0]))
        if cfg.time_range is not None:
            d.has_time_range = 1
            d.time_range[:] = [float(cfg.time_range[0]), float(cfg.time_range[1])]
        grids = model.grids
        d.grid_resolution = cfg.grid_resolution if grids else 0
        d.grid_channels = cfg.grid_channels
        d.n_grids = len(grids)
        d.temporal = 1 if self.temporal else 0
        if self.temporal:
            kt = np.ascontiguousarray(model.keyframes.times, dtype=np.float64)
            keep.append(kt)
            d.keyframe_times = L.dptr(kt)
        if grids:
            quant = getattr(model, "quantized", None)
            # the u8 codes are uploaded only while the grids still hold exactly the values
            # they were loaded as (training or an edit since then makes them stale)
            if quant and getattr(model, "quantized_fp", None) != grid_fingerprint(grids):
                quant = model.quantized = None
            if quant:
                d.grid_precision = L.GRID_U8
                codes = [np.ascontiguousarray(q.codes, dtype=np.uint8) for q in quant]
                keep.extend(codes)
                d.grid_codes = (C.POINTER(C.c_uint8) * len(codes))(
                    *[c.ctypes.data_as(C.POINTER(C.c_uint8)) for c in codes])
                d.grid_mins = (L._f * len(quant))(*[L.fptr(f32(q.mins)) for q in quant])
                d.grid_maxs = (L._f * len(quant))(*[L.fptr(f32(q.maxs)) for q in quant])
            else:
                d.grid_precision = L.GRID_F32
                d.grids = (L._f * len(grids))(*[L.fptr(f32(g.values)) for g in grids])
        d.weights = (L._f * cfg.layers)(*[L.fptr(f32(w)) for w in model.params.weights])
        d.biases = (L._f * cfg.layers)(*[L.fptr(f32(b)) for b in model.params.biases])
        h = C.c_void_p()
        L.check(lib.fvsrn_model_create(C.byref(d), self.device, C.byref(h)))
        self._h = h
        self._lib = lib
        del keep

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        h, self._h = getattr(self, "_h", None), None
        if h:
            self._lib.fvsrn_model_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover - interpreter shutdown
            pass

    def info(self):
        k0, hp, sm = C.c_int32(), C.c_int32(), C.c_int32()
        L.check(self._lib.fvsrn_model_info(self._h, C.byref(k0), C.byref(hp), C.byref(sm)))
        ok, err = C.c_int32(), C.c_float()
        L.check(self._lib.fvsrn_model_sampler(self._h, C.byref(ok), C.byref(err)))
        return {"k0_pad": k0.value, "hidden_pad": hp.value, "smem_bytes": sm.value,
                "texture_sampler_ok": bool(ok.value), "texture_probe_err": err.value}

    # ---------------------------------------------------------------- calls
    def eval_density(self, p, t=None) -> np.ndarray:
        p = np.ascontiguousarray(np.atleast_2d(np.asarray(p, dtype=np.float64)))
        if p.shape[1] != 3:
            raise ValueError(f"positions must have 3 components, got {p.shape}")
        out = np.empty(len(p), dtype=np.float32)
        L.check(self._lib.fvsrn_eval_density(self._h, L.dptr(p), len(p), L.t_arg(t), L.fptr(out)))
        return out

    def eval_color(self, p, d=None, t=None) -> np.ndarray:
        p = np.ascontiguousarray(np.atleast_2d(np.asarray(p, dtype=np.float64)))
        dd = None
        if self.direction_mode != "pos":
            if d is None:
                raise ValueError(f"direction mode {self.direction_mode!r} requires view directions")
            dd = np.ascontiguousarray(np.atleast_2d(np.asarray(d, dtype=np.float64)))
            if dd.shape != p.shape:
                raise ValueError("directions must match positions in shape")
        out = np.empty((len(p), 4), dtype=np.float32)
        L.check(self._lib.fvsrn_eval_color(self._h, L.dptr(p), L.dptr(dd) if dd is not None else None,
                                           len(p), L.t_arg(t), L.fptr(out)))
        return out

    def decode(self, res: int, t=None, out=None) -> np.ndarray:
        n = int(res) ** 3
        if out is None:
            out = L.pooled_empty(n)
        elif out.size != n or out.dtype != np.float32 or not out.flags.c_contiguous:
            raise ValueError(f"out must be a C-contiguous float32 array of {n} elements")
        L.check(self._lib.fvsrn_decode_density(self._h, int(res), L.t_arg(t), L.fptr(out)))
        return out

    def fused_eval(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float32)
        if x.ndim != 2 or x.shape[1] != self.d_in:
            raise ValueError(f"expected assembled inputs (N, {self.d_in}), got {x.shape}")
        oc = 1 if self.head == "density" else 4
        out = np.empty((len(x), oc), dtype=np.float32)
        L.check(self._lib.fvsrn_fused_eval(self._h, L.fptr(x), len(x), L.fptr(out)))
        return out[:, 0] if oc == 1 else out

    def render(self, tf, cam, settings, t=None, out=None):
        """(H,W,4) f32 frame + evaluated-sample count (host buffer, synchronous).

        ``out``: optional C-contiguous float32 (H,W,4) host array to render into
        (e.g. ``pinned_empty`` for full-bandwidth reads)."""
        shape = (cam.height, cam.width, 4)
        if out is None:
            out = L.pooled_empty(shape)
        elif out.shape != shape or out.dtype != np.float32 or not out.flags.c_contiguous:
            raise ValueError(f"out must be a C-contiguous float32 array of shape {shape}")
        cnt = C.c_uint64(0)
        tfd = tf_desc(tf)
        L.check(self._lib.fvsrn_render(self._h, C.byref(tfd.desc) if tfd else None,
                                       C.byref(camera_desc(cam)), C.byref(settings_desc(settings)),
                                       L.t_arg(t), L.fptr(out), C.byref(cnt)))
        return out, int(cnt.value)

    def render_rgba8(self, tf, cam, settings, t=None, out=None):
        """(H,W,4) uint8 frame (png_bytes' quantisation, done on the device) + count."""
        shape = (cam.height, cam.width, 4)
        if out is None:
            out = np.empty(shape, dtype=np.uint8)
        elif out.shape != shape or out.dtype != np.uint8 or not out.flags.c_contiguous:
            raise ValueError(f"out must be a C-contiguous uint8 array of shape {shape}")
        cnt = C.c_uint64(0)
        tfd = tf_desc(tf)
        L.check(self._lib.fvsrn_render_rgba8(self._h, C.byref(tfd.desc) if tfd else None,
                                             C.byref(camera_desc(cam)), C.byref(settings_desc(settings)),
                                             L.t_arg(t), C.c_void_p(out.ctypes.data), C.byref(cnt)))
        return out, int(cnt.value)

    def render_rays(self, tf, origins, dirs, settings, t=None):
        o = np.ascontiguousarray(np.asarray(origins, dtype=np.float64).reshape(-1, 3))
        d = np.ascontiguousarray(np.asarray(dirs, dtype=np.float64).reshape(-1, 3))
        if o.shape != d.shape:
            raise ValueError("origins and dirs must have the same shape")
        out = np.empty((len(o), 4), dtype=np.float32)
        cnt = C.c_uint64(0)
        tfd = tf_desc(tf)
        L.check(self._lib.fvsrn_render_rays(self._h, C.byref(tfd.desc) if tfd else None, L.dptr(o),
                                            L.dptr(d), len(o), C.byref(settings_desc(settings)),
                                            L.t_arg(t), L.fptr(out), C.byref(cnt)))
        return out, int(cnt.value)

    def render_device(self, tf, cam, settings, t, out_ptr: int, count_ptr: int | None,
                      stream_ptr: int, rank: int = 0, world: int = 1, compact: bool = False):
        """Stream-ordered render into a device buffer (e.g. a torch tensor's data_ptr)."""
        tfd = tf_desc(tf)
        sh = L.ShardDesc(int(rank), int(world), 1 if compact else 0)
        L.check(self._lib.fvsrn_render_device(
            self._h, C.byref(tfd.desc) if tfd else None, C.byref(camera_desc(cam)),
            C.byref(settings_desc(settings)), L.t_arg(t), C.byref(sh), C.c_void_p(out_ptr),
            C.c_void_p(count_ptr) if count_ptr else None, C.c_void_p(stream_ptr)))

    def decode_device(self, res: int, t, begin: int, count: int, out_ptr: int, stream_ptr: int):
        L.check(self._lib.fvsrn_decode_density_device(self._h, int(res), L.t_arg(t), int(begin),
                                                      int(count), C.c_void_p(out_ptr),
                                                      C.c_void_p(stream_ptr)))


class DeviceVolume:
    """A ScalarVolume resident on one GPU (f32, reference layout) for ground-truth DVR."""

    def __init__(self, volume, device: int | None = None):
        lib = L.lib()
        self.device = L.current_device() if device is None else int(device)
        v = np.ascontiguousarray(volume.values, dtype=np.float32)
        if v.ndim != 3:
            raise ValueError(f"volume must be 3D, got {v.shape}")
        h = C.c_void_p()
        L.check(lib.fvsrn_volume_create(L.fptr(v), v.shape[0], v.shape[1], v.shape[2],
                                        self.device, C.byref(h)))
        self._h, self._lib, self.shape = h, lib, v.shape

    def close(self) -> None:
        h, self._h = getattr(self, "_h", None), None
        if h:
            self._lib.fvsrn_volume_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover
            pass

    def render(self, tf, cam, settings, out=None):
        shape = (cam.height, cam.width, 4)
        if out is None:
            out = np.empty(shape, dtype=np.float32)
        elif out.shape != shape or out.dtype != np.float32 or not out.flags.c_contiguous:
            raise ValueError(f"out must be a C-contiguous float32 array of shape {shape}")
        cnt = C.c_uint64(0)
        tfd = tf_desc(tf)
        L.check(self._lib.fvsrn_volume_render(self._h, C.byref(tfd.desc), C.byref(camera_desc(cam)),
                                              C.byref(settings_desc(settings)), L.fptr(out),
                                              C.byref(cnt)))
        return out, int(cnt.value)

    def render_rays(self, tf, origins, dirs, settings):
        o = np.ascontiguousarray(np.asarray(origins, dtype=np.float64).reshape(-1, 3))
        d = np.ascontiguousarray(np.asarray(dirs, dtype=np.float64).reshape(-1, 3))
        if o.shape != d.shape:
            raise ValueError("origins and dirs must have the same shape")
        out = np.empty((len(o), 4), dtype=np.float32)
        cnt = C.c_uint64(0)
        tfd = tf_desc(tf)
        L.check(self._lib.fvsrn_volume_render_rays(self._h, C.byref(tfd.desc), L.dptr(o), L.dptr(d),
                                                   len(o), C.byref(settings_desc(settings)),
                                                   L.fptr(out), C.byref(cnt)))
        return out, int(cnt.value)

    def render_device(self, tf, cam, settings, out_ptr: int, stream_ptr: int, rank: int = 0,
                      world: int = 1, compact: bool = False):
        tfd = tf_desc(tf)
        sh = L.ShardDesc(int(rank), int(world), 1 if compact else 0)
        L.check(self._lib.fvsrn_volume_render_device(
            self._h, C.byref(tfd.desc), C.byref(camera_desc(cam)), C.byref(settings_desc(settings)),
            C.byref(sh), C.c_void_p(out_ptr), C.c_void_p(stream_ptr)))


def _handles(dms):
    return (C.c_void_p * len(dms))(*[dm.handle.value for dm in dms])


def render_multi(dms, tf, cam, settings, t=None, out=None):
    """One frame across the devices of ``dms`` (one DeviceModel per GPU, same model):
    fvsrn_render_multi, round-robin 8x8 screen tiles; returns (frame, summed count)."""
    shape = (cam.height, cam.width, 4)
    if out is None:
        out = L.pooled_empty(shape)
    elif out.shape != shape or out.dtype != np.float32 or not out.flags.c_contiguous:
        raise ValueError(f"out must be a C-contiguous float32 array of shape {shape}")
    cnt = C.c_uint64(0)
    tfd = tf_desc(tf)
    L.check(L.lib().fvsrn_render_multi(_handles(dms), len(dms), C.byref(tfd.desc) if tfd else None,
                                       C.byref(camera_desc(cam)), C.byref(settings_desc(settings)),
                                       L.t_arg(t), L.fptr(out), C.byref(cnt)))
    return out, int(cnt.value)


def decode_multi(dms, res: int, t=None, out=None) -> np.ndarray:
    """decode_volume across the devices of ``dms`` (contiguous lattice slabs per GPU)."""
    n = int(res) ** 3
    if out is None:
        out = L.pooled_empty(n)
    elif out.size != n or out.dtype != np.float32 or not out.flags.c_contiguous:
        raise ValueError(f"out must be a C-contiguous float32 array of {n} elements")
    L.check(L.lib().fvsrn_decode_density_multi(_handles(dms), len(dms), int(res), L.t_arg(t),
                                               L.fptr(out)))
    return out


_DEFAULT_DEVICES: list | None = None


def _parse_devices(spec):
    if spec is None:
        return None
    if isinstance(spec, str):
        spec = spec.strip()
        if not spec:
            return None
        if spec == "all":
            return list(range(max(1, int(L.lib().fvsrn_device_count()))))
        return [int(x) for x in spec.split(",") if x.strip()]
    if isinstance(spec, int):
        return [spec]
    return [int(x) for x in spec]


def set_devices(devices) -> list | None:
    """Default GPU set for render_image / decode_volume calls that pass no ``devices=``:
    a list of device ids, "all", or None (one GPU, the current device).  The environment
    variable FVSRN_DEVICES ("all" or "0,1,2,...") sets the initial default, so reference
    callers (service, CLI, evaluate_views) render on several GPUs unchanged.  Returns the
    previous setting."""
    global _DEFAULT_DEVICES
    prev = _DEFAULT_DEVICES
    _DEFAULT_DEVICES = _parse_devices(devices)
    return prev


def resolve_devices(devices=None) -> list | None:
    """The device list a call should use (None = the single-device path)."""
    import os

    devs = _parse_devices(devices) if devices is not None else _DEFAULT_DEVICES
    if devs is None and devices is None:
        devs = _parse_devices(os.environ.get("FVSRN_DEVICES"))
    if devs is not None and not devs:
        raise ValueError("devices must name at least one GPU")
    return devs


_cache_lock = threading.Lock()


def device_model(model, device: int | None = None, sampled_grids: bool = False) -> DeviceModel:
    """Cached upload of ``model``, rebuilt when its parameters changed since the upload
    (param_fingerprint; ``model.invalidate_device()`` forces a rebuild)."""
    dev = L.current_device() if device is None else int(device)
    fp = param_fingerprint(model, sampled_grids)
    with _cache_lock:
        cache = model.__dict__.setdefault("_device", {})
        hit = cache.get(dev)
        if hit is not None and hit[1 if sampled_grids else 2] == fp:
            return hit[0]
        dm = DeviceModel(model, dev)
        cache[dev] = (dm, param_fingerprint(model, True), param_fingerprint(model, False))
        return dm


def tiles_to_frame_device(gathered_ptr: int, width: int, height: int, world: int, frame_ptr: int,
                          stream_ptr: int) -> None:
    L.check(L.lib().fvsrn_tiles_to_frame_device(C.c_void_p(gathered_ptr), int(width), int(height),
                                                int(world), C.c_void_p(frame_ptr),
                                                C.c_void_p(stream_ptr)))


def shard_slots(width: int, height: int, world: int) -> tuple[int, int]:
    """(n_tiles, max_local_tiles * 64): compact per-rank buffer length in pixels."""
    n_tiles = math.ceil(width / 8) * math.ceil(height / 8)
    return n_tiles, math.ceil(n_tiles / world) * 64


DVR_KERNELS = {"auto": 0, "tc": 1, "ws": 2, "warp": 3, "pipe": 4, "dual": 5}


def set_dvr_kernel(name: str) -> str:
    """Select the DVR kernel for the default fV-SRN shapes ("auto", "tc" = tcgen05/TMEM,
    "ws" = warp-specialised mma.sync, "warp" = single-role mma.sync); returns the previous
    selection.  A measurement switch: every choice renders the same image within fp16
    noise (tests/test_gpu_parity.py::test_dvr_kernel_variants)."""
    prev = L.lib().fvsrn_set_dvr_kernel(DVR_KERNELS[name])
    if prev < 0:
        L.check(-prev)
    return {v: k for k, v in DVR_KERNELS.items()}[prev]


GRID_SAMPLERS = {"auto": 0, "tex": 1, "ldg": 2}


def set_grid_sampler(name: str) -> str:
    """Latent-grid sampler for 16-channel grids: "tex" (texture units, hardware trilinear
    with 8-bit fractional weights), "ldg" (LDG.128 + HFMA2 trilinear) or "auto"; returns
    the previous selection."""
    prev = L.lib().fvsrn_set_grid_sampler(GRID_SAMPLERS[name])
    if prev < 0:
        L.check(-prev)
    return {v: k for k, v in GRID_SAMPLERS.items()}[prev]


def kernel_timer(enable: bool = True) -> None:
    """Start (reset) / stop the calling thread's dominant-kernel timer."""
    L.check(L.lib().fvsrn_kernel_timer(1 if enable else 0))


def kernel_timer_read() -> tuple[float, int, int]:
    """(dominant-kernel ms, its launches, all library launches) since the last read."""
    ms, n, tot = C.c_double(), C.c_int64(), C.c_int64()
    L.check(L.lib().fvsrn_kernel_timer_read(C.byref(ms), C.byref(n), C.byref(tot)))
    return ms.value, n.value, tot.value


def kernel_timer_info() -> str:
    """The kernel (instantiation, MMA path, grid sampler) the timer last recorded."""
    buf = C.create_string_buffer(512)
    L.check(L.lib().fvsrn_kernel_timer_info(buf, 512))
    return buf.value.decode()
