"""DVR of an fV-SRN model on the B200 -- drop-in for ``fvsrn.render``.

``render_image(ModelSource(model, tf), camera, settings)`` keeps the reference
call (render.py:314-332) but crosses host->device once per frame: ray setup,
the per-sample network evaluation, transfer function, compositing and early
termination all run inside one fused sm_100a kernel (fvsrn_render), with no
wavefront and no global intermediates.  ``raymarch_forward`` maps to
fvsrn_render_rays over explicit rays (render.py:203-238).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .device import DeviceVolume, decode_multi, device_model, render_multi, resolve_devices
from .imaging import Camera, Image

EPS_BLEND = 1e-5


@dataclass
class RayState:
    color: np.ndarray   # (N, 3) premultiplied rgb, before the background
    alpha: np.ndarray   # (N,)

    def copy(self) -> "RayState":
        return RayState(self.color.copy(), self.alpha.copy())


@dataclass(frozen=True)
class RenderSettings:
    """render.py:49-69: same fields, defaults and validation."""

    stepsize: float = 1.0 / 64.0
    max_steps: int = 4096
    background: tuple = (0.0, 0.0, 0.0)
    early_term_alpha: float = 0.999
    eps_blend: float = EPS_BLEND
    use_fused: bool = False
    threads: int = 1

    def __post_init__(self):
        if self.stepsize <= 0:
            raise ValueError("stepsize must be positive")
        if not 0.0 <= self.early_term_alpha <= 1.0:
            raise ValueError("early termination threshold must lie in [0,1]")

    @classmethod
    def for_voxels(cls, volume_resolution: int, stepsize_voxels: float = 1.0,
                   **kwargs) -> "RenderSettings":
        return cls(stepsize=stepsize_voxels / volume_resolution, **kwargs)


class ModelSource:
    """Model + TF (+ t) bound for rendering; uploads the model once to the GPU.

    Validation follows render.py:147-156.  ``use_fused`` is accepted for
    signature compatibility: every evaluation runs the fused GPU kernel (which
    has no 48 KB capacity limit, so 6x64 networks render too).
    """

    def __init__(self, model, tf=None, t: float | None = None, use_fused: bool = False,
                 device: int | None = None):
        head = model.config.head
        if head == "density" and tf is None:
            raise ValueError("density-head models need a transfer function to render")
        if head == "color" and tf is not None:
            raise ValueError("color-head models do not take a transfer function")
        if t is not None and not model.is_temporal:
            raise ValueError("timestep supplied to a non-temporal model")
        if t is None and model.is_temporal:
            raise ValueError("temporal model requires a timestep to render")
        self.model = model
        self.tf = tf
        self.t = t
        self.use_fused = use_fused
        self._device = device
        device_model(model, device)            # upload now (the per-frame path only checks)
        self.last_eval_count = 0

    @property
    def device_model(self):
        """The model's device copy, re-validated on every call with the cheap parameter
        fingerprint (exact weights/biases, sampled grids: microseconds), so a source bound
        before an optimiser step renders the updated model as the reference would."""
        return device_model(self.model, self._device, sampled_grids=True)

    def device_models(self, devices):
        """One device copy per GPU in ``devices`` (uploaded on first use, re-validated)."""
        return [device_model(self.model, d, sampled_grids=True) for d in devices]

    def sample(self, p, d):
        """The per-sample source protocol (render.py:182-186), evaluated on the GPU."""
        m = self.model
        if m.config.head == "density":
            dens = self.device_model.eval_density(p, self.t)
            dc = np.clip(dens, 0.0, 1.0)
            rgb = np.stack([np.interp(dc, self.tf.xs, self.tf.rgbs[:, c]) for c in range(3)], -1)
            return rgb.astype(np.float32), np.interp(dc, self.tf.xs, self.tf.sigmas).astype(np.float32)
        out = self.device_model.eval_color(p, d, self.t)
        return out[:, :3], out[:, 3]


class VolumeSource:
    """Ground-truth source: trilinear density through a transfer function
    (render.py:132-141).  The volume is uploaded once (f32, reference layout) and
    frames render with fvsrn_volume_render: same ray setup, TF, compositing and early
    termination as ModelSource, densities bit-identical to sample_volume."""

    def __init__(self, volume, tf, device: int | None = None):
        self.volume = volume
        self.tf = tf
        self.device_volume = DeviceVolume(volume, device)
        self.last_eval_count = 0

    def sample(self, p, d):
        """The per-sample source protocol (render.py:139-141) on host arrays: trilinear
        density (volume.py:213-255) through the TF.  Frames and ray batches do not come
        through here; they render on the GPU (fvsrn_volume_render)."""
        from .transfer import tf_eval
        from .volume import sample_volume

        return tf_eval(self.tf, sample_volume(self.volume, p))


EPS_BLEND = 1e-5


def ray_box_intersect(origins: np.ndarray, dirs: np.ndarray):
    """Entry/exit distances against the unit cube (render.py:97-106); host utility on
    host arrays (the renderer does this per ray in f64 in ray_setup_kernel)."""
    d = np.where(np.abs(dirs) < 1e-12, 1e-12, dirs)
    t_lo = (0.0 - origins) / d
    t_hi = (1.0 - origins) / d
    tmin = np.maximum(np.minimum(t_lo, t_hi).max(axis=1), 0.0)
    tmax = np.maximum(t_lo, t_hi).min(axis=1)
    return tmin, tmax, tmax > tmin


def composite_step(c_acc, a_acc, rgb, sigma, ds, eps_blend: float = EPS_BLEND):
    """One front-to-back blend step (render.py:109-117); host utility on host arrays
    (the renderer composites in-kernel)."""
    alpha = np.maximum(np.minimum(1.0 - eps_blend, -np.expm1(-sigma * ds)), 0.0)
    trans = (1.0 - a_acc) * alpha
    return c_acc + trans[..., None] * rgb, a_acc + trans


def composite_invert(c_acc, a_acc, rgb, sigma, ds, eps_blend: float = EPS_BLEND):
    """Exact inverse of composite_step (render.py:120-129); host utility (the GPU
    raymarch_backward inverts the blend in-kernel)."""
    alpha = np.maximum(np.minimum(1.0 - eps_blend, -np.expm1(-sigma * ds)), 0.0)
    if np.any(alpha >= 1.0 - eps_blend / 2 + eps_blend):
        raise FloatingPointError("blend inversion unstable: alpha too close to 1")
    a_prev = (a_acc - alpha) / (1.0 - alpha)
    return c_acc - ((1.0 - a_prev) * alpha)[..., None] * rgb, a_prev


def camera_rays(camera: Camera):
    """Per-pixel (origins, unit dirs), row-major from the top-left (render.py:72-94).

    Host utility kept for API compatibility; the render path builds the same
    rays on the GPU from the per-frame basis (bit-identical, see tests).
    """
    from .device import camera_basis

    fwd, right, up, half_w, half_h = camera_basis(camera)
    w, h = camera.width, camera.height
    xs = ((np.arange(w) + 0.5) / w * 2.0 - 1.0) * half_w
    ys = (1.0 - (np.arange(h) + 0.5) / h * 2.0) * half_h
    gx, gy = np.meshgrid(xs, ys)
    dirs = (fwd + gx[..., None] * right) + gy[..., None] * up
    dirs = dirs.reshape(-1, 3)
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    return np.broadcast_to(camera.eye, dirs.shape).copy(), dirs


def _is_gpu_source(source) -> bool:
    return isinstance(source, (ModelSource, VolumeSource))


def _require_sampler(source):
    if not callable(getattr(source, "sample", None)):
        raise TypeError(f"{type(source).__name__} has no sample(p, d) method (render.py:226)")
    return source


def _march_host_source(source, origins, dirs, settings: RenderSettings, want_states: bool):
    """render.py:203-238 for a caller-defined source: any object with ``sample(p, d) ->
    (rgb (N,3), sigma (N,))`` (the reference's duck-typed protocol).  Its sample() is the
    caller's host code, so the march is a host wavefront: the rays still active at step k
    are sampled together at t = tmin + (k + 1/2) ds and blended front to back in f64
    (composite_step), with early termination unless ``want_states``.  ModelSource and
    VolumeSource never come here: they march on the GPU."""
    o = np.asarray(origins, dtype=np.float64).reshape(-1, 3)
    d = np.asarray(dirs, dtype=np.float64).reshape(-1, 3)
    tmin, tmax, hit = ray_box_intersect(o, d)
    span = np.where(hit, tmax - tmin, 0.0)
    steps = np.zeros(len(o), dtype=np.int64)
    steps[hit] = np.maximum(np.minimum(np.ceil(span[hit] / settings.stepsize).astype(np.int64),
                                       settings.max_steps), 1)
    ds = np.where(steps > 0, span / np.maximum(steps, 1), 0.0)
    color = np.zeros((len(o), 3))
    alpha = np.zeros(len(o))
    live = steps > 0
    for k in range(int(steps.max()) if len(o) else 0):
        live &= k < steps
        idx = np.flatnonzero(live)
        if idx.size == 0:
            break
        pos = o[idx] + (tmin[idx] + (k + 0.5) * ds[idx])[:, None] * d[idx]
        rgb, sigma = source.sample(pos, d[idx])
        color[idx], alpha[idx] = composite_step(color[idx], alpha[idx], np.asarray(rgb, np.float64),
                                                np.asarray(sigma, np.float64), ds[idx],
                                                settings.eps_blend)
        if not want_states:
            live[idx] &= ~(alpha[idx] > settings.early_term_alpha)
    px = np.empty((len(o), 4), dtype=np.float32)
    px[:, :3] = color + (1.0 - alpha)[:, None] * np.asarray(settings.background, dtype=np.float64)
    px[:, 3] = alpha
    return px, (RayState(color, alpha) if want_states else None)


def raymarch_forward(source, origins, dirs, settings: RenderSettings, want_states: bool = False):
    """March explicit rays; returns (pixels (N,4) f32, RayState | None) like render.py:203-238.

    With ``want_states`` early termination is disabled (as in the reference) and
    the terminal (C, A) pair is returned.
    """
    if not _is_gpu_source(source):
        return _march_host_source(_require_sampler(source), origins, dirs, settings, want_states)
    src = source
    if want_states:
        settings = RenderSettings(settings.stepsize, settings.max_steps, settings.background,
                                  1.0, settings.eps_blend)
    if isinstance(src, VolumeSource):
        px, cnt = src.device_volume.render_rays(src.tf, origins, dirs, settings)
    else:
        px, cnt = src.device_model.render_rays(src.tf, origins, dirs, settings, src.t)
    src.last_eval_count = cnt
    states = None
    if want_states:
        a = px[:, 3].astype(np.float64)
        bg = np.asarray(settings.background, dtype=np.float64)
        states = RayState(px[:, :3].astype(np.float64) - (1.0 - a)[:, None] * bg, a)
    return px, states


def render_rays(source, origins, dirs, settings: RenderSettings) -> np.ndarray:
    return raymarch_forward(source, origins, dirs, settings)[0]


def render_image(source, camera: Camera, settings: RenderSettings | None = None,
                 out: np.ndarray | None = None, devices=None) -> Image:
    """Full frame through the fused DVR kernel (render.py:314-332).

    ``settings.threads`` is ignored (the GPU parallelises over rays); the output
    is deterministic and bit-identical across repeats.  The number of network
    evaluations is recorded in ``source.last_eval_count``.  ``out`` (optional,
    new): a float32 (H,W,4) host buffer to render into -- with
    ``pinned_empty`` an interactive viewer reuses one page-locked framebuffer and
    the device->host read runs at full bandwidth; the returned Image views it.
    ``devices`` (optional, new): GPU ids (or "all") to split the frame over by 8x8 screen
    tiles in this process (fvsrn_render_multi); default ``set_devices`` /
    FVSRN_DEVICES, else one GPU.  The frame is bit-identical to the 1-GPU render.
    """
    settings = settings or RenderSettings()
    if not _is_gpu_source(source):
        o, d = camera_rays(camera)
        px, _ = _march_host_source(_require_sampler(source), o, d, settings, False)
        return Image(data=px.reshape(camera.height, camera.width, 4))
    src = source
    devs = resolve_devices(devices)
    if isinstance(src, VolumeSource):
        data, cnt = src.device_volume.render(src.tf, camera, settings, out=out)
    elif devs is not None and len(devs) > 1:
        data, cnt = render_multi(src.device_models(devs), src.tf, camera, settings, src.t, out=out)
    elif devs is not None:
        data, cnt = device_model(src.model, devs[0], sampled_grids=True).render(
            src.tf, camera, settings, src.t, out=out)
    else:
        data, cnt = src.device_model.render(src.tf, camera, settings, src.t, out=out)
    src.last_eval_count = cnt
    return Image._from_device(data)


def render_image_rgba8(source, camera: Camera, settings: RenderSettings | None = None,
                       out: np.ndarray | None = None) -> np.ndarray:
    """``render_image`` followed by the 8-bit quantisation of ``png_bytes``
    (imaging.py:74-80, ``floor(clip(v, 0, 1) * 255 + 0.5)``), fused on the device:
    returns the (H, W, 4) uint8 frame, bit-identical to quantising ``render_image``'s
    output on the host, with a quarter of the device->host bytes.  New (the service's
    render path); ``out`` may be a ``pinned_empty(..., np.uint8)`` buffer."""
    src = source
    if not isinstance(src, ModelSource):
        raise TypeError("render_image_rgba8 renders ModelSource instances")
    settings = settings or RenderSettings()
    data, cnt = src.device_model.render_rgba8(src.tf, camera, settings, src.t, out=out)
    src.last_eval_count = cnt
    return data


def fibonacci_cameras(n: int, width: int, height: int, radius: float = 2.2,
                      fov_y: float = np.pi / 4, center=(0.5, 0.5, 0.5)) -> list:
    """Deterministic orbit on a Fibonacci sphere (train.py:209-224): the measurement views."""
    c = np.asarray(center, dtype=np.float64)
    golden = np.pi * (3.0 - np.sqrt(5.0))
    cams = []
    for i in range(n):
        y = 1.0 - 2.0 * (i + 0.5) / n
        r = np.sqrt(max(0.0, 1.0 - y * y))
        phi = golden * i
        v = np.array([r * np.cos(phi), y, r * np.sin(phi)])
        up = np.array([0.0, 1.0, 0.0]) if abs(v[1]) < 0.95 else np.array([1.0, 0.0, 0.0])
        cams.append(Camera(eye=c + radius * v, target=c, up=up, fov_y=fov_y, width=width,
                           height=height))
    return cams
