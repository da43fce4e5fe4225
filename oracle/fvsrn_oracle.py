"""CPU oracle for the fV-SRN DVR hot path -- TEST INFRASTRUCTURE ONLY.

This module is a plain numpy (+ optional numba) restatement of the reference
algorithm (`/root/reference/pkg/src/fvsrn`, package ``fvsrn`` 0.1.0).  It is the
checker the GPU path is compared against and the CPU baseline timed by
``bench.py``.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  The product package
``paper_2112_01579_b200`` never imports it and has no CPU fallback.

Parity is PINNED: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by the reference itself
(``tests/golden/make_golden.py``, run in the build container where
``/root/reference`` is importable).

Every function cites the reference file:line it restates (paths relative to
``/root/reference/pkg/src/fvsrn/``).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np

try:  # numba is in the image; the oracle still works (slowly) without it
    from numba import njit, prange

    _HAVE_NUMBA = True
except Exception:  # pragma: no cover
    _HAVE_NUMBA = False

EPS_BLEND = 1e-5            # render.py:31
GRID_INIT_STD = 0.1         # grid.py:15
PSNR_CAP_DB = 99.0          # imaging.py:11
ACTIVATIONS = ("relu", "sigmoid", "softplus", "snake", "snake_alt")   # nn.py:15


# --------------------------------------------------------------------------
# configuration + initialisation (model.py:54-187, nn.py:47-168, grid.py:40-44)
# --------------------------------------------------------------------------
@dataclass
class OConfig:
    """Restates ModelConfig (model.py:54-121): same fields, same defaults."""

    head: str = "density"
    layers: int = 4
    hidden: int = 32
    activation: str = "snake_alt"
    fourier_mode: str = "nerf"
    fourier_m: int | None = None
    fourier_sigma: float = 1.0
    grid_resolution: int = 32
    grid_channels: int = 16
    direction_mode: str = "pos"
    time_mode: str = "none"
    time_fourier_count: int = 4
    keyframe_times: list | None = None
    time_range: list | None = None
    seed: int = 0

    @property
    def effective_m(self):                       # model.py:90-94
        if self.fourier_mode == "off":
            return 0
        return self.fourier_m if self.fourier_m is not None else (self.hidden - 4) // 2

    @property
    def spatial_d_in(self):                      # model.py:96-98
        return 6 if self.direction_mode == "dirF" else 3

    @property
    def raw_width(self):                         # model.py:100-102
        return 6 if self.direction_mode in ("dirP", "dirF") else 3

    @property
    def time_width(self):                        # model.py:104-108
        return {"none": 0, "direct": 1, "fourier": 2 * self.time_fourier_count,
                "both": 1 + 2 * self.time_fourier_count}[self.time_mode]

    @property
    def input_width(self):                       # model.py:114-117
        latent = self.grid_channels if self.grid_resolution > 0 else 0
        return self.raw_width + 2 * self.effective_m + self.time_width + latent

    @property
    def output_width(self):                      # model.py:119-121
        return 1 if self.head == "density" else 4


@dataclass
class OModel:
    config: OConfig
    weights: list
    biases: list
    b_matrix: np.ndarray                 # spatial Fourier B (m, d_in) f32
    time_b: np.ndarray | None = None     # time Fourier B (L, 1) f32
    grids: list = field(default_factory=list)   # (R,R,R,F) f32 each
    keyframe_times: list | None = None


def nerf_rows(m, d_in):
    """nn.py:47-57: row i = 2*pi*2^(i//d_in) on axis i%d_in, stored f32."""
    rows = np.zeros((m, d_in), dtype=np.float32)
    for i in range(m):
        block, axis = divmod(i, d_in)
        rows[i, axis] = 2.0 * np.pi * (2.0 ** block)
    return rows


def init_params(layers, hidden, d_in, d_out, seed, dtype=np.float32):
    """nn.py:154-168: Xavier-uniform (out,in) weights drawn in layer order, zero bias."""
    widths = [d_in] + [hidden] * (layers - 1) + [d_out]
    rng = np.random.default_rng(seed)
    ws, bs = [], []
    for i in range(layers):
        fi, fo = widths[i], widths[i + 1]
        bound = np.sqrt(6.0 / (fi + fo))
        ws.append(rng.uniform(-bound, bound, size=(fo, fi)).astype(dtype))
        bs.append(np.zeros(fo, dtype=dtype))
    return ws, bs


def grid_init(res, ch, seed):
    """grid.py:40-44: N(0, 0.1^2) f32, shape (R,R,R,F)."""
    rng = np.random.default_rng(seed)
    return rng.normal(0.0, GRID_INIT_STD, size=(res,) * 3 + (ch,)).astype(np.float32)


def model_init(cfg: OConfig) -> OModel:
    """model.py:165-187 (+ _make_spatial_encoder model.py:124-133, nn.py:60-76)."""
    ws, bs = init_params(cfg.layers, cfg.hidden, cfg.input_width, cfg.output_width, cfg.seed)
    m, d_in = cfg.effective_m, cfg.spatial_d_in
    if m == 0 or cfg.fourier_mode == "off":
        b = np.zeros((0, d_in), dtype=np.float32)
    elif cfg.fourier_mode == "nerf":
        b = nerf_rows(m, d_in)
    else:  # "random": nn.py:69-72 with seed+1000 (model.py:132-133)
        rng = np.random.default_rng(cfg.seed + 1000)
        b = rng.normal(0.0, 2.0 * np.pi * cfg.fourier_sigma, size=(m, d_in)).astype(np.float32)
    tb = None
    if cfg.time_mode in ("fourier", "both"):
        tb = nerf_rows(cfg.time_fourier_count, 1)
    grids = []
    if cfg.grid_resolution > 0:
        if cfg.keyframe_times is not None:
            grids = [grid_init(cfg.grid_resolution, cfg.grid_channels, cfg.seed + 1 + k)
                     for k in range(len(cfg.keyframe_times))]
        else:
            grids = [grid_init(cfg.grid_resolution, cfg.grid_channels, cfg.seed + 1)]
    return OModel(cfg, ws, bs, b, tb, grids,
                  list(cfg.keyframe_times) if cfg.keyframe_times is not None else None)


# --------------------------------------------------------------------------
# latent grid (grid.py:47-84, 206-230)
# --------------------------------------------------------------------------
def _cell_coords(res, p):
    """grid.py:47-53: clip to [0,1], scale by R-1, i0 = min(int, R-2), frac f64."""
    pts = np.atleast_2d(np.asarray(p, dtype=np.float64))
    coords = np.clip(pts, 0.0, 1.0) * (res - 1)
    i0 = np.minimum(coords.astype(np.int64), res - 2)
    return i0, coords - i0


import threading

_TLS = threading.local()   # .serial=True inside render_image's thread pool (no nested pools)


def _serial():
    return getattr(_TLS, "serial", False)


if _HAVE_NUMBA:
    @njit(cache=False, parallel=True, fastmath=False)
    def _gather_nb(values, i0, frac, out):
        n, f = out.shape
        for k in prange(n):
            x0, y0, z0 = i0[k, 0], i0[k, 1], i0[k, 2]
            fx, fy, fz = frac[k, 0], frac[k, 1], frac[k, 2]
            gx, gy, gz = np.float32(1.0) - fx, np.float32(1.0) - fy, np.float32(1.0) - fz
            w = (gx * gy * gz, gx * gy * fz, gx * fy * gz, gx * fy * fz,
                 fx * gy * gz, fx * gy * fz, fx * fy * gz, fx * fy * fz)
            for c in range(f):
                out[k, c] = (w[0] * values[x0, y0, z0, c] + w[1] * values[x0, y0, z0 + 1, c]
                             + w[2] * values[x0, y0 + 1, z0, c]
                             + w[3] * values[x0, y0 + 1, z0 + 1, c]
                             + w[4] * values[x0 + 1, y0, z0, c]
                             + w[5] * values[x0 + 1, y0, z0 + 1, c]
                             + w[6] * values[x0 + 1, y0 + 1, z0, c]
                             + w[7] * values[x0 + 1, y0 + 1, z0 + 1, c])


def grid_sample(values, p):
    """grid.py:115-121 / _gather_kernel grid.py:59-84: f32 weights, 8-corner sum."""
    res = values.shape[0]
    i0, frac = _cell_coords(res, p)
    frac = frac.astype(np.float32)
    out = np.empty((i0.shape[0], values.shape[3]), dtype=np.float32)
    if _HAVE_NUMBA and len(i0) >= 1:
        (_gather_nb_serial if _serial() else _gather_nb)(values, i0, frac, out)
        return out
    x0, y0, z0 = i0[:, 0], i0[:, 1], i0[:, 2]
    fx, fy, fz = frac[:, 0:1], frac[:, 1:2], frac[:, 2:3]
    gx, gy, gz = 1 - fx, 1 - fy, 1 - fz
    v = values
    out[:] = (gx * gy * gz * v[x0, y0, z0] + gx * gy * fz * v[x0, y0, z0 + 1]
              + gx * fy * gz * v[x0, y0 + 1, z0] + gx * fy * fz * v[x0, y0 + 1, z0 + 1]
              + fx * gy * gz * v[x0 + 1, y0, z0] + fx * gy * fz * v[x0 + 1, y0, z0 + 1]
              + fx * fy * gz * v[x0 + 1, y0 + 1, z0] + fx * fy * fz * v[x0 + 1, y0 + 1, z0 + 1])
    return out


def keyframe_bracket(times, t):
    """Scalar form of model.py:200-209 / grid.py:206-219 (t constant per frame)."""
    times = np.asarray(times, dtype=np.float64)
    tc = min(max(float(t), times[0]), times[-1])
    hi = int(np.searchsorted(times, tc, side="left"))
    hi = min(max(hi, 0), len(times) - 1)
    lo = hi - 1 if (hi > 0 and times[hi] != tc) else hi
    w = (tc - times[lo]) / (times[hi] - times[lo]) if hi > lo else 0.0
    return lo, hi, w


def normalize_time(model: OModel, t):
    """model.py:190-197."""
    cfg = model.config
    if cfg.time_range is not None:
        t0, t1 = cfg.time_range
    else:
        t0, t1 = model.keyframe_times[0], model.keyframe_times[-1]
    if t1 == t0:
        return 0.0
    return (min(max(float(t), t0), t1) - t0) / (t1 - t0)


def time_features(model: OModel, t):
    """model.py:236-245 for a per-frame scalar t -> (T,) f64."""
    cfg = model.config
    tn = normalize_time(model, t)
    parts = []
    if cfg.time_mode in ("direct", "both"):
        parts.append(np.array([tn]))
    if cfg.time_mode in ("fourier", "both"):
        ph = tn * model.time_b[:, 0].astype(np.float64)
        parts.extend([np.sin(ph), np.cos(ph)])
    return np.concatenate(parts) if parts else np.zeros(0)


def latent_batch(model: OModel, p, t):
    """model.py:219-233: static grid or (1-w)*lo + w*hi keyframe blend (f32)."""
    if model.keyframe_times is not None:
        lo, hi, w = keyframe_bracket(model.keyframe_times, t)
        z = grid_sample(model.grids[lo], p)
        if hi != lo:
            wk = np.float32(w)
            z = (np.float32(1.0) - wk) * z + wk * grid_sample(model.grids[hi], p)
        return z
    return grid_sample(model.grids[0], p)


def assemble_input(model: OModel, p, d=None, t=None):
    """model.py:248-279: [p (|d) | sin(Bv) | cos(Bv) | time | z], phases f64, cast f32."""
    cfg = model.config
    p = np.atleast_2d(np.asarray(p, dtype=np.float64))
    n = p.shape[0]
    if cfg.direction_mode in ("dirP", "dirF"):
        d = np.atleast_2d(np.asarray(d, dtype=np.float64))
        raw = np.concatenate([p, d], axis=1)
    else:
        raw = p
    parts = [raw]
    if model.b_matrix.shape[0] > 0:
        enc_in = raw if cfg.direction_mode == "dirF" else p
        phase = enc_in @ model.b_matrix.T.astype(np.float64)
        parts.extend([np.sin(phase), np.cos(phase)])
    if cfg.time_width > 0:
        parts.append(np.broadcast_to(time_features(model, t), (n, cfg.time_width)))
    if cfg.grid_resolution > 0:
        parts.append(latent_batch(model, p, t))
    x = np.concatenate(parts, axis=1)
    return np.ascontiguousarray(x, dtype=np.float32)


# --------------------------------------------------------------------------
# MLP + heads (nn.py:18-29, 195-204; model.py:338-365)
# --------------------------------------------------------------------------
def act_eval(kind, x):
    """nn.py:18-29."""
    if kind == "relu":
        return np.maximum(x, 0.0)
    if kind == "sigmoid":
        return 1.0 / (1.0 + np.exp(-x))
    if kind == "softplus":
        return np.logaddexp(0.0, x)
    if kind == "snake":
        return x + np.sin(x) ** 2
    if kind == "snake_alt":
        return 0.5 * x + np.sin(x) ** 2
    raise ValueError(kind)


_ACT = {k: i for i, k in enumerate(ACTIVATIONS)}

if _HAVE_NUMBA:
    @njit(cache=False, parallel=True, fastmath=True)
    def _mlp_nb(x, wflat, bflat, dims, act, out):
        """Per-sample f32 MLP over 32-sample tiles (the blocked evaluator of
        fused.py:142-240, restated); used for large batches (CPU timing)."""
        n = x.shape[0]
        nl = dims.shape[0] - 1
        maxw = 0
        for i in range(nl + 1):
            maxw = max(maxw, dims[i])
        ntile = (n + 31) // 32
        for t in prange(ntile):
            lo = t * 32
            cnt = min(n, lo + 32) - lo
            a = np.zeros((maxw, 32), dtype=np.float32)
            b = np.zeros((maxw, 32), dtype=np.float32)
            for s in range(cnt):
                for j in range(dims[0]):
                    a[j, s] = x[lo + s, j]
            wo = 0
            bo = 0
            for li in range(nl):
                din, dout = dims[li], dims[li + 1]
                for r in range(dout):
                    bias = bflat[bo + r]
                    for s in range(32):
                        b[r, s] = bias
                    for k in range(din):
                        wv = wflat[wo + r * din + k]
                        for s in range(32):
                            b[r, s] += wv * a[k, s]
                    if li < nl - 1:
                        for s in range(32):
                            v = b[r, s]
                            if act == 0:
                                v = max(v, np.float32(0.0))
                            elif act == 1:
                                v = np.float32(1.0) / (np.float32(1.0) + np.exp(-v))
                            elif act == 2:
                                v = np.log1p(np.exp(v)) if v < 20.0 else v
                            else:
                                sv = np.sin(v)
                                v = (v if act == 3 else np.float32(0.5) * v) + sv * sv
                            b[r, s] = v
                wo += din * dout
                bo += dout
                a, b = b, a
            for s in range(cnt):
                for j in range(dims[nl]):
                    out[lo + s, j] = a[j, s]


if _HAVE_NUMBA:
    _gather_nb_serial = njit(cache=False, parallel=False, nogil=True)(_gather_nb.py_func)
    _mlp_nb_serial = njit(cache=False, parallel=False, fastmath=True, nogil=True)(_mlp_nb.py_func)


def mlp_eval(model: OModel, x):
    """nn.py:195-204: h = act(h @ W.T + b) per layer, last layer linear, f32."""
    if _HAVE_NUMBA and len(x) >= 256:
        x = np.ascontiguousarray(x, dtype=np.float32)
        dims = np.array([model.weights[0].shape[1]] + [w.shape[0] for w in model.weights], np.int64)
        wflat = np.concatenate([w.ravel() for w in model.weights]).astype(np.float32)
        bflat = np.concatenate(model.biases).astype(np.float32)
        out = np.empty((len(x), dims[-1]), np.float32)
        (_mlp_nb_serial if _serial() else _mlp_nb)(x, wflat, bflat, dims,
                                                   _ACT[model.config.activation], out)
        return out
    h = np.asarray(x, dtype=np.float32)
    last = len(model.weights) - 1
    for i, (w, b) in enumerate(zip(model.weights, model.biases)):
        h = h @ w.T + b
        if i < last:
            h = act_eval(model.config.activation, h).astype(np.float32)
    return h


def _sigmoid64(x):
    return 1.0 / (1.0 + np.exp(-np.asarray(x, dtype=np.float64)))


def apply_head(model: OModel, raw):
    """model.py:342-343 (density: sigmoid) / model.py:353-357 (color: sigmoid rgb, softplus)."""
    if model.config.head == "density":
        return _sigmoid64(raw[:, 0]).astype(np.float32)
    out = np.empty_like(raw)
    out[:, :3] = _sigmoid64(raw[:, :3])
    out[:, 3] = np.logaddexp(0.0, raw[:, 3])
    return out


def eval_density(model: OModel, p, t=None):
    """model.py:368-373."""
    return apply_head(model, mlp_eval(model, assemble_input(model, p, None, t)))


def eval_color(model: OModel, p, d=None, t=None):
    """model.py:376-382."""
    return apply_head(model, mlp_eval(model, assemble_input(model, p, d, t)))


def decode_volume(model: OModel, res, t=None, chunk=1 << 16):
    """model.py:385-398: linspace(0,1,res)^3 vertex lattice, ij order, [x,y,z]."""
    axis = np.linspace(0.0, 1.0, res)
    gx, gy, gz = np.meshgrid(axis, axis, axis, indexing="ij")
    pts = np.stack([gx, gy, gz], axis=-1).reshape(-1, 3)
    out = np.empty(len(pts), dtype=np.float32)
    for lo in range(0, len(pts), chunk):
        out[lo:lo + chunk] = eval_density(model, pts[lo:lo + chunk], t)
    return out.reshape((res,) * 3)


def checkpoint_load(path) -> OModel:
    """model.py:475-528: 'FVSR' magic, <u32 version, <u32 header length>, JSON header
    (config, sections {name, dtype, shape, offset, bytes}, grid_precision), payload.
    Weights/biases are cast to f32; u8 grids dequantised as grid.py:170-172
    (v = min + code/255 * (max - min), f32)."""
    import json
    import struct

    with open(path, "rb") as f:
        raw = f.read()
    _version, hlen = struct.unpack_from("<II", raw, 4)
    header = json.loads(raw[12:12 + hlen].decode("utf-8"))
    payload = raw[12 + hlen:]
    sec = {}
    for s in header["sections"]:
        a = np.frombuffer(payload[s["offset"]:s["offset"] + s["bytes"]], dtype=s["dtype"])
        sec[s["name"]] = a.reshape(s["shape"])
    model = model_init(OConfig(**header["config"]))
    for i in range(len(model.weights)):
        model.weights[i] = sec[f"w{i}"].astype(np.float32)
        model.biases[i] = sec[f"b{i}"].astype(np.float32)
    for gi in range(len(model.grids)):
        if header["grid_precision"] == "u8":
            mins = sec[f"grid{gi}_mins"].astype(np.float32)
            maxs = sec[f"grid{gi}_maxs"].astype(np.float32)
            codes = sec[f"grid{gi}_codes"].astype(np.float32)
            model.grids[gi] = (mins + codes / 255.0 * (maxs - mins)).astype(np.float32)
        else:
            model.grids[gi] = sec[f"grid{gi}"].astype(np.float32)
    return model


# --------------------------------------------------------------------------
# transfer function (transfer.py:57-65, 89-113)
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class OTF:
    xs: np.ndarray
    rgbs: np.ndarray
    sigmas: np.ndarray


def tf_from_points(points):
    return OTF(np.asarray([p[0] for p in points], np.float32),
               np.asarray([p[1] for p in points], np.float32),
               np.asarray([p[2] for p in points], np.float32))


_BLACK = (0.0, 0.0, 0.0)
TF_PRESETS = {   # transfer.py:89-113
    "grayscale": tf_from_points([(0.0, _BLACK, 0.0), (1.0, (1.0, 1.0, 1.0), 10.0)]),
    "warm": tf_from_points([(0.0, _BLACK, 0.0), (0.33, (0.8, 0.1, 0.05), 3.0),
                            (0.66, (1.0, 0.8, 0.1), 6.0), (1.0, (1.0, 1.0, 1.0), 10.0)]),
    "two_peaks": tf_from_points([(0.0, _BLACK, 0.0), (0.3, (0.6, 0.1, 0.9), 25.0),
                                 (0.45, _BLACK, 0.0), (0.6, (1.0, 0.9, 0.1), 25.0),
                                 (0.75, _BLACK, 0.0), (1.0, _BLACK, 0.0)]),
}


def tf_eval(tf: OTF, density):
    """transfer.py:57-65: clamp to [0,1], np.interp per channel, cast f32."""
    d = np.clip(np.asarray(density, dtype=np.float32), 0.0, 1.0)
    rgb = np.stack([np.interp(d, tf.xs, tf.rgbs[:, c]) for c in range(3)], axis=-1)
    sigma = np.interp(d, tf.xs, tf.sigmas)
    return rgb.astype(np.float32), sigma.astype(np.float32)


# --------------------------------------------------------------------------
# cameras + ray geometry (render.py:72-106, 189-200; train.py:209-224)
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class OCamera:
    eye: np.ndarray
    target: np.ndarray
    up: np.ndarray
    fov_y: float
    width: int
    height: int


def camera_rays(cam: OCamera):
    """render.py:72-94: pinhole, pixel centres, row-major from top-left, f64."""
    eye = np.asarray(cam.eye, np.float64)
    forward = np.asarray(cam.target, np.float64) - eye
    forward = forward / np.linalg.norm(forward)
    right = np.cross(forward, np.asarray(cam.up, np.float64))
    right = right / np.linalg.norm(right)
    up = np.cross(right, forward)
    h, w = cam.height, cam.width
    half_h = np.tan(cam.fov_y / 2.0)
    half_w = half_h * w / h
    xs = ((np.arange(w) + 0.5) / w * 2.0 - 1.0) * half_w
    ys = (1.0 - (np.arange(h) + 0.5) / h * 2.0) * half_h
    gx, gy = np.meshgrid(xs, ys)
    dirs = forward[None, None] + gx[..., None] * right[None, None] + gy[..., None] * up[None, None]
    dirs = dirs.reshape(-1, 3)
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    origins = np.broadcast_to(eye, dirs.shape).copy()
    return origins, dirs


def camera_basis(cam: OCamera):
    """The per-frame (forward, right, up, half_w, half_h) of render.py:78-86."""
    eye = np.asarray(cam.eye, np.float64)
    forward = np.asarray(cam.target, np.float64) - eye
    forward = forward / np.linalg.norm(forward)
    right = np.cross(forward, np.asarray(cam.up, np.float64))
    right = right / np.linalg.norm(right)
    up = np.cross(right, forward)
    half_h = np.tan(cam.fov_y / 2.0)
    half_w = half_h * cam.width / cam.height
    return forward, right, up, half_w, half_h


def ray_box_intersect(o, d):
    """render.py:97-106: slab test vs [0,1]^3."""
    dd = np.where(np.abs(d) < 1e-12, 1e-12, d)
    t_lo = (0.0 - o) / dd
    t_hi = (1.0 - o) / dd
    tmin = np.minimum(t_lo, t_hi).max(axis=1)
    tmax = np.maximum(t_lo, t_hi).min(axis=1)
    tmin = np.maximum(tmin, 0.0)
    return tmin, tmax, tmax > tmin


def march_geometry(o, d, stepsize, max_steps):
    """render.py:189-200: n = min(ceil(L/step), max_steps), n >= 1 if hit; ds = L/n."""
    tmin, tmax, valid = ray_box_intersect(o, d)
    length = np.where(valid, tmax - tmin, 0.0)
    n = np.zeros(len(o), dtype=np.int64)
    n[valid] = np.minimum(np.ceil(length[valid] / stepsize).astype(np.int64), max_steps)
    n[valid] = np.maximum(n[valid], 1)
    ds = np.where(n > 0, length / np.maximum(n, 1), 0.0)
    return tmin, ds, n


def fibonacci_cameras(n, width, height, radius=2.2, fov_y=np.pi / 4, center=(0.5, 0.5, 0.5)):
    """train.py:209-224."""
    center = np.asarray(center, dtype=np.float64)
    golden = np.pi * (3.0 - np.sqrt(5.0))
    cams = []
    for i in range(n):
        y = 1.0 - 2.0 * (i + 0.5) / n
        r = np.sqrt(max(0.0, 1.0 - y * y))
        phi = golden * i
        dv = np.array([r * np.cos(phi), y, r * np.sin(phi)])
        up = np.array([0.0, 1.0, 0.0]) if abs(dv[1]) < 0.95 else np.array([1.0, 0.0, 0.0])
        cams.append(OCamera(center + radius * dv, center, up, fov_y, width, height))
    return cams


# --------------------------------------------------------------------------
# compositing + march (render.py:109-117, 203-238, 314-332)
# --------------------------------------------------------------------------
def composite_step(c, a, rgb, sigma, ds, eps_blend=EPS_BLEND):
    """render.py:109-117 (f64)."""
    alpha = np.minimum(1.0 - eps_blend, -np.expm1(-sigma * ds))
    alpha = np.maximum(alpha, 0.0)
    tr = (1.0 - a) * alpha
    return c + tr[..., None] * rgb, a + tr


def model_sample(model: OModel, tf: OTF | None, p, d, t):
    """ModelSource.sample render.py:168-186 (density head -> tf_eval)."""
    if model.config.head == "density":
        return tf_eval(tf, eval_density(model, p, t))
    out = eval_color(model, p, d if model.config.direction_mode != "pos" else None, t)
    return out[:, :3], out[:, 3]


def sample_volume(values, p):
    """volume.py:213-255 (_trilinear): clip, per-axis (dims-1) scale, i0 = max(min(int,
    dims-2), 0), f32 fractions, lerp x then y then z (f32)."""
    p = np.atleast_2d(np.asarray(p, np.float64))
    dims = np.asarray(values.shape[:3])
    coords = np.clip(p, 0.0, 1.0) * (dims - 1)
    i0 = np.maximum(np.minimum(coords.astype(np.int64), dims - 2), 0)
    f = (coords - i0).astype(values.dtype)
    x0, y0, z0 = i0[:, 0], i0[:, 1], i0[:, 2]
    fx, fy, fz = f[:, 0], f[:, 1], f[:, 2]
    v = values
    c00 = v[x0, y0, z0] * (1 - fx) + v[x0 + 1, y0, z0] * fx
    c10 = v[x0, y0 + 1, z0] * (1 - fx) + v[x0 + 1, y0 + 1, z0] * fx
    c01 = v[x0, y0, z0 + 1] * (1 - fx) + v[x0 + 1, y0, z0 + 1] * fx
    c11 = v[x0, y0 + 1, z0 + 1] * (1 - fx) + v[x0 + 1, y0 + 1, z0 + 1] * fx
    c0 = c00 * (1 - fy) + c10 * fy
    c1 = c01 * (1 - fy) + c11 * fy
    return c0 * (1 - fz) + c1 * fz


@dataclass
class OVolume:
    """A ground-truth source: VolumeSource(volume, tf) of render.py:132-141."""

    values: np.ndarray


def raymarch_forward(model, tf, o, d, stepsize, max_steps=4096, background=(0, 0, 0),
                     et_alpha=0.999, eps_blend=EPS_BLEND, t=None, counter=None):
    """render.py:203-238 wavefront march; counter[0] += evaluated samples.
    ``model`` may be an OModel or an OVolume (ground-truth VolumeSource)."""
    o = np.asarray(o, np.float64)
    d = np.asarray(d, np.float64)
    n = len(o)
    tmin, ds, nst = march_geometry(o, d, stepsize, max_steps)
    c = np.zeros((n, 3))
    a = np.zeros(n)
    term = np.zeros(n, dtype=bool)
    max_n = int(nst.max()) if n else 0
    for k in range(max_n):
        active = (k < nst) & ~term
        if not active.any():
            break
        idx = np.nonzero(active)[0]
        tk = tmin[idx] + (k + 0.5) * ds[idx]
        p = o[idx] + tk[:, None] * d[idx]
        if isinstance(model, OVolume):
            rgb, sig = tf_eval(tf, sample_volume(model.values, p))
        else:
            rgb, sig = model_sample(model, tf, p, d[idx], t)
        if counter is not None:
            counter[0] += len(idx)
        c[idx], a[idx] = composite_step(c[idx], a[idx], rgb.astype(np.float64),
                                        sig.astype(np.float64), ds[idx], eps_blend)
        term[idx] |= a[idx] > et_alpha
    bg = np.asarray(background, np.float64)
    px = np.empty((n, 4), np.float32)
    px[:, :3] = c + (1.0 - a)[:, None] * bg
    px[:, 3] = a
    return px


def render_image(model, tf, cam: OCamera, stepsize, max_steps=4096, background=(0, 0, 0),
                 et_alpha=0.999, t=None, counter=None, rows=None, threads=1):
    """render.py:314-332 -> (H,W,4) f32; ``threads`` > 1 splits the rays into
    threads*4 chunks on a thread pool exactly like render.py:320-331.  ``rows``
    restricts to a row subset (the bounded CPU-baseline sample; other rows stay 0)."""
    o, d = camera_rays(cam)
    img = np.zeros((cam.height * cam.width, 4), np.float32)
    if rows is None:
        sel = np.arange(cam.height * cam.width)
    else:
        sel = (np.asarray(rows)[:, None] * cam.width + np.arange(cam.width)[None]).reshape(-1)
    if threads <= 1 or len(sel) < 4096:
        chunks = [sel[lo:lo + (1 << 16)] for lo in range(0, len(sel), 1 << 16)]
    else:
        chunks = [c for c in np.array_split(sel, threads * 4) if len(c)]
    counts = [[0] for _ in chunks]

    def run(i):
        _TLS.serial = threads > 1
        c = chunks[i]
        img[c] = raymarch_forward(model, tf, o[c], d[c], stepsize, max_steps, background,
                                  et_alpha, t=t, counter=counts[i])

    if threads <= 1:
        for i in range(len(chunks)):
            run(i)
    else:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=threads) as pool:
            list(pool.map(run, range(len(chunks))))
    if counter is not None:
        counter[0] += sum(c[0] for c in counts)
    return img.reshape(cam.height, cam.width, 4)


def metric_psnr(a, b):
    """imaging.py:117-126: all channels, peak 1, capped at 99 dB."""
    x = np.asarray(a, np.float64)
    y = np.asarray(b, np.float64)
    mse = float(np.mean((x - y) ** 2))
    if mse <= 10 ** (-PSNR_CAP_DB / 10.0):
        return PSNR_CAP_DB
    return float(10.0 * np.log10(1.0 / mse))


def set_threads(n: int | None = None):
    """Pin numba's pool (the reference's NUMBA_NUM_THREADS knob)."""
    if _HAVE_NUMBA:
        import numba
        numba.set_num_threads(n or os.cpu_count() or 1)
