"""fV-SRN model: config, seeded init, checkpoint I/O (host) and GPU evaluation.

Host-side mirror of ``fvsrn.model`` (model.py:54-528).  ``eval_density``,
``eval_color`` and ``decode_volume`` keep the reference signatures but run on
the B200 through the C ABI (``fvsrn_eval_density`` / ``fvsrn_eval_color`` /
``fvsrn_decode_density``); there is no CPU evaluation path.
"""

from __future__ import annotations

import dataclasses
import json
import struct
from dataclasses import dataclass

import numpy as np

from .grid import (KeyframeGrids, LatentGrid, QuantizedLatentGrid, grid_dequantize, grid_init,
                   grid_quantize)
from .nn import FourierEncoder, MlpParams, fourier_make, init_params, nerf_rows

DIRECTION_MODES = ("pos", "dirP", "dirF")
TIME_MODES = ("none", "direct", "fourier", "both")
_MAGIC = b"FVSN"
_VERSION = 1


class CheckpointError(ValueError):
    pass


@dataclass
class ModelConfig:
    """Same fields, defaults and validation as the reference (model.py:54-121)."""

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

    def __post_init__(self):
        if self.head not in ("density", "color"):
            raise ValueError(f"unknown head {self.head!r}")
        if self.direction_mode not in DIRECTION_MODES:
            raise ValueError(f"unknown direction mode {self.direction_mode!r}")
        if self.time_mode not in TIME_MODES:
            raise ValueError(f"unknown time mode {self.time_mode!r}")
        if self.direction_mode != "pos" and self.head != "color":
            raise ValueError("directional input encodings require the color head")
        if self.fourier_m is not None and self.fourier_m < 0:
            raise ValueError("fourier_m must be non-negative")
        if self.time_mode != "none" and self.keyframe_times is None:
            raise ValueError("time encodings require keyframe_times")
        if self.keyframe_times is not None and self.grid_resolution == 0:
            raise ValueError("temporal models need a latent grid for their keyframes")
        if self.layers < 1 or self.hidden < 1:
            raise ValueError("layers and hidden must be positive")

    @property
    def effective_m(self) -> int:
        if self.fourier_mode == "off":
            return 0
        return (self.hidden - 4) // 2 if self.fourier_m is None else self.fourier_m

    @property
    def spatial_d_in(self) -> int:
        return 6 if self.direction_mode == "dirF" else 3

    @property
    def raw_width(self) -> int:
        return 3 if self.direction_mode == "pos" else 6

    @property
    def time_width(self) -> int:
        n = self.time_fourier_count
        return {"none": 0, "direct": 1, "fourier": 2 * n, "both": 1 + 2 * n}[self.time_mode]

    @property
    def is_temporal(self) -> bool:
        return self.keyframe_times is not None

    @property
    def input_width(self) -> int:
        z = self.grid_channels if self.grid_resolution > 0 else 0
        return self.raw_width + 2 * self.effective_m + self.time_width + z

    @property
    def output_width(self) -> int:
        return 1 if self.head == "density" else 4


def _spatial_encoder(cfg: ModelConfig) -> FourierEncoder:
    m, d = cfg.effective_m, cfg.spatial_d_in
    if m == 0 or cfg.fourier_mode == "off":
        return fourier_make("off", 0, d)
    if cfg.fourier_mode == "nerf":     # truncated stacked identity also for m % d != 0
        return FourierEncoder("nerf", nerf_rows(m, d), d)
    return fourier_make("random", m, d, sigma=cfg.fourier_sigma, seed=cfg.seed + 1000)


@dataclass
class FvsrnModel:
    config: ModelConfig
    params: MlpParams
    spatial_encoder: FourierEncoder
    time_encoder: FourierEncoder | None = None
    grid: LatentGrid | None = None
    keyframes: KeyframeGrids | None = None
    # u8 codes as loaded from a checkpoint (uploaded as-is while the grids still equal
    # their dequantised values, i.e. quantized_fp matches; see device.py)
    quantized: list | None = None
    quantized_fp: tuple | None = None

    @property
    def grids(self) -> list:
        if self.keyframes is not None:
            return self.keyframes.grids
        return [] if self.grid is None else [self.grid]

    @property
    def is_temporal(self) -> bool:
        return self.keyframes is not None

    def trainable_arrays(self) -> list:
        """[*weights, *biases, *grid values] (model.py:155-157): the Adam / gradient order."""
        return [*self.params.weights, *self.params.biases, *(g.values for g in self.grids)]

    def grad_buffer(self):
        """Zero GradientBuffer shaped like the trainable set (model.py:159-162)."""
        from .train import GradientBuffer

        return GradientBuffer.zeros_like_params(self.params, grid_shapes=[g.values.shape for g in self.grids])

    def invalidate_device(self) -> None:
        """Drop the cached device copy (call after mutating parameters in place)."""
        self.__dict__.pop("_device", None)


def model_init(config: ModelConfig) -> FvsrnModel:
    """Seeded initialisation, bit-identical to the reference (model.py:165-187)."""
    params = init_params(config.layers, config.hidden, config.input_width, config.output_width,
                         seed=config.seed, activation=config.activation)
    time_enc = None
    if config.time_mode in ("fourier", "both"):
        time_enc = FourierEncoder("nerf", nerf_rows(config.time_fourier_count, 1), 1)
    grid = keyframes = None
    if config.grid_resolution > 0:
        if config.keyframe_times is None:
            grid = grid_init(config.grid_resolution, config.grid_channels, seed=config.seed + 1)
        else:
            keyframes = KeyframeGrids(
                list(config.keyframe_times),
                [grid_init(config.grid_resolution, config.grid_channels, seed=config.seed + 1 + k)
                 for k in range(len(config.keyframe_times))])
    return FvsrnModel(config, params, _spatial_encoder(config), time_enc, grid, keyframes)


# ------------------------------------------------------------------ GPU evaluation
def _device(model: FvsrnModel):
    from .device import device_model

    return device_model(model)


def eval_density(model: FvsrnModel, p, t=None) -> np.ndarray:
    """Densities in [0,1] at positions (N,3) -- fvsrn_eval_density (model.py:368-373)."""
    if model.config.head != "density":
        raise ValueError("eval_density requires a density-head model")
    return _device(model).eval_density(p, t)


def eval_color(model: FvsrnModel, p, d=None, t=None) -> np.ndarray:
    """(N,4) rgb + sigma -- fvsrn_eval_color (model.py:376-382)."""
    if model.config.head != "color":
        raise ValueError("eval_color requires a color-head model")
    return _device(model).eval_color(p, d, t)


def decode_volume(model: FvsrnModel, resolution: int, t: float | None = None, chunk: int = 1 << 16,
                  out: np.ndarray | None = None, devices=None):
    """Dense density on the linspace(0,1,res)^3 vertex lattice (model.py:385-398).

    ``chunk`` is accepted for signature compatibility; the GPU decodes the
    whole lattice in one launch.  ``out`` (optional): float32 host buffer of
    res^3 values (e.g. ``pinned_empty``) to decode into.  ``devices`` (optional): GPU ids
    (or "all") to split the lattice over in contiguous slabs (fvsrn_decode_density_multi);
    default ``set_devices`` / FVSRN_DEVICES, else one GPU.
    """
    from .device import decode_multi, device_model, resolve_devices
    from .volume import ScalarVolume

    if model.config.head != "density":
        raise ValueError("decode_volume requires a density-head model")
    flat = None if out is None else out.reshape(-1)
    devs = resolve_devices(devices)
    if devs is not None and len(devs) > 1:
        vals = decode_multi([device_model(model, d) for d in devs], resolution, t, out=flat)
    elif devs is not None:
        vals = device_model(model, devs[0]).decode(resolution, t, out=flat)
    else:
        vals = _device(model).decode(resolution, t, out=flat)
    # finite / [0,1] (volume.py:41-49) was checked in the decode kernel (ValueError above)
    return ScalarVolume._validated(vals.reshape((resolution,) * 3))


# ------------------------------------------------------------------ footprint + checkpoints
_PREC_BYTES = {"f16": 2, "f32": 4, "u8": 1}


def memory_footprint(model: FvsrnModel, weight_precision: str = "f16",
                     grid_precision: str = "f32") -> dict:
    """Byte breakdown {network, grid, total} (model.py:404-419)."""
    if weight_precision not in ("f16", "f32"):
        raise ValueError(f"weight precision must be f16 or f32, got {weight_precision!r}")
    if grid_precision not in ("u8", "f32"):
        raise ValueError(f"grid precision must be u8 or f32, got {grid_precision!r}")
    net = model.params.param_count * _PREC_BYTES[weight_precision]
    grid = 0
    for g in model.grids:
        n = g.resolution ** 3 * g.channels
        grid += n + 8 * g.channels if grid_precision == "u8" else 4 * n
    return {"network": net, "grid": grid, "total": net + grid}


def checkpoint_save(model: FvsrnModel, path, weight_precision: str = "f32",
                    grid_precision: str = "f32") -> None:
    """Write the reference ``.fvsrn`` format (model.py:430-472)."""
    if weight_precision not in ("f16", "f32"):
        raise ValueError(f"bad weight precision {weight_precision!r}")
    if grid_precision not in ("u8", "f32"):
        raise ValueError(f"bad grid precision {grid_precision!r}")
    wd = "<f2" if weight_precision == "f16" else "<f4"
    entries, payload, offset = [], [], 0

    def put(name, arr, dtype):
        nonlocal offset
        raw = np.ascontiguousarray(arr, dtype=dtype).tobytes()
        entries.append({"name": name, "shape": list(np.shape(arr)), "dtype": dtype,
                        "offset": offset, "bytes": len(raw)})
        payload.append(raw)
        offset += len(raw)

    for i, (w, b) in enumerate(zip(model.params.weights, model.params.biases)):
        put(f"w{i}", w, wd)
        put(f"b{i}", b, wd)
    for gi, g in enumerate(model.grids):
        if grid_precision == "u8":
            q = grid_quantize(g)
            put(f"grid{gi}_codes", q.codes, "u1")
            put(f"grid{gi}_mins", q.mins, "<f4")
            put(f"grid{gi}_maxs", q.maxs, "<f4")
        else:
            put(f"grid{gi}", g.values, "<f4")
    header = json.dumps({"config": dataclasses.asdict(model.config),
                         "weight_precision": weight_precision, "grid_precision": grid_precision,
                         "sections": entries, "payload_bytes": offset}).encode("utf-8")
    with open(path, "wb") as f:
        f.write(_MAGIC + struct.pack("<II", _VERSION, len(header)) + header)
        for raw in payload:
            f.write(raw)


def checkpoint_load(path) -> FvsrnModel:
    """Read a reference-written ``.fvsrn`` (model.py:475-528), incl. u8 grids.

    u8 grids are dequantised on the host exactly like the reference (for
    ``model.grids``) and their raw codes are kept in ``model.quantized`` so the
    GPU upload can sample the codes directly.
    """
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < 12 or raw[:4] != _MAGIC:
        raise CheckpointError(f"bad checkpoint magic in {path}")
    version, hlen = struct.unpack_from("<II", raw, 4)
    if version != _VERSION:
        raise CheckpointError(f"unsupported checkpoint version {version}")
    if len(raw) < 12 + hlen:
        raise CheckpointError("truncated checkpoint header")
    try:
        header = json.loads(raw[12:12 + hlen].decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as e:
        raise CheckpointError(f"unreadable checkpoint header: {e}") from e
    body = raw[12 + hlen:]
    if len(body) != header["payload_bytes"]:
        raise CheckpointError(f"payload length {len(body)} does not match header "
                              f"({header['payload_bytes']})")
    arrays = {}
    for sec in header["sections"]:
        lo, hi = sec["offset"], sec["offset"] + sec["bytes"]
        if hi > len(body):
            raise CheckpointError(f"section {sec['name']} overruns the payload")
        arrays[sec["name"]] = np.frombuffer(body[lo:hi], dtype=sec["dtype"]).reshape(sec["shape"])
    cfg = ModelConfig(**header["config"])
    model = model_init(cfg)
    quant = []
    try:
        for i in range(model.params.layer_count):
            model.params.weights[i] = arrays[f"w{i}"].astype(np.float32)
            model.params.biases[i] = arrays[f"b{i}"].astype(np.float32)
        grids = []
        for gi in range(len(model.grids)):
            if header["grid_precision"] == "u8":
                q = QuantizedLatentGrid(arrays[f"grid{gi}_codes"].astype(np.uint8),
                                        arrays[f"grid{gi}_mins"].astype(np.float32),
                                        arrays[f"grid{gi}_maxs"].astype(np.float32))
                quant.append(q)
                grids.append(grid_dequantize(q))
            else:
                grids.append(LatentGrid(arrays[f"grid{gi}"].astype(np.float32)))
    except KeyError as e:
        raise CheckpointError(f"checkpoint header inconsistent with payload: missing {e}") from e
    if model.keyframes is not None:
        model.keyframes = KeyframeGrids(list(cfg.keyframe_times), grids)
    elif grids:
        model.grid = grids[0]
    model.quantized = quant or None
    if quant:
        from .device import grid_fingerprint

        model.quantized_fp = grid_fingerprint(model.grids)
    return model


# ------------------------------------------------------------------ standalone pieces
def assemble_input(model: FvsrnModel, p, d=None, t=None) -> np.ndarray:
    """Network input batch [raw | sin(Bx) | cos(Bx) | time | z] for positions (and
    directions / timesteps) (model.py:248-279), evaluated on the GPU in the reference's
    arithmetic (f64 phases, f32 trilinear latent lookup)."""
    from .f32ops import NetDesc

    cfg = model.config
    p = np.atleast_2d(np.asarray(p, dtype=np.float64))
    n = p.shape[0]
    if cfg.direction_mode in ("dirP", "dirF"):
        if d is None:
            raise ValueError(f"direction mode {cfg.direction_mode!r} requires view directions")
        d = np.atleast_2d(np.asarray(d, dtype=np.float64))
        if d.shape != p.shape:
            raise ValueError("directions must match positions in shape")
    else:
        d = None
    if cfg.is_temporal:
        if t is None:
            raise ValueError("temporal model requires timesteps")
        t = np.broadcast_to(np.asarray(t, dtype=np.float64), (n,))
    elif t is not None:
        raise ValueError("timestep supplied to a non-temporal model")
    return NetDesc.for_model(model).run(0, n, cfg.input_width, p=p, d=d, t=t)


def _check_inputs(model, p, d, t):
    cfg = model.config
    p = np.atleast_2d(np.asarray(p, dtype=np.float64))
    n = p.shape[0]
    if cfg.direction_mode in ("dirP", "dirF"):
        if d is None:
            raise ValueError(f"direction mode {cfg.direction_mode!r} requires view directions")
        d = np.atleast_2d(np.asarray(d, dtype=np.float64))
        if d.shape != p.shape:
            raise ValueError("directions must match positions in shape")
    else:
        d = None
    if cfg.is_temporal:
        if t is None:
            raise ValueError("temporal model requires timesteps")
        t = np.broadcast_to(np.asarray(t, dtype=np.float64), (n,)).copy()
    elif t is not None:
        raise ValueError("timestep supplied to a non-temporal model")
    return p, d, t


@dataclass
class ModelForwardContext:
    """What model_backward needs (model.py:280-288).  The GPU backward recomputes the
    layer caches from the positions (same f32 arithmetic), so ``cache`` is None; the
    view directions are kept for direction-mode models."""

    inputs: np.ndarray
    cache: object
    positions: np.ndarray
    times: np.ndarray | None
    dirs: np.ndarray | None = None


def model_forward(model: FvsrnModel, p, d=None, t=None):
    """Raw (pre-head) outputs plus the context for model_backward (model.py:290-299),
    on the GPU f32 evaluator.  ``t`` may be a scalar or one timestep per sample."""
    from .f32ops import NetDesc

    p, d, t = _check_inputs(model, p, d, t)
    nd = NetDesc.for_model(model)
    n, cfg = p.shape[0], model.config
    x = nd.run(0, n, cfg.input_width, p=p, d=d, t=t)
    raw = nd.run(2, n, cfg.output_width, p=p, d=d, t=t)
    return raw, ModelForwardContext(inputs=x, cache=None, positions=p, times=t, dirs=d)


def model_backward(model: FvsrnModel, ctx: ModelForwardContext, raw_bar, grads=None):
    """Accumulate the gradients of sum(raw_bar * raw) into a GradientBuffer
    (model.py:302-335): one CUDA kernel recomputes the forward with its caches, runs the
    MLP backward and adds the latent-grid adjoint into the gradient grids with the
    deterministic scatter (both bracketing keyframe grids for temporal models, weights
    1-w / w); the weight and bias reductions run on the tensor cores (fvsrn_layer_grads)."""
    import ctypes as C

    import torch

    from . import _lib as L
    from .f32ops import NetDesc
    from .train import GradientBuffer

    cfg = model.config
    p, d, t = ctx.positions, ctx.dirs, ctx.times
    n = p.shape[0]
    rb = np.ascontiguousarray(np.asarray(raw_bar, dtype=np.float32).reshape(n, cfg.output_width))
    nd = NetDesc.for_model(model)
    dev = nd.dev
    L_ = model.params.layer_count
    w_in = [cfg.input_width] + [cfg.hidden] * (L_ - 1)
    w_out = [cfg.hidden] * (L_ - 1) + [cfg.output_width]
    f64 = lambda a: None if a is None else torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)  # noqa: E731
    pd, dd, td = f64(p), f64(d), f64(t)
    rbd = torch.as_tensor(rb, device=dev)
    inputs = torch.empty(max(1, n * sum(w_in)), dtype=torch.float32, device=dev)
    deltas = torch.empty(max(1, n * sum(w_out)), dtype=torch.float32, device=dev)
    preacts = torch.empty(max(1, (L_ - 1) * n * cfg.hidden), dtype=torch.float32, device=dev)
    gsizes = [int(g.values.size) for g in model.grids]
    ggrad = torch.zeros(max(1, sum(gsizes)), dtype=torch.float32, device=dev)
    ptr = lambda a: C.c_void_p(a.data_ptr() if a is not None else None)  # noqa: E731
    stream = torch.cuda.current_stream(dev).cuda_stream
    L.check(L.lib().fvsrn_model_grads(C.byref(nd.desc), ptr(nd.params), ptr(pd), ptr(dd), ptr(td),
                                      ptr(rbd), n, C.c_void_p(ggrad.data_ptr() if gsizes else None),
                                      ptr(inputs), ptr(preacts), ptr(deltas), C.c_void_p(stream)))
    # nn.py:252-253 on the tensor cores (fvsrn_layer_grads), in the parameter layout
    nw = sum(int(w.size) for w in model.params.weights)
    flat = torch.zeros(nw + sum(int(b.size) for b in model.params.biases), dtype=torch.float32,
                       device=dev)
    L.check(L.lib().fvsrn_layer_grads(C.byref(nd.desc), ptr(inputs), ptr(deltas), n, n, ptr(flat), 0,
                                      C.c_void_p(stream)))
    host_wb = flat.cpu().numpy()
    gw, gb, o = [], [], 0
    for w in model.params.weights:
        gw.append(host_wb[o:o + w.size].reshape(w.shape).copy())
        o += w.size
    for b in model.params.biases:
        gb.append(host_wb[o:o + b.size].copy())
        o += b.size
    gg, off = [], 0
    host = ggrad.cpu().numpy()
    for g, sz in zip(model.grids, gsizes):
        gg.append(host[off:off + sz].reshape(g.values.shape))
        off += sz
    if grads is None:
        return GradientBuffer(weights=gw, biases=gb, grids=gg)
    for acc, g in zip(grads.weights, gw):
        acc += g
    for acc, g in zip(grads.biases, gb):
        acc += g
    for acc, g in zip(grads.grids, gg):
        acc += g
    return grads


def softplus(x: np.ndarray) -> np.ndarray:
    """Host utility (model.py:338-339); the kernels apply the heads in-kernel."""
    return np.logaddexp(0.0, x)


def apply_density_head(raw: np.ndarray) -> np.ndarray:
    """sigmoid(raw[:, 0]) (model.py:342-343); host utility on host arrays."""
    return (1.0 / (1.0 + np.exp(-np.asarray(raw)[:, 0]))).astype(np.asarray(raw).dtype)


def density_head_backward(raw: np.ndarray, y_bar: np.ndarray) -> np.ndarray:
    """Adjoint of apply_density_head (model.py:346-350); host utility on host arrays."""
    raw = np.asarray(raw)
    s = 1.0 / (1.0 + np.exp(-raw[:, 0]))
    out = np.zeros_like(raw)
    out[:, 0] = y_bar * s * (1.0 - s)
    return out


def color_head_backward(raw: np.ndarray, y_bar: np.ndarray) -> np.ndarray:
    """Adjoint of apply_color_head (model.py:360-365); host utility on host arrays."""
    raw = np.asarray(raw)
    out = np.empty_like(raw)
    s = 1.0 / (1.0 + np.exp(-raw[:, :3]))
    out[:, :3] = y_bar[:, :3] * s * (1.0 - s)
    out[:, 3] = y_bar[:, 3] * (1.0 / (1.0 + np.exp(-raw[:, 3])))
    return out


def apply_color_head(raw: np.ndarray) -> np.ndarray:
    """sigmoid rgb, softplus sigma (model.py:353-357); host utility on host arrays."""
    raw = np.asarray(raw)
    out = np.empty_like(raw)
    out[:, :3] = 1.0 / (1.0 + np.exp(-raw[:, :3]))
    out[:, 3] = softplus(raw[:, 3])
    return out
