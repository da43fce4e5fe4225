"""Latent feature grids (host containers; sampling happens inside the CUDA kernels).

Mirrors ``fvsrn.grid`` (grid.py:18-44, 140-203): (R,R,R,F) f32 vertex grids
(z fastest, channels innermost), the u8 quantised form with per-channel
min/max, and keyframe sequences for time-varying models.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

GRID_INIT_STD = 0.1


@dataclass
class LatentGrid:
    values: np.ndarray   # (R, R, R, F) float32

    def __post_init__(self):
        v = self.values
        if v.ndim != 4 or len({v.shape[0], v.shape[1], v.shape[2]}) != 1:
            raise ValueError(f"grid values must be (R,R,R,F), got {v.shape}")
        if v.shape[0] < 2 or v.shape[3] < 1:
            raise ValueError("need R >= 2 and F >= 1")

    @property
    def resolution(self) -> int:
        return int(self.values.shape[0])

    @property
    def channels(self) -> int:
        return int(self.values.shape[3])


def grid_init(resolution: int, channels: int, seed: int = 0) -> LatentGrid:
    """N(0, 0.1^2) draws from default_rng(seed), stored f32."""
    draws = np.random.default_rng(seed).normal(0.0, GRID_INIT_STD,
                                               size=(resolution, resolution, resolution, channels))
    return LatentGrid(draws.astype(np.float32))


@dataclass(frozen=True)
class QuantizedLatentGrid:
    codes: np.ndarray    # (R,R,R,F) uint8
    mins: np.ndarray     # (F,) float32
    maxs: np.ndarray     # (F,) float32

    @property
    def resolution(self) -> int:
        return int(self.codes.shape[0])

    @property
    def channels(self) -> int:
        return int(self.codes.shape[3])


def grid_quantize(grid: LatentGrid) -> QuantizedLatentGrid:
    """Per-channel affine map of [min, max] onto 0..255, rounding half up."""
    v = grid.values
    lo = v.min(axis=(0, 1, 2))
    hi = v.max(axis=(0, 1, 2))
    span = hi - lo
    scale = np.where(span > 0, span, 1.0)
    q = np.clip(np.floor((v - lo) / scale * 255.0 + 0.5), 0, 255).astype(np.uint8)
    q[..., span <= 0] = 0
    return QuantizedLatentGrid(q, lo.astype(np.float32), hi.astype(np.float32))


def grid_dequantize(q: QuantizedLatentGrid) -> LatentGrid:
    vals = q.mins + q.codes.astype(np.float32) / 255.0 * (q.maxs - q.mins)
    return LatentGrid(vals.astype(np.float32))


@dataclass
class KeyframeGrids:
    times: list
    grids: list

    def __post_init__(self):
        if not self.grids:
            raise ValueError("need at least one keyframe")
        if len(self.times) != len(self.grids):
            raise ValueError("times and grids must pair up")
        if any(b <= a for a, b in zip(self.times[:-1], self.times[1:])):
            raise ValueError("keyframe times must be strictly increasing")
        shapes = {(g.resolution, g.channels) for g in self.grids}
        if len(shapes) != 1:
            raise ValueError("all keyframe grids must share (R, F)")

    @property
    def resolution(self) -> int:
        return self.grids[0].resolution

    @property
    def channels(self) -> int:
        return self.grids[0].channels

    @property
    def span(self):
        return self.times[0], self.times[-1]


def _positions(p) -> tuple[np.ndarray, bool]:
    arr = np.asarray(p, dtype=np.float64)
    single = arr.ndim == 1
    pts = np.atleast_2d(arr)
    if pts.shape[1] != 3:
        raise ValueError(f"positions must have 3 components, got {np.shape(p)}")
    return np.ascontiguousarray(pts), single


def grid_sample(grid: LatentGrid, p) -> np.ndarray:
    """Trilinear lookup at positions (N,3) or (3,) -> (N,F) or (F,) (grid.py:115-121),
    evaluated on the GPU with the reference's f32 arithmetic."""
    from .f32ops import NetDesc

    pts, single = _positions(p)
    F = grid.channels
    nd = NetDesc([np.zeros((1, 3 + F), np.float32)], [np.zeros(1, np.float32)], "snake_alt", "density",
                 3 + F, grids=[grid.values])
    out = nd.run(1, len(pts), F, p=pts)
    return out[0] if single else out


def grid_sample_backward(grid: LatentGrid, p, z_bar, grad: np.ndarray) -> None:
    """Scatter-add trilinear-weighted adjoints into ``grad`` (shaped like grid.values), in
    place (grid.py:123-137), by a CUDA scatter kernel (``fvsrn_grid_sample_backward``).
    Positions receive no gradient.  Device atomics replace the reference's sequential
    loop: sums agree up to f32 rounding order."""
    import ctypes as C

    import torch

    from . import _lib as L

    if grad.shape != grid.values.shape:
        raise ValueError(f"gradient shape {grad.shape} does not match grid {grid.values.shape}")
    pts, _ = _positions(p)
    zb = np.atleast_2d(np.asarray(z_bar, dtype=np.float32))
    if zb.shape != (len(pts), grid.channels):
        raise ValueError(f"adjoint shape {zb.shape} does not match (N,{grid.channels})")
    dev = torch.device("cuda", L.current_device())
    pd = torch.as_tensor(np.ascontiguousarray(pts, dtype=np.float64), device=dev)
    zd = torch.as_tensor(np.ascontiguousarray(zb), device=dev)
    gd = torch.as_tensor(np.ascontiguousarray(grad, dtype=np.float32), device=dev).contiguous()
    L.check(L.lib().fvsrn_grid_sample_backward(int(grid.resolution), int(grid.channels),
                                               C.c_void_p(pd.data_ptr()), C.c_void_p(zd.data_ptr()),
                                               len(pts), C.c_void_p(gd.data_ptr()),
                                               C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    grad[...] = gd.cpu().numpy().reshape(grad.shape)


def keyframe_bracket(kfg: "KeyframeGrids", t: float) -> tuple[int, int, float]:
    """Indices of the bracketing keyframes and the blend weight of the upper one
    (grid.py:206-219)."""
    times = kfg.times
    tc = min(max(float(t), times[0]), times[-1])
    hi = int(np.searchsorted(times, tc, side="left"))
    if hi == 0:
        return 0, 0, 0.0
    lo = hi - 1
    if hi >= len(times):
        return len(times) - 1, len(times) - 1, 0.0
    if times[hi] == tc:
        return hi, hi, 0.0
    return lo, hi, float((tc - times[lo]) / (times[hi] - times[lo]))


def keyframe_sample(kfg: "KeyframeGrids", p, t: float) -> np.ndarray:
    """Latent vectors at positions and a continuous timestep (grid.py:222-230), GPU."""
    from .f32ops import NetDesc

    if not np.isfinite(t):
        raise ValueError("timestep must be finite")
    pts, single = _positions(p)
    F = kfg.channels
    nd = NetDesc([np.zeros((1, 3 + F), np.float32)], [np.zeros(1, np.float32)], "snake_alt", "density",
                 3 + F, grids=[g.values for g in kfg.grids], keyframe_times=list(kfg.times))
    out = nd.run(1, len(pts), F, p=pts, t=np.full(len(pts), float(t)))
    return out[0] if single else out
