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
