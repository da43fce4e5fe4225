"""Minimal scalar-volume container: the return type of ``decode_volume``.

Mirrors ``fvsrn.volume.ScalarVolume`` (volume.py:30-57).  Volume file I/O and
synthetic fields are outside the DVR hot path and not rebuilt.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class ScalarVolume:
    values: np.ndarray                    # (X, Y, Z) float32 in [0, 1], indexed [x, y, z]
    f32_range: tuple | None = None

    def __post_init__(self):
        v = np.asarray(self.values, dtype=np.float32)
        if v.ndim != 3 or min(v.shape) < 1:
            raise ValueError(f"volume must be 3D with positive dims, got {v.shape}")
        if not np.isfinite(v).all():
            raise ValueError("volume contains non-finite values")
        if v.min() < -1e-6 or v.max() > 1 + 1e-6:
            raise ValueError("volume values must lie in [0,1]")
        object.__setattr__(self, "values", v)

    @classmethod
    def _validated(cls, values: np.ndarray) -> "ScalarVolume":
        """Wrap float32 (X,Y,Z) values whose invariants (finite, in [0,1]) were already
        checked on the device by the decode kernel: no second pass over the host copy."""
        obj = object.__new__(cls)
        object.__setattr__(obj, "values", values)
        object.__setattr__(obj, "f32_range", None)
        return obj

    @property
    def dims(self):
        return self.values.shape

    @property
    def resolution(self) -> int:
        return int(max(self.values.shape))


def sample_volume(vol: ScalarVolume, p: np.ndarray) -> np.ndarray:
    """Host trilinear lookup at positions in [0,1]^3 (volume.py:213-255), the training
    targets' ground truth; clamped, exact at vertices, f32 lerps in x, y, z order.
    (The renderer's VolumeSource does the same lookup on the device.)"""
    values = vol.values
    pts = np.atleast_2d(np.asarray(p, dtype=np.float64))
    single = np.asarray(p).ndim == 1
    dims = np.asarray(values.shape[:3])
    coords = np.clip(pts, 0.0, 1.0) * (dims - 1)
    i0 = np.maximum(np.minimum(coords.astype(np.int64), dims - 2), 0)
    f = (coords - i0).astype(values.dtype)
    x0, y0, z0 = i0[:, 0], i0[:, 1], i0[:, 2]
    fx, fy, fz = f[:, 0], f[:, 1], f[:, 2]
    c00 = values[x0, y0, z0] * (1 - fx) + values[x0 + 1, y0, z0] * fx
    c10 = values[x0, y0 + 1, z0] * (1 - fx) + values[x0 + 1, y0 + 1, z0] * fx
    c01 = values[x0, y0, z0 + 1] * (1 - fx) + values[x0 + 1, y0, z0 + 1] * fx
    c11 = values[x0, y0 + 1, z0 + 1] * (1 - fx) + values[x0 + 1, y0 + 1, z0 + 1] * fx
    c0 = c00 * (1 - fy) + c10 * fy
    c1 = c01 * (1 - fy) + c11 * fy
    out = c0 * (1 - fz) + c1 * fz
    return out[0] if single else out
