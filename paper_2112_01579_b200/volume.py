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
