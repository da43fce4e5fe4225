"""Cameras, float images and the parity metric (imaging.py:14-126 of the reference)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

PSNR_CAP_DB = 99.0


@dataclass(frozen=True)
class Camera:
    """Pinhole camera: eye/target/up in world space, vertical FOV (radians)."""

    eye: np.ndarray
    target: np.ndarray
    up: np.ndarray
    fov_y: float
    width: int
    height: int

    def __post_init__(self):
        eye, target, up = (np.asarray(v, dtype=np.float64) for v in (self.eye, self.target, self.up))
        if eye.shape != (3,) or target.shape != (3,) or up.shape != (3,):
            raise ValueError("eye, target, up must be 3-vectors")
        view = target - eye
        if np.linalg.norm(view) < 1e-12:
            raise ValueError("eye and target coincide")
        if np.linalg.norm(np.cross(view, up)) < 1e-12:
            raise ValueError("up is parallel to the view direction")
        if not 0.0 < self.fov_y < np.pi:
            raise ValueError("fov_y must be in (0, pi)")
        if self.width < 1 or self.height < 1:
            raise ValueError("image dimensions must be positive")
        object.__setattr__(self, "eye", eye)
        object.__setattr__(self, "target", target)
        object.__setattr__(self, "up", up)


@dataclass(frozen=True)
class Image:
    """(H, W, 4) float32: premultiplied rgb + accumulated opacity."""

    data: np.ndarray

    def __post_init__(self):
        d = np.asarray(self.data, dtype=np.float32)
        if d.ndim != 3 or d.shape[2] != 4:
            raise ValueError(f"image data must be (H, W, 4), got {d.shape}")
        if not np.isfinite(d).all():
            raise ValueError("image contains non-finite values")
        object.__setattr__(self, "data", d)

    @classmethod
    def _from_device(cls, data: np.ndarray) -> "Image":
        """Wrap a renderer framebuffer without the host-side scan: fvsrn_render
        already enforced the finiteness invariant on the device."""
        obj = object.__new__(cls)
        object.__setattr__(obj, "data", data)
        return obj

    @property
    def width(self) -> int:
        return int(self.data.shape[1])

    @property
    def height(self) -> int:
        return int(self.data.shape[0])


def _values(a) -> np.ndarray:
    if isinstance(a, Image):
        return a.data
    if hasattr(a, "values"):
        return a.values
    return np.asarray(a)


def metric_psnr(a, b) -> float:
    """PSNR (dB, peak 1) over every element incl. alpha, capped at 99 dB."""
    x = _values(a).astype(np.float64)
    y = _values(b).astype(np.float64)
    if x.shape != y.shape:
        raise ValueError(f"shape mismatch: {x.shape} vs {y.shape}")
    mse = float(np.mean(np.square(x - y)))
    if mse <= 10.0 ** (-PSNR_CAP_DB / 10.0):
        return PSNR_CAP_DB
    return float(-10.0 * np.log10(mse))


def png_bytes(img: Image) -> bytes:
    """8-bit RGBA PNG encoding (imaging.py:74-80), for the service caller."""
    import io

    from PIL import Image as PILImage

    u8 = np.floor(np.clip(img.data, 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)
    buf = io.BytesIO()
    PILImage.fromarray(u8, mode="RGBA").save(buf, format="PNG")
    return buf.getvalue()


def write_png(img: Image, path) -> None:
    with open(path, "wb") as f:
        f.write(png_bytes(img))
