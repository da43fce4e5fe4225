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


# ------------------------------------------------------------------ SSIM (host metric)
_SSIM_WIN, _SSIM_SIGMA, _SSIM_C1, _SSIM_C2 = 11, 1.5, 0.01 ** 2, 0.03 ** 2


def _luma(a: np.ndarray) -> np.ndarray:
    """Rec. 709 luminance of the rgb channels, or the array itself if 2-D (f64)."""
    if a.ndim == 3:
        return (0.2126 * a[:, :, 0] + 0.7152 * a[:, :, 1] + 0.0722 * a[:, :, 2]).astype(np.float64)
    return a.astype(np.float64)


def _gauss_mean(img: np.ndarray) -> np.ndarray:
    """Separable normalised Gaussian window mean, zero padding, fully supported windows."""
    from scipy.ndimage import correlate1d

    r = np.arange(_SSIM_WIN, dtype=np.float64) - (_SSIM_WIN - 1) / 2.0
    k = np.exp(-(r ** 2) / (2.0 * _SSIM_SIGMA ** 2))
    k /= k.sum()
    out = correlate1d(correlate1d(img, k, axis=0, mode="constant"), k, axis=1, mode="constant")
    h = (_SSIM_WIN - 1) // 2
    return out[h:-h, h:-h]


def metric_ssim(a, b) -> float:
    """Mean local SSIM of the luminance, 11x11 Gaussian window, sigma 1.5, K = (0.01, 0.03)
    on a unit dynamic range (imaging.py:156-177); a host metric like metric_psnr."""
    x = a.data if isinstance(a, Image) else np.asarray(getattr(a, "values", a))
    y = b.data if isinstance(b, Image) else np.asarray(getattr(b, "values", b))
    if x.shape != y.shape:
        raise ValueError(f"shape mismatch: {x.shape} vs {y.shape}")
    gx, gy = _luma(x), _luma(y)
    if min(gx.shape) < _SSIM_WIN:
        raise ValueError(f"image smaller than the {_SSIM_WIN}x{_SSIM_WIN} SSIM window")
    mx, my = _gauss_mean(gx), _gauss_mean(gy)
    vx = _gauss_mean(gx * gx) - mx ** 2
    vy = _gauss_mean(gy * gy) - my ** 2
    cxy = _gauss_mean(gx * gy) - mx * my
    s = ((2 * mx * my + _SSIM_C1) * (2 * cxy + _SSIM_C2)) / ((mx ** 2 + my ** 2 + _SSIM_C1) * (vx + vy + _SSIM_C2))
    return float(s.mean())
