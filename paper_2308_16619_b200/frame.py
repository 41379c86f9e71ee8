"""Frame bookkeeping around the batched cache decode, on the GPU.

Drop-in mirrors of the reference's LOD selection and palette visibility
(csvol/render.py:145-158, :174-187) computed by CUDA kernels (csrc/csv_cache.cu)
over a device-resident volume, plus the minimal `Camera` / `TransferFunction`
value types they read (render.py:37-98).  The renderer itself is out of scope.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .device import GpuVolume, _ptr, _stream_handle
from .errors import ConfigError


@dataclass(frozen=True)
class Camera:
    """Pinhole camera (render.py:37-60): only position, fov and height enter LOD selection."""

    position: tuple[float, float, float]
    forward: tuple[float, float, float] = (0.0, 0.0, 1.0)
    up: tuple[float, float, float] = (0.0, 1.0, 0.0)
    fov: float = math.pi / 3
    width: int = 256
    height: int = 256

    def __post_init__(self):
        if not 0 < self.fov < math.pi:
            raise ConfigError(f"fov must be in (0, pi), got {self.fov}")
        if self.width < 1 or self.height < 1:
            raise ConfigError("image must be at least 1x1")


@dataclass(frozen=True)
class TransferFunction:
    """Label -> opacity mapping (render.py:74-98); overrides map label -> (r, g, b, a)."""

    default_alpha: float = 1.0
    overrides: dict = field(default_factory=dict)

    def tables(self) -> tuple[np.ndarray, np.ndarray]:
        if not self.overrides:
            return np.empty(0, np.uint32), np.empty((0, 4), np.float64)
        labels = np.array(sorted(self.overrides), dtype=np.uint32)
        rgba = np.array([self.overrides[int(l)] for l in labels], dtype=np.float64)
        return labels, rgba


def _volume(v):
    if isinstance(v, GpuVolume):
        return v, False
    # a CsvContainer: upload directory + palettes for this call (geometry and
    # palettes are all these kernels read; the detail section stays on the host)
    return v.to_device(cold_detail=True), True


def desired_lods_device(volume: GpuVolume, camera: Camera, out=None, stream=None):
    """Per-brick LOD (uint8 CUDA tensor over the volume's brick range), render.py:145-158."""
    torch = volume._torch
    if out is None:
        out = torch.empty(max(volume.n_bricks, 1), dtype=torch.uint8, device=volume.device)
    px, py, pz = (float(c) for c in camera.position)
    with torch.cuda.device(volume.device):
        _lib.check(_lib.lib().csv_desired_lods(volume._h, px, py, pz, math.tan(camera.fov / 2.0),
                                                float(camera.height), _ptr(out), _stream_handle(torch, stream)))
    return out[: volume.n_bricks]


def visibility_mask_device(volume: GpuVolume, tf: TransferFunction, out=None, stream=None):
    """Per-brick visibility (uint8 CUDA tensor, 1 = some palette label has alpha > 0), render.py:174-187."""
    torch = volume._torch
    labels, rgba = tf.tables()
    if out is None:
        out = torch.empty(max(volume.n_bricks, 1), dtype=torch.uint8, device=volume.device)
    lab = torch.from_numpy(np.ascontiguousarray(labels, dtype=np.uint32).view(np.int32)).to(volume.device)
    alp = torch.from_numpy(np.ascontiguousarray(rgba[:, 3] if rgba.size else np.zeros(0), dtype=np.float64)).to(
        volume.device)
    with torch.cuda.device(volume.device):
        _lib.check(_lib.lib().csv_visibility_mask(volume._h, volume.palette_entries, _ptr(lab) if labels.size else 0,
                                                   _ptr(alp) if labels.size else 0, int(labels.size),
                                                   float(tf.default_alpha), _ptr(out), _stream_handle(torch, stream)))
    return out[: volume.n_bricks]


def desired_lods(container, camera: Camera) -> np.ndarray:
    """Reference-shaped API: numpy uint8 per brick (render.py:145-158), computed on the GPU."""
    v, own = _volume(container)
    try:
        return desired_lods_device(v, camera).cpu().numpy()
    finally:
        if own:
            v.close()


def visibility_mask(container, tf: TransferFunction) -> np.ndarray:
    """Reference-shaped API: numpy bool per brick (render.py:174-187), computed on the GPU."""
    v, own = _volume(container)
    try:
        return visibility_mask_device(v, tf).cpu().numpy().astype(bool)
    finally:
        if own:
            v.close()
