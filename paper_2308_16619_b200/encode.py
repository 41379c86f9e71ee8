"""GPU encoder and synthetic volumes.

`compress_volume` keeps the reference signature (container.py:374-453) and
returns a host CsvContainer whose bytes equal the reference's; the work runs
in csrc/csv_encode.cu (pyramid, parallel reuse ops, one-warp palette replay,
reverse rANS lanes, ordered assembly).  `compress_volume_device` keeps the
result in HBM and hands it to the decoder without a host round trip.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .codec import DIRECTORY_DTYPE
from .container import CompressionConfig, CsvContainer, _parse_head
from .errors import ConfigError


class GpuEncoded:
    """A container produced on the GPU, resident in HBM (csv_encoded handle)."""

    def __init__(self, handle, device, keepalive=None):
        self._h = handle
        self.device = device
        self._keep = keepalive
        L = _lib.lib()
        head = (ctypes.c_uint8 * 120)()
        n = ctypes.c_uint64()
        sizes = (ctypes.c_uint64 * 3)()
        _lib.check(L.csv_encoded_info(self._h, head, ctypes.byref(n), sizes))
        self.head = bytes(head)
        self.n_bricks = n.value
        self.sizes = tuple(sizes)     # palette entries, coarse bytes, detail bytes
        ptrs = [ctypes.c_void_p() for _ in range(4)]
        _lib.check(L.csv_encoded_device_ptrs(self._h, *[ctypes.byref(p) for p in ptrs]))
        self.ptrs = tuple(p.value or 0 for p in ptrs)

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().csv_encoded_free(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def payload_bytes(self) -> int:
        return self.sizes[0] * 4 + self.sizes[1] + self.sizes[2]

    def to_container(self) -> CsvContainer:
        """Copy to host: the same CsvContainer the reference's compress_volume returns."""
        meta, tables, _ = _parse_head(self.head)
        directory = np.zeros(self.n_bricks, dtype=DIRECTORY_DTYPE)
        pal = np.zeros(max(self.sizes[0], 1), dtype=np.uint32)
        coarse = np.zeros(max(self.sizes[1], 1), dtype=np.uint8)
        detail = np.zeros(max(self.sizes[2], 1), dtype=np.uint8)
        import torch
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().csv_encoded_copy_to_host(
                self._h, directory.ctypes.data, pal.ctypes.data, coarse.ctypes.data, detail.ctypes.data,
                torch.cuda.current_stream().cuda_stream))
        return CsvContainer(meta, tables, directory, pal[: self.sizes[0]], coarse[: self.sizes[1]],
                            detail[: self.sizes[2]])

    def to_volume(self, brick_range=None):
        """A GpuVolume over the encoded blobs (borrowed; keep this object alive)."""
        from .device import GpuVolume
        b0, b1 = brick_range if brick_range is not None else (0, self.n_bricks)
        dp, pp, cp, xp = self.ptrs
        vol = GpuVolume(self.head, (dp + 44 * b0, b1 - b0), (pp, self.sizes[0]), (cp, self.sizes[1]),
                        (xp, self.sizes[2]), brick_begin=b0, brick_end=b1, device=self.device, on_device=True)
        vol._keep = (self,)
        return vol


def _check_volume(volume) -> tuple[np.ndarray, int]:
    """Input validation of compress_volume (container.py:377-386)."""
    if volume.ndim != 3 or min(volume.shape) < 1:
        raise ConfigError(f"need a non-empty 3-D volume, got shape {volume.shape}")
    if volume.dtype not in (np.uint16, np.uint32):
        if np.issubdtype(volume.dtype, np.integer):
            if volume.size and (int(volume.min()) < 0 or int(volume.max()) > 0xFFFFFFFF):
                raise ConfigError("labels must fit an unsigned 32-bit range")
        else:
            raise ConfigError(f"labels must be integers, got dtype {volume.dtype}")
    if volume.dtype == np.uint16:
        return np.ascontiguousarray(volume), 16
    return np.ascontiguousarray(volume, dtype=np.uint32), 32


def compress_volume_device(d_volume, config: CompressionConfig | None = None, width: int | None = None,
                           label_width: int | None = None, stream=None) -> GpuEncoded:
    """Encode a (Z, Y, X) CUDA tensor (int32/uint32 storage, or int16/uint16 with width=16)."""
    torch = _lib.require_cuda()
    config = config or CompressionConfig()
    if width is None:
        width = 16 if d_volume.element_size() == 2 else 32
    if d_volume.element_size() * 8 != width or not d_volume.is_contiguous() or d_volume.dim() != 3:
        raise ConfigError("device volume must be a contiguous 3-D tensor of the given width")
    z, y, x = d_volume.shape
    h = ctypes.c_void_p()
    with torch.cuda.device(d_volume.device):
        s = stream or torch.cuda.current_stream()
        _lib.check(_lib.lib().csv_encode_volume(
            d_volume.device.index, d_volume.data_ptr(), width, x, y, z, config.brick_log2, config.prepass_stride,
            1 if config.entropy else 0, label_width or width, s.cuda_stream, ctypes.byref(h)))
    return GpuEncoded(h, d_volume.device)


def compress_volume(volume: np.ndarray, config: CompressionConfig | None = None,
                    width: int | None = None) -> CsvContainer:
    """Compress a (z, y, x) label volume into an in-memory container (container.py:374-453), on the GPU."""
    torch = _lib.require_cuda()
    config = config or CompressionConfig()
    vol, w = _check_volume(volume)
    if width is None:
        width = w
    t = torch.from_numpy(vol.view(np.int16 if w == 16 else np.int32)).cuda()
    enc = compress_volume_device(t, config, width=w, label_width=width)
    try:
        return enc.to_container()
    finally:
        enc.close()


def synth_voronoi(dims, cells_per_axis: int, seed: int = 0, membrane: bool = True, drift: float = 0.0,
                  drift_seed: int = 0, device=None, out=None):
    """(Z, Y, X) int32 CUDA tensor of jittered-grid Voronoi labels (see csv_synth_voronoi)."""
    torch = _lib.require_cuda()
    x, y, z = dims
    if out is None:
        out = torch.empty((z, y, x), dtype=torch.int32, device=device or "cuda")
    with torch.cuda.device(out.device):
        _lib.check(_lib.lib().csv_synth_voronoi(out.data_ptr(), x, y, z, cells_per_axis, seed & 0xFFFFFFFF,
                                                1 if membrane else 0, float(drift), drift_seed & 0xFFFFFFFF,
                                                torch.cuda.current_stream().cuda_stream))
    return out
