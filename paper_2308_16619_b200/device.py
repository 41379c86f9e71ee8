"""Device-resident volumes: the Python side of the C-ABI decode path.

`GpuVolume` owns one `csv_volume` handle (include/csvgpu.h): the container's
directory, palette/coarse/detail blobs and decode tables uploaded to HBM,
plus the decode workspace.  PyTorch provides device buffers and streams only;
all decode work runs in libcsvgpu.so's sm_100a kernels.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import CorruptStreamError

ERROR_TEXT = {   # codec.py:487-495
    1: "stream underrun",
    2: "invalid opcode 7",
    3: "palette index out of range",
    4: "palette back-reference before palette start",
    5: "entropy stream desynchronized",
    6: "neighbor reference outside the brick",
    7: "stop bit set on a leaf-level entry",
}
STREAM_NAMES = ("coarse", "detail")
ST_EMPTY_PALETTE = 8


def status_error(status: int, stream: int, pos: int) -> Exception:
    """The exception the reference raises for one kernel status (codec.py:510-511, :540-543)."""
    if status == ST_EMPTY_PALETTE:
        return CorruptStreamError("empty palette")
    if status in ERROR_TEXT:
        return CorruptStreamError(f"{ERROR_TEXT[status]} ({STREAM_NAMES[stream]} stream, nibble {pos})")
    return RuntimeError(f"decoder returned invalid status {status}")


def _ptr(a) -> int:
    """Address of a numpy array / torch tensor / None."""
    if a is None:
        return 0
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def _check_buffer(name: str, t, device, itemsize: int, shape=None, min_numel: int = 0) -> None:
    """Refuse a caller buffer the kernels would index out of bounds: wrong device,
    element size, a non-contiguous layout, a shape other than ``shape`` or fewer
    than ``min_numel`` elements."""
    if t.device != device:
        raise ValueError(f"{name} is on {t.device}, the volume on {device}")
    if t.element_size() != itemsize or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous tensor of {itemsize}-byte elements")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    if t.numel() < min_numel:
        raise ValueError(f"{name} has {t.numel()} elements, needs at least {min_numel}")


def _stream_handle(torch, stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _on_stream(torch, device, stream):
    """Enter `device` and make `stream` torch's current stream, so that tensors allocated,
    uploaded or read back around a C-ABI call are ordered with the kernels it launches."""
    import contextlib
    st = contextlib.ExitStack()
    st.enter_context(torch.cuda.device(device))
    if stream is not None:
        st.enter_context(torch.cuda.stream(stream))
    return st


class GpuVolume:
    """One container (or a brick range of it) resident on a CUDA device.

    ``head120`` is the 120-byte CSV1 head, ``directory`` the structured
    44-byte directory rows of bricks [brick_begin, brick_end), and the blobs
    are numpy arrays (host upload) or torch CUDA tensors (borrowed, with
    >=64 readable bytes past their end) starting at the given global bases.
    """

    def __init__(self, head120: bytes, directory: np.ndarray, palette, coarse, detail,
                 brick_begin: int = 0, brick_end: int | None = None,
                 palette_base: int = 0, coarse_base: int = 0, detail_base: int = 0,
                 device=None, stream=None, on_device: bool = False, deferred: bool = False):
        torch = _lib.require_cuda()
        self._torch = torch
        L = _lib.lib()
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else
                                   torch.device(device).index or 0)
        if brick_end is None:
            if on_device:
                raise ValueError("device-resident volumes need an explicit brick_end")
            brick_end = brick_begin + directory.shape[0]
        self.brick_begin, self.brick_end = int(brick_begin), int(brick_end)
        self._keep = (head120, directory, palette, coarse, detail)   # borrowed/host buffers stay alive
        head = np.frombuffer(bytes(head120[:120]), dtype=np.uint8).copy()
        self._head = head
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            sh = _stream_handle(torch, stream)
            if on_device:
                # device blobs: either tensors or raw (ptr, count) pairs; borrowed, not copied
                def pc(x):
                    return (x[0], x[1]) if isinstance(x, tuple) else (_ptr(x), x.numel())
                dp, _ = pc(directory) if isinstance(directory, tuple) else (_ptr(directory), 0)
                pp, pn = pc(palette)
                cp, cn = pc(coarse)
                xp, xn = pc(detail)
                rc = L.csv_volume_create_device(
                    self.device.index, _ptr(head), dp, self.brick_begin, self.brick_end,
                    pp, palette_base, pn, cp, coarse_base, cn, xp, detail_base, xn, sh, ctypes.byref(handle))
                self.palette_entries = int(pn)
            elif deferred:
                # blobs allocated now, filled by upload(); palette/coarse/detail are their lengths
                d = np.ascontiguousarray(directory).view(np.uint8)
                self._keep = (head120, d)
                rc = L.csv_volume_create_deferred(
                    self.device.index, _ptr(head), _ptr(d), self.brick_begin, self.brick_end,
                    palette_base, int(palette), coarse_base, int(coarse), detail_base, int(detail), sh,
                    ctypes.byref(handle))
                self.palette_entries = int(palette)
            else:
                d = np.ascontiguousarray(directory).view(np.uint8)
                pal = np.ascontiguousarray(palette, dtype="<u4")
                cb = np.ascontiguousarray(coarse, dtype=np.uint8)
                db = np.ascontiguousarray(detail, dtype=np.uint8) if detail is not None else np.zeros(0, np.uint8)
                self._keep = (head120, d, pal, cb, db)
                rc = L.csv_volume_create(
                    self.device.index, _ptr(head), _ptr(d), self.brick_begin, self.brick_end,
                    _ptr(pal), palette_base, pal.size, _ptr(cb), coarse_base, cb.size,
                    _ptr(db), detail_base, db.size, sh, ctypes.byref(handle))
                self.palette_entries = int(pal.size)
            _lib.check(rc)
        self._h = handle
        dims = (ctypes.c_int64 * 3)()
        grid = (ctypes.c_int64 * 3)()
        bl2 = ctypes.c_int()
        ent = ctypes.c_int()
        _lib.check(L.csv_volume_info(self._h, dims, grid, ctypes.byref(bl2), ctypes.byref(ent)))
        self.dims = tuple(dims)          # (x, y, z)
        self.grid = tuple(grid)
        self.brick_log2 = bl2.value
        self.entropy = bool(ent.value)

    # ------------------------------------------------------------------ lifetime
    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().csv_volume_free(self._h)
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
    def n_bricks(self) -> int:
        return self.brick_end - self.brick_begin

    def crop(self, t: int) -> tuple[int, int, int]:
        """(z, y, x) extent of the volume at LOD t (container.py:476-478)."""
        x, y, z = self.dims
        return tuple(-(-d // (1 << t)) for d in (z, y, x))

    def slab(self, t: int) -> tuple[int, int]:
        """LOD-t z rows covered by this volume's bricks (whole bz layers assumed)."""
        gx, gy, _ = self.grid
        side = (1 << self.brick_log2) >> t
        z0 = (self.brick_begin // (gx * gy)) * side
        z1 = min(-(-self.brick_end // (gx * gy)) * side, self.crop(t)[0])
        return z0, z1

    # ------------------------------------------------------------------ decode
    def decode(self, t: int = 0, out=None, z_range=None, results=None, stream=None):
        """Raster decode (K1 + K2/K3) into a (z1-z0, cy, cx) uint32 CUDA tensor."""
        torch = self._torch
        if not 0 <= t <= self.brick_log2:
            raise ValueError(f"LOD {t} outside [0, {self.brick_log2}]")
        z0, z1 = z_range if z_range is not None else self.slab(t)
        _, cy, cx = self.crop(t)
        with _on_stream(torch, self.device, stream):
            if out is None:
                out = torch.empty((max(z1 - z0, 0), cy, cx), dtype=torch.int32, device=self.device)
            if results is None:
                results = torch.empty((max(self.n_bricks, 1), 4), dtype=torch.int64, device=self.device)
            _check_buffer("out", out, self.device, 4, shape=(max(z1 - z0, 0), cy, cx))
            _check_buffer("results", results, self.device, 8, min_numel=4 * self.n_bricks)
            _lib.check(_lib.lib().csv_decode_volume(self._h, t, _ptr(out), z0, z1, _ptr(results),
                                                    _stream_handle(torch, stream)))
        return out, results

    def decode_into(self, t: int, out_ptr: int, z_range, results, stream=None) -> None:
        """Raster decode into raw device memory (z_range rows of the cropped volume at
        out_ptr, row pitch cx): the peer-memory gather writes through pointers into
        another rank's volume, which no local tensor describes."""
        torch = self._torch
        if not 0 <= t <= self.brick_log2:
            raise ValueError(f"LOD {t} outside [0, {self.brick_log2}]")
        _check_buffer("results", results, self.device, 8, min_numel=4 * self.n_bricks)
        with _on_stream(torch, self.device, stream):
            _lib.check(_lib.lib().csv_decode_volume(self._h, t, int(out_ptr), z_range[0], z_range[1], _ptr(results),
                                                    _stream_handle(torch, stream)))

    def upload(self, blob: int, host: np.ndarray, offset: int, stream=None) -> None:
        """Fill bytes [offset, offset + host.nbytes) of blob 0 palette / 1 coarse / 2 detail (deferred volumes)."""
        torch = self._torch
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().csv_volume_upload(self._h, blob, _ptr(host), offset, host.nbytes,
                                                    _stream_handle(torch, stream)))

    def decode_range(self, t: int, brick_first: int, brick_last: int, out, z_range, results, stream=None):
        """Raster decode of bricks [brick_first, brick_last) into the z-slab `out` (rows z_range)."""
        torch = self._torch
        _, cy, cx = self.crop(t)
        _check_buffer("out", out, self.device, 4, min_numel=max(z_range[1] - z_range[0], 0) * cy * cx)
        if out.dim() != 3 or tuple(out.shape[1:]) != (cy, cx):
            raise ValueError(f"out has shape {tuple(out.shape)}, expected (>= {z_range[1] - z_range[0]}, {cy}, {cx})")
        _check_buffer("results", results, self.device, 8, min_numel=4 * max(brick_last - brick_first, 0))
        with _on_stream(torch, self.device, stream):
            _lib.check(_lib.lib().csv_decode_volume_range(self._h, t, brick_first, brick_last, _ptr(out),
                                                          z_range[0], z_range[1], _ptr(results),
                                                          _stream_handle(torch, stream)))
        return out

    def decode_bricks(self, bricks, lods, dst, pool, results=None, stream=None):
        """Batched Morton decode (K1 + K2/K4) of (brick, lod) requests into pool[dst:...]."""
        torch = self._torch
        n = int(bricks.numel())
        with _on_stream(torch, self.device, stream):
            if results is None:
                results = torch.empty((max(n, 1), 4), dtype=torch.int64, device=self.device)
            for name, buf, size in (("lods", lods, 1), ("dst", dst, 8)):
                _check_buffer(name, buf, self.device, size, min_numel=n)
            _check_buffer("bricks", bricks, self.device, 4)
            _check_buffer("pool", pool, self.device, 4)
            _check_buffer("results", results, self.device, 8, min_numel=4 * n)
            _lib.check(_lib.lib().csv_decode_bricks(self._h, n, _ptr(bricks), _ptr(lods), _ptr(dst), _ptr(pool),
                                                    _ptr(results), _stream_handle(torch, stream)))
        return results

    def decode_streams(self, bricks, t: int, stream=None):
        """K1 alone: (entries u8 tensor, offsets [2n+1], per-stream results [2n] structured)."""
        torch = self._torch
        L = _lib.lib()
        n = int(bricks.numel())
        cap = ctypes.c_uint64()
        _lib.check(L.csv_streams_capacity(self._h, n, t, ctypes.byref(cap)))
        entries = torch.zeros(max(int(cap.value), 16), dtype=torch.uint8, device=self.device)
        offs = torch.zeros(2 * n + 1, dtype=torch.int64, device=self.device)
        sres = torch.zeros((max(2 * n, 1), 4), dtype=torch.int32, device=self.device)
        with torch.cuda.device(self.device):
            _lib.check(L.csv_decode_streams(self._h, n, _ptr(bricks), t, _ptr(entries), entries.numel(),
                                            _ptr(offs), _ptr(sres), _stream_handle(torch, stream)))
        return entries, offs, sres

    def op_counts(self, stream=None):
        """K1 in count mode: (per-op totals int64[8], per-stream results [2n] structured)."""
        torch = self._torch
        n = self.n_bricks
        counts = torch.zeros(8, dtype=torch.int64, device=self.device)
        sres = torch.zeros((max(2 * n, 1), 4), dtype=torch.int32, device=self.device)
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().csv_volume_op_counts(self._h, _ptr(counts), _ptr(sres), _stream_handle(torch, stream)))
        return counts.cpu().numpy(), sres[: 2 * n].cpu().numpy().view(_lib.STREAM_RESULT_DTYPE).reshape(2 * n)

    def set_timing(self, enable: bool = True) -> None:
        _lib.check(_lib.lib().csv_volume_set_timing(self._h, 1 if enable else 0))

    def last_timing(self) -> tuple[float, float, float]:
        """(plan, K1, K2) milliseconds of the last decode call (CUDA events on its stream)."""
        ms = (ctypes.c_float * 3)()
        _lib.check(_lib.lib().csv_volume_get_timing(self._h, ms))
        return tuple(ms)

    # ------------------------------------------------------------------ results
    @staticmethod
    def results_host(results, n: int) -> np.ndarray:
        arr = results[:n].contiguous().cpu().numpy()
        return arr.view(_lib.RESULT_DTYPE).reshape(n)

    @staticmethod
    def raise_first(results, n: int) -> None:
        """Raise the reference's exception for the lowest failing index, if any."""
        if n == 0:
            return
        status = results[:n, 0].view(results.dtype)  # low 32 bits hold status (little-endian)
        st32 = (status & 0xFFFFFFFF)
        bad = st32.nonzero()
        if bad.numel() == 0:
            return
        i = int(bad[0, 0])
        row = results[i].cpu().numpy().view(_lib.RESULT_DTYPE)[0]
        raise status_error(int(row["status"]), int(row["stream"]), int(row["pos"]))
