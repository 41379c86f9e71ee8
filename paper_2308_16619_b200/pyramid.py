"""Per-brick resolution pyramid (csvol/pyramid.py), built on the GPU.

``build_pyramid`` folds a Morton-ordered brick level by level with the
reference's rule -- mode of the 8 children, ties to the first occurrence,
subtree-constant flag (pyramid.py:43-78) -- in ``csv_build_pyramid`` (one
thread per parent node, csrc/csv_rans.cu).  ``downsample_level`` applies the
same rule to a (z, y, x) grid (``csv_downsample``, pyramid.py:81-96).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .morton import BrickConfig, grid_to_morton, morton_to_grid


@dataclass
class Pyramid:
    """Resolution stack of one brick (pyramid.py:23-40): ``levels[l]`` holds the
    Morton-ordered labels of level l, ``constant[l]`` the subtree-is-constant flags."""

    config: BrickConfig
    levels: list
    constant: list

    def level_grid(self, level: int) -> np.ndarray:
        return morton_to_grid(self.levels[level], self.config.level_side(level))

    @property
    def root_label(self) -> int:
        return int(self.levels[-1][0])


def build_pyramids(bricks: np.ndarray, config: BrickConfig) -> list:
    """Pyramids of many Morton-ordered bricks at once: ``bricks`` is (n, 8**N)."""
    torch = _lib.require_cuda()
    N = config.brick_log2
    n_leaf = 8 ** N
    arr = np.ascontiguousarray(bricks, dtype=np.uint32).reshape(-1, n_leaf)
    n = arr.shape[0]
    total = (8 ** (N + 1) - 1) // 7
    dev = torch.device("cuda", torch.cuda.current_device())
    d_in = torch.from_numpy(arr.view(np.int32)).to(dev)
    d_lev = torch.empty((max(n, 1), total), dtype=torch.int32, device=dev)
    d_const = torch.empty((max(n, 1), total), dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().csv_build_pyramid(d_in.data_ptr(), n, N, d_lev.data_ptr(), d_const.data_ptr(),
                                                torch.cuda.current_stream(dev).cuda_stream))
    lev = d_lev[:n].cpu().numpy().view(np.uint32)
    cst = d_const[:n].cpu().numpy().astype(bool)
    out = []
    for b in range(n):
        levels, constant, off = [], [], 0
        for l in range(N + 1):
            size = 8 ** (N - l)
            levels.append(lev[b, off: off + size].copy())
            constant.append(cst[b, off: off + size].copy())
            off += size
        out.append(Pyramid(config, levels, constant))
    return out


def build_pyramid(brick_labels: np.ndarray, config: BrickConfig) -> Pyramid:
    """Build the full resolution stack for one Morton-ordered brick (pyramid.py:65-78)."""
    n = config.side ** 3
    if brick_labels.shape != (n,):
        raise ValueError(f"brick has {brick_labels.shape} entries, expected ({n},) for b={config.side}")
    return build_pyramids(brick_labels.reshape(1, n), config)[0]


def downsample_level(child_grid: np.ndarray) -> np.ndarray:
    """Halve a (z, y, x) label grid with the mode-with-tie rule (pyramid.py:81-96)."""
    torch = _lib.require_cuda()
    nz, ny, nx = child_grid.shape
    if nz % 2 or ny % 2 or nx % 2:
        raise ValueError(f"grid sides must be even, got {child_grid.shape}")
    dev = torch.device("cuda", torch.cuda.current_device())
    src = np.ascontiguousarray(child_grid).astype(np.uint32, copy=False)
    d_in = torch.from_numpy(src.view(np.int32)).to(dev)
    d_out = torch.empty((nz // 2, ny // 2, nx // 2), dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().csv_downsample(d_in.data_ptr(), nz, ny, nx, d_out.data_ptr(),
                                             torch.cuda.current_stream(dev).cuda_stream))
    return d_out.cpu().numpy().view(np.uint32).astype(child_grid.dtype, copy=False)


def downsample_volume(volume: np.ndarray, steps: int) -> np.ndarray:
    """Apply :func:`downsample_level` ``steps`` times (pyramid.py:99-104)."""
    out = volume
    for _ in range(steps):
        out = downsample_level(out)
    return out


def pyramid_from_grid(brick_grid: np.ndarray, config: BrickConfig) -> Pyramid:
    """Convenience wrapper taking a (z, y, x) brick cube (pyramid.py:107-109)."""
    return build_pyramid(grid_to_morton(brick_grid), config)
