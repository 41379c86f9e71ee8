"""ctypes binding of libcsvgpu.so (C-ABI declared in include/csvgpu.h).

There is no CPU fallback: if the shared library is missing or no CUDA device
is visible, every decode entry point raises ``RuntimeError`` loudly.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CSVGPU_LIB") or os.path.join(_PKG, "libcsvgpu.so")   # override: build variants
_lib = None

# C-ABI return codes (include/csvgpu.h)
CSV_E_ARG, CSV_E_CUDA, CSV_E_NOMEM, CSV_E_FORMAT, CSV_E_CAPACITY = -1, -2, -3, -4, -5

RESULT_DTYPE = np.dtype([("status", "<i4"), ("stream", "<i4"), ("pos", "<i8"), ("ci", "<i8"), ("di", "<i8")])
STREAM_RESULT_DTYPE = np.dtype([("n_entries", "<u4"), ("fail_nibble", "<u4"), ("flags", "<u4"), ("partial_op", "<u4")])

EXPORTS = (
    "csv_version", "csv_last_error", "csv_volume_create", "csv_volume_create_device", "csv_volume_free",
    "csv_decode_volume", "csv_decode_bricks", "csv_decode_streams", "csv_streams_capacity", "csv_volume_info",
    "csv_encode_volume", "csv_encoded_info", "csv_encoded_device_ptrs", "csv_encoded_copy_to_host",
    "csv_encoded_free", "csv_synth_voronoi", "csv_volume_set_timing", "csv_volume_get_timing",
    "csv_volume_op_counts", "csv_decode_volume_range", "csv_volume_create_deferred", "csv_volume_upload",
    "csv_desired_lods", "csv_visibility_mask", "csv_cache_create", "csv_cache_free", "csv_cache_begin_frame",
    "csv_cache_mark_used", "csv_cache_assign", "csv_cache_state", "csv_cache_counters", "csv_cache_stack_heights",
    "csv_cache_read_state", "csv_cache_plan", "csv_cache_decode_fills", "csv_volume_stage_detail",
    "csv_cache_read_fills", "csv_detail_plan_greedy", "csv_rans_decode", "csv_rans_encode", "csv_build_pyramid",
    "csv_downsample", "csv_decode_bricks_host", "csv_decode_brick_streams", "csv_peer_alloc", "csv_peer_free", "csv_peer_open", "csv_peer_close",
)


def build(force: bool = False) -> str:
    """Compile the CUDA sources for sm_100a into the package directory."""
    csrc = os.path.join(_PKG, "csrc")
    srcs = [os.path.join(csrc, f) for f in os.listdir(csrc) if f.endswith((".cu", ".cuh"))]
    srcs.append(os.path.join(os.path.dirname(_PKG), "include", "csvgpu.h"))
    newest = max(os.path.getmtime(s) for s in srcs)
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < newest:
        subprocess.run(["make", "-s", "-C", csrc], check=True)
    return LIB_PATH


def lib():
    """Load libcsvgpu.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        P, U64, I64, I, UP = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
        L.csv_version.restype = I
        L.csv_last_error.restype = ctypes.c_char_p
        L.csv_volume_create.restype = I
        L.csv_volume_create.argtypes = [I, P, P, U64, U64, P, U64, U64, P, U64, U64, P, U64, U64, UP, P]
        L.csv_volume_create_device.restype = I
        L.csv_volume_create_device.argtypes = [I, P, P, U64, U64, P, U64, U64, P, U64, U64, P, U64, U64, UP, P]
        L.csv_volume_free.restype = I
        L.csv_volume_free.argtypes = [P]
        L.csv_decode_volume.restype = I
        L.csv_decode_volume.argtypes = [P, I, P, I64, I64, P, UP]
        L.csv_decode_bricks.restype = I
        L.csv_decode_bricks.argtypes = [P, U64, P, P, P, P, P, UP]
        L.csv_decode_streams.restype = I
        L.csv_decode_streams.argtypes = [P, U64, P, I, P, U64, P, P, UP]
        L.csv_streams_capacity.restype = I
        L.csv_streams_capacity.argtypes = [P, U64, I, P]
        L.csv_volume_info.restype = I
        L.csv_volume_info.argtypes = [P, P, P, P, P]
        L.csv_encode_volume.restype = I
        L.csv_encode_volume.argtypes = [I, P, I, I64, I64, I64, I, I64, I, I, UP, P]
        L.csv_encoded_info.restype = I
        L.csv_encoded_info.argtypes = [P, P, P, P]
        L.csv_encoded_device_ptrs.restype = I
        L.csv_encoded_device_ptrs.argtypes = [P, P, P, P, P]
        L.csv_encoded_copy_to_host.restype = I
        L.csv_encoded_copy_to_host.argtypes = [P, P, P, P, P, UP]
        L.csv_encoded_free.restype = I
        L.csv_encoded_free.argtypes = [P]
        L.csv_synth_voronoi.restype = I
        L.csv_synth_voronoi.argtypes = [P, I64, I64, I64, I, ctypes.c_uint32, I, ctypes.c_double, ctypes.c_uint32, UP]
        L.csv_volume_create_deferred.restype = I
        L.csv_volume_create_deferred.argtypes = [I, P, P, U64, U64, U64, U64, U64, U64, U64, U64, UP, P]
        L.csv_volume_upload.restype = I
        L.csv_volume_upload.argtypes = [P, I, P, U64, U64, UP]
        L.csv_decode_volume_range.restype = I
        L.csv_decode_volume_range.argtypes = [P, I, U64, U64, P, I64, I64, P, UP]
        L.csv_volume_op_counts.restype = I
        L.csv_volume_op_counts.argtypes = [P, P, P, UP]
        L.csv_volume_set_timing.restype = I
        L.csv_volume_set_timing.argtypes = [P, I]
        L.csv_volume_get_timing.restype = I
        L.csv_volume_get_timing.argtypes = [P, P]
        D = ctypes.c_double
        L.csv_desired_lods.restype = I
        L.csv_desired_lods.argtypes = [P, D, D, D, D, D, P, UP]
        L.csv_visibility_mask.restype = I
        L.csv_visibility_mask.argtypes = [P, U64, P, P, ctypes.c_uint32, D, P, UP]
        L.csv_cache_create.restype = I
        L.csv_cache_create.argtypes = [I, U64, I, U64, P]
        L.csv_cache_free.restype = I
        L.csv_cache_free.argtypes = [P]
        L.csv_cache_begin_frame.restype = I
        L.csv_cache_begin_frame.argtypes = [P, UP]
        L.csv_cache_mark_used.restype = I
        L.csv_cache_mark_used.argtypes = [P, P, P, U64, UP]
        L.csv_cache_assign.restype = I
        L.csv_cache_assign.argtypes = [P, P, P, P, U64, P, P, P, P, UP]
        L.csv_cache_state.restype = I
        L.csv_cache_state.argtypes = [P, P, P, P, P, P, P]
        L.csv_cache_plan.restype = I
        L.csv_cache_plan.argtypes = [P, P, P, U64, P, P, UP]
        L.csv_cache_decode_fills.restype = I
        L.csv_cache_decode_fills.argtypes = [P, P, P, P, UP]
        L.csv_volume_stage_detail.restype = I
        L.csv_volume_stage_detail.argtypes = [P, P, P, P, U64, P, U64, UP]
        L.csv_cache_read_fills.restype = I
        L.csv_cache_read_fills.argtypes = [P, P, P, U64, P]
        L.csv_detail_plan_greedy.restype = I
        L.csv_detail_plan_greedy.argtypes = [P, U64, U64, P, P]
        L.csv_cache_read_state.restype = I
        L.csv_cache_read_state.argtypes = [P, P, P]
        L.csv_cache_counters.restype = I
        L.csv_cache_counters.argtypes = [P, P]
        L.csv_cache_stack_heights.restype = I
        L.csv_cache_stack_heights.argtypes = [P, P]
        L.csv_rans_decode.restype = I
        L.csv_rans_decode.argtypes = [P, P, P, P, U64, P, P, P, P, UP]
        L.csv_rans_encode.restype = I
        L.csv_rans_encode.argtypes = [P, P, P, U64, P, P, P, P, UP]
        L.csv_build_pyramid.restype = I
        L.csv_build_pyramid.argtypes = [P, U64, I, P, P, UP]
        L.csv_peer_alloc.restype = I
        L.csv_peer_alloc.argtypes = [I, U64, P, P]
        L.csv_peer_free.restype = I
        L.csv_peer_free.argtypes = [I, P]
        L.csv_peer_open.restype = I
        L.csv_peer_open.argtypes = [I, P, P]
        L.csv_peer_close.restype = I
        L.csv_peer_close.argtypes = [I, P]
        L.csv_decode_bricks_host.restype = I
        L.csv_decode_bricks_host.argtypes = [P, U64, P, P, P, P, UP]
        L.csv_decode_brick_streams.restype = I
        L.csv_decode_brick_streams.argtypes = [I, P, P, U64, P, U64, ctypes.c_uint32, P, U64, ctypes.c_uint32, I, P, P, UP]
        L.csv_downsample.restype = I
        L.csv_downsample.argtypes = [P, I64, I64, I64, P, UP]
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().csv_last_error().decode(errors="replace")
        raise RuntimeError(f"libcsvgpu error {rc}: {msg}")


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2308_16619_b200 decodes on a CUDA device; none is visible (no CPU fallback)")
    return torch
