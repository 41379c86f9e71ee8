"""B200-native decoder for CSV compressed segmentation volumes (arXiv 2308.16619).

Drop-in for the reference ``csvol`` decode/brick-access API: same names,
argument meaning and errors; the per-brick decompression (rANS entropy
decode + coarse-to-fine operation replay) runs in hand-written sm_100a CUDA
kernels (csrc/) reached through the C-ABI in include/csvgpu.h.
"""

from .cache import BrickCache, CacheStats, DeviceBrickCache
from .codec import BrickEncoding, decode_brick, decode_brick_entropy, decode_root, encode_brick, iter_operations
from .container import (CompressionConfig, CsvContainer, VolumeMeta, decompress_volume,
                        decompress_volume_device, stats)
from .detail import DetailStore, DeviceDetailStream
from .device import GpuVolume
from .frame import Camera, TransferFunction, desired_lods, desired_lods_device, visibility_mask, visibility_mask_device
from .encode import GpuEncoded, compress_volume, compress_volume_device, synth_voronoi
from .errors import (CacheCapacityError, ConfigError, CorruptStreamError, CsvolError, EncodabilityError,
                     IngestionError)
from .morton import BrickConfig, NodeCoord, morton_decode, morton_encode, outside_neighbor
from .pyramid import Pyramid, build_pyramid, downsample_level, downsample_volume, pyramid_from_grid
from .rans import FrequencyTable, TablePair, build_frequency_tables, quantize_counts, rans_decode, rans_encode

__version__ = "0.1.0"

__all__ = [
    "BrickCache", "BrickConfig", "DetailStore", "DeviceDetailStream", "Camera", "DeviceBrickCache", "TransferFunction", "desired_lods",
    "desired_lods_device", "visibility_mask", "visibility_mask_device", "BrickEncoding", "CacheCapacityError", "CacheStats", "CompressionConfig",
    "ConfigError", "CorruptStreamError", "CsvContainer", "CsvolError", "EncodabilityError", "FrequencyTable",
    "GpuEncoded", "GpuVolume", "compress_volume", "compress_volume_device", "synth_voronoi", "IngestionError", "NodeCoord", "TablePair", "VolumeMeta", "build_frequency_tables",
    "decode_brick", "decode_brick_entropy", "decode_root", "decompress_volume", "decompress_volume_device",
    "iter_operations", "stats", "morton_decode", "morton_encode", "outside_neighbor", "quantize_counts",
    "encode_brick", "Pyramid", "build_pyramid", "downsample_level", "downsample_volume", "pyramid_from_grid",
    "rans_decode", "rans_encode",
]
