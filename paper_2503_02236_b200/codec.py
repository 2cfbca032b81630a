"""Quantized-tensor containers of the drop-in API, plus GPU dequantization.

Same public surface and semantics as vqforge.codec (pkg/src/vqforge/codec.py):

* :class:`Sharing`          codec.py:23-57   codebook-sharing granularity
* :class:`VQConfig`         codec.py:60-96   <vector_size, log2(entries), residuals> + sharing
* :class:`Codebook`         codec.py:104-123 one (2^b, v) fp32 entry table per (region, level)
* :func:`region_layout`     codec.py:135-177 region id of every sub-vector
* :class:`QuantizedTensor`  codec.py:180-226 codes (R, S) level-major + level-major books
* :func:`dequantize`        codec.py:391-408 — here executed by the CUDA kernel
  ``vqb_dequant`` (bit-exact fp32), never on the CPU.

Codebook *training* / nearest-centroid quantization (codec.py:239-388) is offline
CPU work and out of scope; quantized tensors come from
the reference, from a VQLF container, or from synthetic generators.
"""

from dataclasses import dataclass, field

import numpy as np

from . import bitpack
from .errors import ConfigError, ShapeError

VALID_VECTOR_SIZES = (2, 4, 8, 16)
SHARING_KINDS = ("whole", "tile", "channel_group")


@dataclass(frozen=True)
class Sharing:
    """How codebooks are shared over a tensor.

    ``whole``: one region. ``tile``: one region per (tile_rows x tile_cols) tile of
    the last two axes, partial edge tiles allowed, shared over leading axes.
    ``channel_group``: one region per ``group_width`` trailing channels, and per
    head on 4-D (B, H, T, C) tensors.
    """

    kind: str
    tile_rows: int = 0
    tile_cols: int = 0
    group_width: int = 0

    def __post_init__(self):
        if self.kind not in SHARING_KINDS:
            raise ConfigError(f"unknown sharing granularity {self.kind!r}")
        if self.kind == "tile" and min(self.tile_rows, self.tile_cols) <= 0:
            raise ConfigError("tile sharing needs positive tile_rows/tile_cols")
        if self.kind == "channel_group" and self.group_width <= 0:
            raise ConfigError("channel_group sharing needs positive group_width")

    @classmethod
    def whole_tensor(cls) -> "Sharing":
        return cls("whole")

    @classmethod
    def per_tile(cls, rows: int, cols: int) -> "Sharing":
        return cls("tile", tile_rows=rows, tile_cols=cols)

    @classmethod
    def per_channel_group(cls, width: int) -> "Sharing":
        return cls("channel_group", group_width=width)


@dataclass(frozen=True)
class VQConfig:
    """VQ<vector_size, log2_entries, residuals> plus the sharing granularity."""

    vector_size: int
    log2_entries: int
    residuals: int
    sharing: Sharing = field(default_factory=Sharing.whole_tensor)

    def __post_init__(self):
        if self.vector_size not in VALID_VECTOR_SIZES:
            raise ConfigError(
                f"vector_size must be one of {VALID_VECTOR_SIZES}, got {self.vector_size}")
        if not 1 <= self.log2_entries <= 16:
            raise ConfigError(f"log2_entries must be in [1, 16], got {self.log2_entries}")
        if self.residuals < 1:
            raise ConfigError(f"residuals must be >= 1, got {self.residuals}")
        sh = self.sharing
        if sh.kind == "channel_group" and sh.group_width % self.vector_size:
            raise ConfigError("group_width must be a multiple of vector_size")
        if sh.kind == "tile" and sh.tile_cols % self.vector_size:
            raise ConfigError("tile_cols must be a multiple of vector_size")

    @property
    def n_entries(self) -> int:
        return 2 ** self.log2_entries

    @property
    def bits_per_element(self) -> float:
        return self.residuals * self.log2_entries / self.vector_size

    @property
    def entry_bytes(self) -> int:
        """Footprint of one entry at fp16 (2 bytes / element), as the paper models it."""
        return 2 * self.vector_size


def compression_ratio(config: VQConfig) -> float:
    """Compressed bits over fp16 bits (codec.py:99-101)."""
    return config.residuals * config.log2_entries / (16 * config.vector_size)


@dataclass
class Codebook:
    """Entries (n_entries, vector_size) fp32 of one (region, residual level)."""

    entries: np.ndarray
    residual_level: int
    region_id: int

    def __post_init__(self):
        self.entries = np.ascontiguousarray(self.entries, dtype=np.float32)
        if self.entries.ndim != 2:
            raise ShapeError("codebook entries must be a 2-D matrix")

    @property
    def n_entries(self) -> int:
        return int(self.entries.shape[0])

    @property
    def vector_size(self) -> int:
        return int(self.entries.shape[1])


def _check_last_axis(shape, v: int) -> None:
    if shape[-1] % v:
        raise ShapeError(f"last axis {shape[-1]} not divisible by vector_size {v}")


def subvector_count(shape, config: VQConfig) -> int:
    shape = tuple(int(s) for s in shape)
    _check_last_axis(shape, config.vector_size)
    return int(np.prod(shape, dtype=np.int64)) // config.vector_size


def region_count(shape, config: VQConfig) -> int:
    """Regions per residual level, without materialising per-sub-vector ids."""
    shape = tuple(int(s) for s in shape)
    _check_last_axis(shape, config.vector_size)
    sh = config.sharing
    cols = shape[-1]
    if sh.kind == "whole":
        return 1
    if sh.kind == "channel_group":
        if cols % sh.group_width:
            raise ShapeError(f"last axis {cols} not divisible by group_width {sh.group_width}")
        groups = cols // sh.group_width
        return groups * shape[1] if len(shape) == 4 else groups
    if len(shape) < 2:
        raise ShapeError("tile sharing requires at least 2-D tensors")
    return -(-shape[-2] // sh.tile_rows) * -(-cols // sh.tile_cols)


def region_layout(shape, config: VQConfig):
    """(n_regions, int32 region id per sub-vector in row-major sub-vector order)."""
    shape = tuple(int(s) for s in shape)
    n_regions = region_count(shape, config)
    v = config.vector_size
    cols = shape[-1]
    per_row = cols // v
    n_rows = int(np.prod(shape[:-1], dtype=np.int64)) if len(shape) > 1 else 1
    sh = config.sharing
    if sh.kind == "whole":
        return n_regions, np.zeros(n_rows * per_row, dtype=np.int32)
    col0 = np.arange(per_row, dtype=np.int64) * v          # first column of each sub-vector
    rows = np.arange(n_rows, dtype=np.int64)
    if sh.kind == "channel_group":
        grp = col0 // sh.group_width
        if len(shape) == 4:
            heads = (rows // shape[2]) % shape[1]
            ids = heads[:, None] * (cols // sh.group_width) + grp[None, :]
        else:
            ids = np.broadcast_to(grp[None, :], (n_rows, per_row))
        return n_regions, np.ascontiguousarray(ids, dtype=np.int32).reshape(-1)
    n_tile_cols = -(-cols // sh.tile_cols)
    local = rows % shape[-2]
    ids = (local // sh.tile_rows)[:, None] * n_tile_cols + (col0 // sh.tile_cols)[None, :]
    return n_regions, np.ascontiguousarray(ids, dtype=np.int32).reshape(-1)


@dataclass
class QuantizedTensor:
    """Codes (R, S) int32 level-major plus R * n_regions level-major codebooks.

    ``codebooks[level * n_regions + region]`` serves (level, region), exactly as in
    the reference (codec.py:208-209).
    """

    codes: np.ndarray
    shape: tuple
    config: VQConfig
    codebooks: list
    n_regions: int

    def __post_init__(self):
        self.codes = np.ascontiguousarray(self.codes, dtype=np.int32)
        self.shape = tuple(int(s) for s in self.shape)
        want = (self.config.residuals, subvector_count(self.shape, self.config))
        if self.codes.shape != want:
            raise ShapeError(f"codes shape {self.codes.shape} != {want}")
        n_books = self.config.residuals * self.n_regions
        if len(self.codebooks) != n_books:
            raise ShapeError(f"expected {n_books} codebooks, got {len(self.codebooks)}")

    def codebook_for(self, level: int, region: int) -> Codebook:
        return self.codebooks[level * self.n_regions + region]

    @property
    def total_codes(self) -> int:
        return int(self.codes.size)

    @property
    def packed_bit_length(self) -> int:
        return self.total_codes * self.config.log2_entries

    def packed_codes(self) -> bytes:
        """The level-major LSB-first stream (byte padded at the end only)."""
        return bitpack.pack_indices(self.codes, self.config.log2_entries)

    @property
    def region_ids(self) -> np.ndarray:
        return region_layout(self.shape, self.config)[1]

    def stacked_entries(self) -> np.ndarray:
        """All books as one (R * n_regions, K, v) fp32 array (device upload order)."""
        return np.stack([cb.entries for cb in self.codebooks])


def split_subvectors(data, config: VQConfig) -> np.ndarray:
    """(n_subvectors, vector_size) fp32 view of ``data`` (codec.py:229-236)."""
    arr = np.ascontiguousarray(data, dtype=np.float32)
    _check_last_axis(arr.shape, config.vector_size)
    return arr.reshape(-1, config.vector_size)


def dequantize(q, device=None, out_dtype=None):
    """Reconstruct the dense tensor on the GPU (``vqb_dequant``).

    ``q`` is a host :class:`QuantizedTensor` (returns a float32 ndarray bit-identical
    to vqforge.codec.dequantize) or a :class:`~.device.DeviceVQTensor` (returns a
    device tensor of ``out_dtype``, default float32).
    """
    from .device import DeviceVQTensor
    from .ops import vq_dequantize

    if isinstance(q, DeviceVQTensor):
        return vq_dequantize(q, out_dtype=out_dtype)
    dq = DeviceVQTensor.from_quantized(q, device=device, codebook_dtype="float32", layout="plain")
    out = vq_dequantize(dq, out_dtype=out_dtype)
    return out.cpu().numpy() if out_dtype is None else out
