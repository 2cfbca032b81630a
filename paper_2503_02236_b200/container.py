"""VQLF container I/O with device ingest (vqforge.container, pkg/src/vqforge/container.py:25-94).

The byte format is the reference's: magic "VQLF", version u16, the config block
(vector_size, log2_entries, residuals u16; sharing kind u8 + tile_rows, tile_cols,
group_width u32), ndim u8 + dims u64, n_regions and n_books u32, per book
(level u16, region u32, float32 entries), then the packed code stream (bit length
u64 + LSB-first bytes, V/bitpack.py:13-28).

``load_vqlf`` parses the small header on the host and ships the packed stream to the
GPU untouched; the bit unpacking and the interleave into the kernels' layout happen
on the device (``vqb_repack``), so a checkpoint never takes the host unpack path the
reference uses (V/container.py:88-89). ``dump_vqlf`` writes the identical bytes as
the reference's ``dump_quantized`` for a host ``QuantizedTensor``.
"""

import struct

import numpy as np

from .codec import QuantizedTensor, Sharing, VQConfig
from .errors import ConfigError

MAGIC = b"VQLF"
VERSION = 1
_SHARING_KIND = {"whole": 0, "tile": 1, "channel_group": 2}
_SHARING_NAME = {v: k for k, v in _SHARING_KIND.items()}


def parse_header(data: bytes):
    """(config, shape, n_regions, books (n_books, K, v) float32, levels, regions,
    bit_length, stream offset) — V/container.py:52-86."""
    if data[:4] != MAGIC:
        raise ConfigError(f"bad magic {bytes(data[:4])!r}, expected {MAGIC!r}")
    off = 4
    (version,) = struct.unpack_from("<H", data, off)
    off += 2
    if version != VERSION:
        raise ConfigError(f"unsupported container version {version}")
    vec, log2e, res = struct.unpack_from("<HHH", data, off)
    off += 6
    kind, t_rows, t_cols, g_width = struct.unpack_from("<BxIII", data, off)
    off += 14
    if kind not in _SHARING_NAME:
        raise ConfigError(f"unknown sharing kind {kind}")
    sharing = Sharing(_SHARING_NAME[kind], tile_rows=t_rows, tile_cols=t_cols, group_width=g_width)
    cfg = VQConfig(vec, log2e, res, sharing)
    (ndim,) = struct.unpack_from("<B3x", data, off)
    off += 4
    shape = tuple(struct.unpack_from(f"<{ndim}Q", data, off))
    off += 8 * ndim
    n_regions, n_books = struct.unpack_from("<II", data, off)
    off += 8
    k = cfg.n_entries
    books = np.empty((n_books, k, vec), np.float32)
    levels, regions = np.empty(n_books, np.int64), np.empty(n_books, np.int64)
    for i in range(n_books):
        levels[i], regions[i] = struct.unpack_from("<HxxI", data, off)
        off += 8
        books[i] = np.frombuffer(data, dtype="<f4", count=k * vec, offset=off).reshape(k, vec)
        off += k * vec * 4
    (bit_length,) = struct.unpack_from("<Q", data, off)
    off += 8
    return cfg, shape, n_regions, books, levels, regions, bit_length, off


def load_vqlf(data: bytes, device=None, codebook_dtype="float16", layout: str = "auto"):
    """A DeviceVQTensor straight from VQLF bytes: books in the kernels' level-major
    (R * n_regions, K, v) order, codes unpacked and interleaved on the GPU."""
    from .device import DeviceVQTensor, auto_layout

    cfg, shape, n_regions, books, levels, regions, bit_length, off = parse_header(data)
    order = np.argsort(levels * n_regions + regions, kind="stable")
    if not np.array_equal(levels[order] * n_regions + regions[order], np.arange(len(order))):
        raise ConfigError("container codebooks do not cover (level, region) exactly once")
    n_codes = int(np.prod(shape)) // cfg.vector_size * cfg.residuals
    if bit_length != n_codes * cfg.log2_entries:
        raise ConfigError(f"packed stream holds {bit_length} bits, expected {n_codes * cfg.log2_entries}")
    stream = bytes(data[off:off + (bit_length + 7) // 8])
    if layout == "auto":
        layout = auto_layout(shape, cfg)
    return DeviceVQTensor.from_packed(stream, shape, cfg, books[order], device=device,
                                      codebook_dtype=codebook_dtype, layout=layout)


def dump_vqlf(q: QuantizedTensor) -> bytes:
    """The reference's byte layout (V/container.py:25-49) for a host QuantizedTensor."""
    cfg = q.config
    out = bytearray(MAGIC)
    out += struct.pack("<H", VERSION)
    out += struct.pack("<HHH", cfg.vector_size, cfg.log2_entries, cfg.residuals)
    out += struct.pack("<BxIII", _SHARING_KIND[cfg.sharing.kind], cfg.sharing.tile_rows, cfg.sharing.tile_cols,
                       cfg.sharing.group_width)
    out += struct.pack("<B3x", len(q.shape))
    out += struct.pack(f"<{len(q.shape)}Q", *q.shape)
    out += struct.pack("<II", q.n_regions, len(q.codebooks))
    for cb in q.codebooks:
        out += struct.pack("<HxxI", cb.residual_level, cb.region_id)
        out += np.ascontiguousarray(cb.entries, dtype="<f4").tobytes()
    out += struct.pack("<Q", q.packed_bit_length)
    out += q.packed_codes()
    return bytes(out)
