"""Host codec for the reference's packed index stream.

Format (pkg/src/vqforge/bitpack.py:13-43): every index occupies exactly ``bits``
bits, least-significant bit first, indices back to back with no per-index
padding; only the end of the stream is padded to a byte. The device kernels read
the same stream directly (layout VQB_LAYOUT_PACKED, csrc/common.cuh:code_at), so
these helpers are only needed to produce / consume it on the host.

Implementation: each index is scattered into a little-endian uint64 word array
with two shifted ORs (an index of <= 32 bits straddles at most two words), which
avoids materialising a bit matrix.
"""

import numpy as np

from .errors import CodeRangeError


def packed_length(count: int, bits: int) -> int:
    """Bytes needed for ``count`` indices of ``bits`` bits each."""
    return (int(count) * int(bits) + 7) // 8


def _check_bits(bits: int) -> None:
    if not 1 <= bits <= 32:
        raise ValueError(f"bits must be in [1, 32], got {bits}")


def pack_indices(values, bits: int) -> bytes:
    """Pack non-negative integers < 2**bits into the contiguous LSB-first stream."""
    _check_bits(bits)
    vals = np.ascontiguousarray(values, dtype=np.int64).reshape(-1)
    if vals.size == 0:
        return b""
    if int(vals.min()) < 0 or int(vals.max()) >= (1 << bits):
        raise CodeRangeError(f"code out of range for {bits}-bit packing")
    u = vals.astype(np.uint64)
    bitpos = np.arange(vals.size, dtype=np.uint64) * np.uint64(bits)
    word = (bitpos >> np.uint64(6)).astype(np.int64)
    shift = bitpos & np.uint64(63)
    n_words = (vals.size * bits + 63) // 64 + 1
    words = np.zeros(n_words, dtype=np.uint64)
    np.bitwise_or.at(words, word, u << shift)
    spill = shift + np.uint64(bits) > np.uint64(64)
    if spill.any():
        hi = u[spill] >> (np.uint64(64) - shift[spill])
        np.bitwise_or.at(words, word[spill] + 1, hi)
    raw = words.astype("<u8").tobytes()
    return raw[: packed_length(vals.size, bits)]


def unpack_indices(data: bytes, bits: int, count: int) -> np.ndarray:
    """Inverse of :func:`pack_indices`; returns an int32 array of ``count`` codes."""
    _check_bits(bits)
    if count == 0:
        return np.zeros(0, dtype=np.int32)
    need = packed_length(count, bits)
    if len(data) < need:
        raise ValueError(f"packed stream truncated: {len(data)} < {need} bytes")
    buf = np.zeros(((need + 7) // 8 + 1) * 8, dtype=np.uint8)
    buf[:need] = np.frombuffer(data, dtype=np.uint8, count=need)
    words = buf.view("<u8").astype(np.uint64)
    bitpos = np.arange(count, dtype=np.uint64) * np.uint64(bits)
    word = (bitpos >> np.uint64(6)).astype(np.int64)
    shift = bitpos & np.uint64(63)
    lo = words[word] >> shift
    # bits that continue in the next word (shift + bits > 64)
    take_hi = shift + np.uint64(bits) > np.uint64(64)
    hi = np.zeros(count, dtype=np.uint64)
    if take_hi.any():
        hi[take_hi] = words[word[take_hi] + 1] << (np.uint64(64) - shift[take_hi])
    mask = np.uint64((1 << bits) - 1)
    return ((lo | hi) & mask).astype(np.int32)
