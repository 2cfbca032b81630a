"""GPU-resident quantized tensors (weights or KV cache) in the kernels' layouts.

``DeviceVQTensor`` is the device twin of :class:`~.codec.QuantizedTensor`
(pkg/src/vqforge/codec.py:180-226): the same config / shape / region
bookkeeping, with codes held in HBM as

* ``plain``   — the reference ``codes`` array (R, S) in u8/u16 (VQB_LAYOUT_PLAIN)
* ``packed``  — the reference bit stream (bitpack.py:13-28, VQB_LAYOUT_PACKED)
* ``gemv``    — weights interleaved for 128-bit lane loads (VQB_LAYOUT_GEMV_IL)
* ``kv``      — KV cache interleaved for the attention kernel (VQB_LAYOUT_KV_IL)

and codebooks as one contiguous (R * n_regions, K, v) tensor in fp16 (the
paper's 2-byte entries, codec.py:93-96), bf16 or fp32 (parity mode). Host codes
are range-checked once at upload (CodeRangeError with the reference's message,
codec.py:401-405); after that every kernel call is host-synchronisation free.
Interleaved layouts are produced on the GPU by ``vqb_repack``.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .codec import QuantizedTensor, VQConfig, region_count, subvector_count
from .errors import CodeRangeError, ConfigError

_DTYPES = {
    "float32": torch.float32, "fp32": torch.float32, torch.float32: torch.float32,
    "float16": torch.float16, "fp16": torch.float16, torch.float16: torch.float16,
    "bfloat16": torch.bfloat16, "bf16": torch.bfloat16, torch.bfloat16: torch.bfloat16,
}
_ENUM = {torch.float32: N.F32, torch.float16: N.F16, torch.bfloat16: N.BF16}
_LAYOUTS = {"packed": N.LAYOUT_PACKED, "gemv": N.LAYOUT_GEMV_IL, "kv": N.LAYOUT_KV_IL,
            "plain": N.LAYOUT_PLAIN}


def torch_dtype(d) -> torch.dtype:
    try:
        return _DTYPES[d]
    except KeyError:
        raise ConfigError(f"unsupported dtype {d!r}") from None


def dtype_enum(d) -> int:
    return _ENUM[torch_dtype(d)]


def default_device(device=None) -> torch.device:
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device: the B200 kernels have no CPU fallback")
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def stack_codebooks(q) -> np.ndarray:
    """All of ``q``'s books as one (R * n_regions, K, v) fp32 array, level-major
    (book index ``level * n_regions + region``, codec.py:208-209).

    Uses only the attributes vqforge's own ``QuantizedTensor`` has (``codebooks``,
    a list of ``Codebook`` with ``.entries``; pkg/src/vqforge/codec.py:180-197), so
    the reference's objects upload unchanged."""
    books = getattr(q, "codebooks", None)
    if not books:
        raise ConfigError("quantized tensor has no codebooks")
    return np.ascontiguousarray(np.stack([np.asarray(cb.entries, dtype=np.float32) for cb in books]))


def host_codes(q) -> tuple:
    """(codes narrowed to u8/u16 as a byte array, largest code) of a host quantized
    tensor, range-checked with the reference's CodeRangeError message
    (codec.py:401-405). Accepts vqforge's QuantizedTensor (int32 ``codes`` (R, S))."""
    cfg = q.config
    k = cfg.n_entries
    codes = np.asarray(q.codes)
    hi = -1
    if codes.size:
        lo, hi = int(codes.min()), int(codes.max())
        if lo < 0 or hi >= k:
            for r in range(codes.shape[0]):
                row = codes[r]
                bad = row[(row < 0) | (row >= k)]
                if bad.size:
                    raise CodeRangeError(
                        f"code out of range: {int(bad[0])} not in [0, {k}) at residual level {r}")
    narrow = np.uint8 if cfg.log2_entries <= 8 else np.uint16
    return np.ascontiguousarray(codes.astype(narrow)).view(np.uint8), hi


def auto_layout(shape, config: VQConfig) -> str:
    """Pick the interleaved layout the fast kernels read, else ``plain``."""
    b = config.log2_entries
    if len(shape) == 2 and b in (8, 16) and shape[0] % (16 if b <= 8 else 8) == 0:
        return "gemv"
    if len(shape) == 4 and b <= 8:
        groups = shape[3] // config.vector_size
        if groups in (32, 64) and shape[2] % 32 == 0:
            return "kv"
    return "plain"


@dataclass
class DeviceVQTensor:
    config: VQConfig
    shape: tuple
    n_regions: int
    codes: torch.Tensor        # uint8 / int16-viewed-as-u16 / uint8 bytes for packed
    layout: str
    codebooks: torch.Tensor    # (R * n_regions, K, v)
    max_code: int = -1         # largest code present (-1 unknown): lets kernels drop the global tier

    # -- construction ------------------------------------------------------------------------

    @classmethod
    def from_quantized(cls, q: QuantizedTensor, device=None, codebook_dtype="float16",
                       layout: str = "auto") -> "DeviceVQTensor":
        dev = default_device(device)
        cfg = q.config
        host, hi = host_codes(q)
        t = torch.from_numpy(host).to(dev)
        books = torch.from_numpy(stack_codebooks(q)).to(dev).to(torch_dtype(codebook_dtype)).contiguous()
        plain = cls(cfg, tuple(q.shape), q.n_regions, t, "plain", books, hi)
        if layout == "auto":
            layout = auto_layout(q.shape, cfg)
        return plain if layout == "plain" else plain.relayout(layout)

    @classmethod
    def empty_cache(cls, shape, config: VQConfig, codebooks: torch.Tensor, layout: str = "kv") -> "DeviceVQTensor":
        """A zero-coded (B, H, T_capacity, C) KV cache over `codebooks`, filled token by
        token by ops.vq_quantize_kv (the online quantizer)."""
        shape = tuple(int(s) for s in shape)
        n_regions = region_count(shape, config)
        dev = codebooks.device
        probe = cls(config, shape, n_regions, torch.empty(0, dtype=torch.uint8, device=dev), "plain",
                    codebooks.contiguous())
        need = N.check(N.lib().vqb_layout_bytes(probe.struct(), _LAYOUTS[layout]))
        codes = torch.zeros(need, dtype=torch.uint8, device=dev)
        return cls(config, shape, n_regions, codes, layout, codebooks.contiguous(), config.n_entries - 1)

    @classmethod
    def from_packed(cls, stream: bytes, shape, config: VQConfig, codebooks, device=None,
                    codebook_dtype="float16", layout: str = "packed") -> "DeviceVQTensor":
        """Ingest the reference packed stream as-is (no host unpacking)."""
        dev = default_device(device)
        shape = tuple(int(s) for s in shape)
        n_regions = region_count(shape, config)
        pad = (-len(stream)) % 4 + 4
        raw = np.frombuffer(bytes(stream) + b"\0" * pad, dtype=np.uint8)
        t = torch.from_numpy(raw.copy()).to(dev)
        if isinstance(codebooks, torch.Tensor):
            books = codebooks.to(dev)
        else:
            books = torch.from_numpy(np.stack([np.asarray(getattr(c, "entries", c), np.float32)
                                               for c in codebooks])).to(dev)
        books = books.to(torch_dtype(codebook_dtype)).contiguous()
        out = cls(config, shape, n_regions, t, "packed", books)
        return out if layout == "packed" else out.relayout(layout)

    @classmethod
    def from_device_codes(cls, codes: torch.Tensor, shape, config: VQConfig, codebooks: torch.Tensor,
                          layout: str = "plain") -> "DeviceVQTensor":
        """Wrap codes already on the GPU ((R, S) integer array for ``plain``)."""
        shape = tuple(int(s) for s in shape)
        n_regions = region_count(shape, config)
        max_code = -1
        if layout == "plain" and codes.dtype not in (torch.uint8,):
            if codes.numel():
                lo, hi = int(codes.min()), int(codes.max())
                if lo < 0 or hi >= config.n_entries:
                    raise CodeRangeError(f"code out of range: {lo if lo < 0 else hi} not in "
                                         f"[0, {config.n_entries})")
                max_code = hi
            narrow = torch.uint8 if config.log2_entries <= 8 else torch.int16
            codes = codes.to(narrow).contiguous().view(torch.uint8)
        return cls(config, shape, n_regions, codes.contiguous().view(torch.uint8), layout,
                   codebooks.contiguous(), max_code)

    # -- views -------------------------------------------------------------------------------

    @property
    def device(self) -> torch.device:
        return self.codes.device

    @property
    def codebook_dtype(self) -> torch.dtype:
        return self.codebooks.dtype

    @property
    def n_subvectors(self) -> int:
        return subvector_count(self.shape, self.config)

    @property
    def code_bytes(self) -> int:
        return int(self.codes.numel())

    def algorithmic_bytes(self, working_entries=None) -> int:
        """Packed code bytes + codebook bytes (at the stored dtype) of the working set."""
        cfg = self.config
        codes = (cfg.residuals * self.n_subvectors * cfg.log2_entries + 7) // 8
        k = min(working_entries or cfg.n_entries, cfg.n_entries)
        books = cfg.residuals * self.n_regions * k * cfg.vector_size * self.codebooks.element_size()
        return codes + books

    def struct(self) -> N.VqbTensor:
        cfg = self.config
        s = N.VqbTensor()
        s.vector_size = cfg.vector_size
        s.log2_entries = cfg.log2_entries
        s.residuals = cfg.residuals
        s.sharing = N.SHARE[cfg.sharing.kind]
        s.tile_rows = cfg.sharing.tile_rows
        s.tile_cols = cfg.sharing.tile_cols
        s.group_width = cfg.sharing.group_width
        s.ndim = len(self.shape)
        for i, d in enumerate(self.shape):
            s.dims[i] = d
        s.n_regions = self.n_regions
        s.layout = _LAYOUTS[self.layout]
        s.d_codes = self.codes.data_ptr()
        s.codes_bytes = self.codes.numel()
        s.codebook_dtype = _ENUM[self.codebooks.dtype]
        s.d_codebooks = self.codebooks.data_ptr()
        s.max_code = int(self.max_code)
        bt = self.books_per_head()
        s.d_codebooks_t = bt.data_ptr() if bt is not None else None
        return s

    def books_per_head(self):
        """Channel-group books of a KV cache re-laid [H][K][C/v][v] (cached): the
        attention kernel loads a head's K or V books with one bulk copy (64 KB at
        CQ-4, C = 128) instead of a strided gather-and-transpose."""
        cfg = self.config
        if (len(self.shape) != 4 or cfg.sharing.kind != "channel_group" or cfg.sharing.group_width != cfg.vector_size
                or cfg.residuals != 1 or self.layout != "kv" or self.codebooks.dtype != torch.float16):
            return None
        bt = self.__dict__.get("_books_t")
        if bt is None or bt.data_ptr() == 0:
            h, c, v = self.shape[1], self.shape[3], cfg.vector_size
            bt = self.codebooks.view(h, c // v, cfg.n_entries, v).permute(0, 2, 1, 3).contiguous()
            self.__dict__["_books_t"] = bt
        return bt

    def relayout(self, layout: str) -> "DeviceVQTensor":
        if layout == self.layout:
            return self
        if layout == "packed":
            raise ConfigError("repacking to the bit stream is a host operation (bitpack)")
        src = self.struct()
        L = N.lib()
        need = N.check(L.vqb_layout_bytes(src, _LAYOUTS[layout]))
        out = torch.empty(need, dtype=torch.uint8, device=self.device)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        N.check(L.vqb_repack(src, _LAYOUTS[layout], out.data_ptr(), need, stream))
        return DeviceVQTensor(self.config, self.shape, self.n_regions, out, layout, self.codebooks,
                              self.max_code)

    def with_codebook_dtype(self, dtype) -> "DeviceVQTensor":
        d = torch_dtype(dtype)
        if d == self.codebooks.dtype:
            return self
        return DeviceVQTensor(self.config, self.shape, self.n_regions, self.codes, self.layout,
                              self.codebooks.to(d), self.max_code)
