"""Tensor parallelism for the fused VQ layers (one process per GPU, NCCL over NVLink).

The reference is single-process; the north star shards layers
tensor-parallel: GEMV/GEMM by output channel (column-parallel, all-gather) or by
input channel (row-parallel, all-reduce), decode attention by head. Sub-vectors
run along the last axis (pkg/src/vqforge/codec.py:229-236), so a column shard
must start on a sub-vector boundary — and on a codebook-region boundary for tile
or channel-group sharing, because a shard is itself a reference-format
QuantizedTensor whose regions restart at its own column 0 (codec.py:135-177).
Whole-tensor codebooks are replicated to every rank.

Local compute defaults to the CUDA kernels; ``compute`` can be replaced (the
multi-process CPU tests run the sharding and collectives with the oracle).
"""

import ctypes
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch
import torch.distributed as dist

from .codec import Codebook, QuantizedTensor, region_count
from .errors import ConfigError, ShapeError


def _split(extent: int, world: int, rank: int, align: int):
    if extent % world:
        raise ShapeError(f"extent {extent} not divisible by tensor-parallel size {world}")
    part = extent // world
    if part % align:
        raise ConfigError(f"shard width {part} is not a multiple of {align} (sub-vector / codebook region)")
    return rank * part, (rank + 1) * part


def _col_align(q: QuantizedTensor) -> int:
    sh = q.config.sharing
    if sh.kind == "tile":
        return sh.tile_cols
    if sh.kind == "channel_group":
        return sh.group_width
    return q.config.vector_size


def shard_columns(q: QuantizedTensor, rank: int, world: int) -> QuantizedTensor:
    """Column-parallel shard of a 2-D weight (M, N): columns [n0, n1) with their books."""
    if len(q.shape) != 2:
        raise ShapeError("column sharding expects a 2-D (M, N) weight")
    m, n = q.shape
    v = q.config.vector_size
    n0, n1 = _split(n, world, rank, _col_align(q))
    per_row = n // v
    codes = q.codes.reshape(q.config.residuals, m, per_row)[:, :, n0 // v:n1 // v]
    codes = np.ascontiguousarray(codes).reshape(q.config.residuals, -1)
    shape = (m, n1 - n0)
    nreg = region_count(shape, q.config)
    sh = q.config.sharing
    if sh.kind == "whole":
        books = list(q.codebooks)
    else:
        # regions of the shard, expressed in the parent's region numbering
        if sh.kind == "tile":
            n_tc_parent = -(-n // sh.tile_cols)
            n_tr = -(-m // sh.tile_rows)
            n_tc = (n1 - n0) // sh.tile_cols
            parent = [tr * n_tc_parent + n0 // sh.tile_cols + tc for tr in range(n_tr) for tc in range(n_tc)]
        else:
            g0 = n0 // sh.group_width
            parent = [g0 + gi for gi in range(nreg)]
        books = []
        for lvl in range(q.config.residuals):
            for local, p in enumerate(parent):
                src = q.codebook_for(lvl, p)
                books.append(Codebook(src.entries, lvl, local))
    return QuantizedTensor(codes, shape, q.config, books, nreg)


def shard_rows(q: QuantizedTensor, rank: int, world: int) -> QuantizedTensor:
    """Row-parallel shard (input channels [m0, m1)) of a 2-D weight."""
    if len(q.shape) != 2:
        raise ShapeError("row sharding expects a 2-D (M, N) weight")
    m, n = q.shape
    sh = q.config.sharing
    align = sh.tile_rows if sh.kind == "tile" else 1
    m0, m1 = _split(m, world, rank, align)
    per_row = n // q.config.vector_size
    codes = q.codes.reshape(q.config.residuals, m, per_row)[:, m0:m1, :]
    codes = np.ascontiguousarray(codes).reshape(q.config.residuals, -1)
    shape = (m1 - m0, n)
    nreg = region_count(shape, q.config)
    if sh.kind == "tile":
        n_tc = -(-n // sh.tile_cols)
        tr0 = m0 // sh.tile_rows
        books = [Codebook(q.codebook_for(lvl, (tr0 + r // n_tc) * n_tc + r % n_tc).entries, lvl, r)
                 for lvl in range(q.config.residuals) for r in range(nreg)]
    else:
        books = list(q.codebooks)
    return QuantizedTensor(codes, shape, q.config, books, nreg)


def shard_heads(q: QuantizedTensor, rank: int, world: int) -> QuantizedTensor:
    """Head shard of a (B, H, T, C) KV tensor; channel-group books move with their heads."""
    if len(q.shape) != 4:
        raise ShapeError("head sharding expects a (B, H, T, C) tensor")
    b, h, t, c = q.shape
    h0, h1 = _split(h, world, rank, 1)
    v = q.config.vector_size
    codes = q.codes.reshape(q.config.residuals, b, h, t, c // v)[:, :, h0:h1]
    codes = np.ascontiguousarray(codes).reshape(q.config.residuals, -1)
    shape = (b, h1 - h0, t, c)
    nreg = region_count(shape, q.config)
    sh = q.config.sharing
    if sh.kind == "channel_group":
        per_head = c // sh.group_width
        books = [Codebook(q.codebook_for(lvl, (h0 * per_head) + r).entries, lvl, r)
                 for lvl in range(q.config.residuals) for r in range(nreg)]
    elif sh.kind == "whole":
        books = list(q.codebooks)
    else:
        raise ConfigError("tile-shared KV tensors are shared across heads; shard them by columns instead")
    return QuantizedTensor(codes, shape, q.config, books, nreg)


def _backend(group) -> str:
    try:
        return dist.get_backend(group)
    except Exception:  # pragma: no cover
        return "nccl"


def all_gather_into(out: torch.Tensor, y: torch.Tensor, group=None) -> None:
    """all_gather_into_tensor (NCCL); gloo (the CPU / single-GPU multi-process tests)
    gathers into a list and concatenates."""
    if _backend(group) == "nccl":
        dist.all_gather_into_tensor(out, y, group=group)
        return
    parts = list(out.view((dist.get_world_size(group),) + tuple(y.shape)).unbind(0))
    dist.all_gather(parts, y, group=group)


def device_shard(w, rows=None, col_ranges=None):
    """Shard of a device-resident 2-D weight with a whole-tensor codebook (replicated):
    input rows [r0, r1) and/or the concatenation of output column ranges
    [(c0, c1), ...] — e.g. one rank's q | k | v head columns of a fused qkv weight.
    Done on the GPU from the plain codes; returns a DeviceVQTensor in the input's layout."""
    from .device import DeviceVQTensor
    cfg = w.config
    if cfg.sharing.kind != "whole" or len(w.shape) != 2:
        raise ConfigError("device_shard handles 2-D weights with whole-tensor codebooks")
    m, n = w.shape
    v = cfg.vector_size
    plain = w.relayout("plain")
    s = m * n // v
    if cfg.log2_entries <= 8:
        codes = plain.codes[: cfg.residuals * s].view(cfg.residuals, m, n // v).to(torch.int32)
    else:
        codes = (plain.codes[: 2 * cfg.residuals * s].view(torch.int16).to(torch.int32) & 0xFFFF).view(
            cfg.residuals, m, n // v)
    r0, r1 = rows if rows is not None else (0, m)
    codes = codes[:, r0:r1]
    if col_ranges is not None:
        for c0, c1 in col_ranges:
            if c0 % v or c1 % v:
                raise ConfigError(f"column range ({c0}, {c1}) is not on a sub-vector boundary")
        codes = torch.cat([codes[:, :, c0 // v:c1 // v] for c0, c1 in col_ranges], dim=2)
    shape = (r1 - r0, codes.shape[2] * v)
    out = DeviceVQTensor.from_device_codes(codes.reshape(cfg.residuals, -1).contiguous(), shape, cfg,
                                           w.codebooks, layout="plain")
    out.max_code = w.max_code
    return out if w.layout == "plain" else out.relayout(w.layout)


def _default_linear(w, x):
    from .device import DeviceVQTensor
    from .ops import vq_gemm, vq_gemv

    d = w if isinstance(w, DeviceVQTensor) else DeviceVQTensor.from_quantized(w, device=x.device)
    return vq_gemv(d, x) if (x.dim() == 1 or x.shape[0] <= 8) else vq_gemm(d, x)


def _default_attention(k, v, q):
    from .device import DeviceVQTensor
    from .ops import vq_attention

    kd = k if isinstance(k, DeviceVQTensor) else DeviceVQTensor.from_quantized(k, device=q.device)
    vd = v if isinstance(v, DeviceVQTensor) else DeviceVQTensor.from_quantized(v, device=q.device)
    return vq_attention(kd, vd, q)


class PeerComm:
    """Fused tensor-parallel collectives over peer memory (csrc/tp.cu, include/vqb.h
    VqbPeerComm): one symmetric buffer per rank, mapped on every peer through CUDA IPC
    (handles exchanged over the process group, any backend). ``linear`` runs the
    decode GEMV whose epilogue pushes each finished output element into every rank's
    slot, then the finish kernel waits for all ranks and reduces (row-parallel) or
    gathers (column-parallel) — the NCCL call after the linear disappears from the
    critical path. One process per GPU on an NVLink node; the tests run two
    processes on one GPU (IPC within a device)."""

    def __init__(self, max_rows: int, max_n: int, group=None, device=None):
        from . import _native as N
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world > N.TP_MAX_WORLD:
            raise ConfigError(f"fused TP collectives support up to {N.TP_MAX_WORLD} ranks, got {self.world}")
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        # a slot holds rows x N (all-reduce) or rows x N x world (all-gather) fp32
        self.slot_elems = int(max_rows) * int(max_n) * self.world
        lib = N.lib()
        nbytes = N.check(lib.vqb_tp_buffer_bytes(self.world, self.slot_elems))
        self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)
        handle = (ctypes.c_uint8 * 64)()
        off = ctypes.c_int64(0)
        N.check(lib.vqb_ipc_get_handle(ctypes.c_void_p(self.buf.data_ptr()), handle, ctypes.byref(off)))
        torch.cuda.synchronize(self.device)
        mine = (bytes(handle), int(off.value))
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        self._opened = []
        ptrs = []
        for r, (h, o) in enumerate(allh):
            if r == self.rank:
                ptrs.append(self.buf.data_ptr())
                continue
            hb = (ctypes.c_uint8 * 64).from_buffer_copy(h)
            p = ctypes.c_void_p(0)
            N.check(lib.vqb_ipc_open_handle(hb, int(o), ctypes.byref(p)))
            self._opened.append(p.value)
            ptrs.append(p.value)
        self.c = N.VqbPeerComm()
        self.c.rank, self.c.world, self.c.slot_elems = self.rank, self.world, self.slot_elems
        for r, p in enumerate(ptrs):
            self.c.d_peer[r] = p
        dist.barrier(group=group)

    def linear(self, w, x: torch.Tensor, mode: str = "row", out_dtype=torch.float16) -> torch.Tensor:
        """y = collective(x @ dequant(W_shard)): ``row`` sums the partial outputs of
        every rank, ``column`` concatenates their column blocks along N."""
        from . import _native as N
        from .ops import _stream, dtype_enum, torch_dtype, workspace
        x2 = x.reshape(1, -1) if x.dim() == 1 else x
        x2 = x2.contiguous()
        rows = x2.shape[0]
        m, n = w.shape
        md = N.TP_ALLREDUCE if mode == "row" else N.TP_ALLGATHER
        L = N.VqbLaunch()
        lib = N.lib()
        s = w.struct()
        need = N.check(lib.vqb_workspace_bytes(N.KERNEL_GEMV, s, rows, L))
        ws = workspace(need, w.device)
        st = _stream(w.device)
        N.check(lib.vqb_gemv_tp(s, x2.data_ptr(), dtype_enum(x2.dtype), rows, md, ctypes.byref(self.c), L,
                                ws.data_ptr(), ws.numel(), st))
        od = torch_dtype(out_dtype)
        y = torch.empty((rows, n * (self.world if md == N.TP_ALLGATHER else 1)), dtype=od, device=w.device)
        N.check(lib.vqb_tp_finish(ctypes.byref(self.c), md, rows, n, y.data_ptr(), dtype_enum(od), st))
        return y[0] if x.dim() == 1 else y

    def take_error(self) -> int:
        from . import _native as N
        v = ctypes.c_int32(0)
        N.check(N.lib().vqb_tp_take_error(ctypes.byref(self.c), ctypes.byref(v)))
        return int(v.value)

    def close(self) -> None:
        from . import _native as N
        torch.cuda.synchronize(self.device)
        for p in self._opened:
            N.check(N.lib().vqb_ipc_close_handle(ctypes.c_void_p(p)))
        self._opened = []


@dataclass
class TPLinear:
    """A VQ linear layer sharded over a process group.

    ``mode="column"``: every rank holds N/world output columns; ``forward`` all-gathers
    the full output. ``mode="row"``: every rank holds M/world input rows and takes the
    matching slice of x; ``forward`` all-reduces the partial sums.
    """

    weight: object
    mode: str = "column"
    group: Optional[object] = None
    compute: Callable = _default_linear
    comm: Optional[PeerComm] = None  # fused peer-memory collective instead of NCCL (decode GEMV sizes)

    @classmethod
    def from_full(cls, q: QuantizedTensor, mode="column", group=None, compute=None, device=None):
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        shard = shard_columns(q, rank, world) if mode == "column" else shard_rows(q, rank, world)
        w = shard
        if compute is None:
            from .device import DeviceVQTensor
            w = DeviceVQTensor.from_quantized(shard, device=device)
        return cls(w, mode, group, compute or _default_linear)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        world = dist.get_world_size(self.group)
        if self.comm is not None and (x.dim() == 1 or x.shape[0] <= 8):
            if self.mode == "column":
                return self.comm.linear(self.weight, x, "column", out_dtype=x.dtype)
            rank = dist.get_rank(self.group)
            m_local = self.weight.shape[0]
            return self.comm.linear(self.weight, x[..., rank * m_local:(rank + 1) * m_local], "row",
                                    out_dtype=x.dtype)
        if self.mode == "column":
            y = self.compute(self.weight, x).contiguous()
            out = torch.empty((world * y.shape[0],) + tuple(y.shape[1:]), dtype=y.dtype, device=y.device)
            all_gather_into(out, y, group=self.group)
            out = out.view((world,) + tuple(y.shape))
            # (world, ..., N/world) -> (..., N)
            return torch.movedim(out, 0, -2).reshape(tuple(y.shape[:-1]) + (world * y.shape[-1],))
        rank = dist.get_rank(self.group)
        m_local = self.weight.shape[0]
        xs = x[..., rank * m_local:(rank + 1) * m_local].contiguous()
        y = self.compute(self.weight, xs).contiguous()
        dist.all_reduce(y, group=self.group)
        return y

    __call__ = forward


@dataclass
class TPAttention:
    """Decode attention sharded by head; the output is all-gathered over heads."""

    k: object
    v: object
    group: Optional[object] = None
    compute: Callable = _default_attention

    @classmethod
    def from_full(cls, kq: QuantizedTensor, vq: QuantizedTensor, group=None, compute=None, device=None):
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        ks, vs = shard_heads(kq, rank, world), shard_heads(vq, rank, world)
        if compute is None:
            from .device import DeviceVQTensor
            ks = DeviceVQTensor.from_quantized(ks, device=device)
            vs = DeviceVQTensor.from_quantized(vs, device=device)
        return cls(ks, vs, group, compute or _default_attention)

    def forward(self, q: torch.Tensor) -> torch.Tensor:
        world, rank = dist.get_world_size(self.group), dist.get_rank(self.group)
        h_local = self.k.shape[1]
        qs = q[:, rank * h_local:(rank + 1) * h_local].contiguous()
        o = self.compute(self.k, self.v, qs).contiguous()
        out = torch.empty((world * o.shape[0],) + tuple(o.shape[1:]), dtype=o.dtype, device=o.device)
        all_gather_into(out, o, group=self.group)
        out = out.view((world,) + tuple(o.shape))
        return torch.movedim(out, 0, 1).reshape(o.shape[0], world * h_local, o.shape[2])

    __call__ = forward
