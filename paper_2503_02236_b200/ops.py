"""Functional torch-facing entry points: vq_dequantize / vq_gemv / vq_gemm / vq_attention.

Every call goes straight to the C ABI (include/vqb.h) on the tensor's device and
the current CUDA stream; nothing here computes on the host. Shapes follow the
reference: weights W (M, N) with y = x @ W (pkg/src/vqforge/sim.py:136-144);
attention q (B, H, C) with K, V (B, H, T, C) (sim.py:145-155).
"""

import contextlib
import threading

import torch

from . import _native as N
from .device import DeviceVQTensor, dtype_enum, torch_dtype
from .errors import CapacityError, ConfigError, ShapeError

# -- workspace arena ----------------------------------------------------------------------------
# One zero-initialised byte buffer per (device, stream). The kernels keep split
# arrival counters / tagged slots in its head and reset them themselves, so it is
# zeroed only when (re)allocated. Objects that capture CUDA graphs must not use
# the shared arena (a later, larger request would free the buffer a graph baked in,
# and two graphs sharing one slot head must never replay concurrently): they own a
# ``Workspace`` and route their ops to it with ``use_workspace``.

_ws = {}
_ws_lock = threading.Lock()
_tls = threading.local()


class Workspace:
    """A private, growable zeroed arena for one graph-owning object (decoder, stack)."""

    def __init__(self, device, nbytes: int = 1 << 20):
        self.device = torch.device(device)
        self.buf = torch.zeros(max(int(nbytes), 1 << 20), dtype=torch.uint8, device=self.device)

    def get(self, nbytes: int) -> torch.Tensor:
        if self.buf.numel() < nbytes:
            if torch.cuda.is_current_stream_capturing():
                raise CapacityError(f"private workspace of {self.buf.numel()} B cannot grow to {nbytes} B "
                                    "during graph capture (run the step once eagerly first)")
            self.buf = torch.zeros(max(int(nbytes), 2 * self.buf.numel()), dtype=torch.uint8, device=self.device)
        return self.buf


@contextlib.contextmanager
def use_workspace(ws: Workspace):
    """Every op on this thread takes its workspace from ``ws`` inside the block."""
    prev = getattr(_tls, "ws", None)
    _tls.ws = ws
    try:
        yield ws
    finally:
        _tls.ws = prev


def workspace(nbytes: int, device: torch.device) -> torch.Tensor:
    own = getattr(_tls, "ws", None)
    if own is not None and own.device == torch.device(device):
        return own.get(nbytes)
    stream = torch.cuda.current_stream(device).cuda_stream
    key = (device.index, stream)
    with _ws_lock:
        buf = _ws.get(key)
        if buf is None or buf.numel() < nbytes:
            size = max(int(nbytes), 1 << 20)
            if buf is not None:
                size = max(size, 2 * buf.numel())
            buf = torch.zeros(size, dtype=torch.uint8, device=device)
            _ws[key] = buf
        return buf


def launch_struct(plans=None, n_shared=None, split_factor=None, split_axis=None, force_generic=False,
                  grid_limit=0) -> N.VqbLaunch:
    """VqbLaunch from FusedPlans (sim.py:229-236) and/or explicit knobs."""
    L = N.VqbLaunch()
    if plans is not None:
        cp, fp = plans.cache_plan, plans.dataflow_plan
        L.n_reg = int(cp.n_reg)
        L.n_shared = int(cp.n_shared)
        L.split_axis = ord(fp.split_axis) if fp.split_axis else 0
        L.split_factor = int(fp.split_factor)
        L.fusion_level = 0 if plans.fusion_level == "register" else 1
    if n_shared is not None:
        L.n_shared = int(n_shared)
    if split_factor is not None:
        L.split_factor = int(split_factor)
    if split_axis is not None:
        L.split_axis = ord(split_axis) if split_axis else 0
    if force_generic:
        L.flags |= N.FLAG_FORCE_GENERIC
    L.grid_limit = int(grid_limit)
    return L


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def vq_dequantize(w: DeviceVQTensor, out_dtype=None) -> torch.Tensor:
    """Dense reconstruction (codec.py:391-408); fp32 output is bit-exact."""
    dt = torch_dtype(out_dtype or torch.float32)
    out = torch.empty(w.shape, dtype=dt, device=w.device)
    N.check(N.lib().vqb_dequant(w.struct(), out.data_ptr(), dtype_enum(dt), _stream(w.device)))
    return out


def _matmul(kind: int, w: DeviceVQTensor, x: torch.Tensor, out_dtype, launch) -> torch.Tensor:
    if len(w.shape) != 2:
        raise ShapeError(f"quantized weight must be 2-D, got {w.shape}")
    m, n = w.shape
    squeeze = x.dim() == 1
    x2 = x.reshape(1, -1) if squeeze else x
    if x2.dim() != 2 or x2.shape[1] != m:
        raise ShapeError(f"activation {tuple(x.shape)} does not match M={m}")
    if x2.device != w.device:
        raise ConfigError(f"activation on {x2.device}, weight on {w.device}")
    x2 = x2.contiguous()
    rows = x2.shape[0]
    od = torch_dtype(out_dtype or torch.float32)
    y = torch.empty((rows, n), dtype=od, device=w.device)
    L = launch if launch is not None else N.VqbLaunch()
    lib = N.lib()
    s = w.struct()
    need = N.check(lib.vqb_workspace_bytes(kind, s, rows, L))
    ws = workspace(need, w.device)
    fn = lib.vqb_gemv if kind == N.KERNEL_GEMV else lib.vqb_gemm
    N.check(fn(s, x2.data_ptr(), dtype_enum(x2.dtype), rows, y.data_ptr(), dtype_enum(od), L,
               ws.data_ptr(), ws.numel(), _stream(w.device)))
    return y[0] if squeeze else y


def vq_gemv(w: DeviceVQTensor, x: torch.Tensor, out_dtype=None, launch=None) -> torch.Tensor:
    """Decode GEMV y = x @ dequant(W) for x of shape (M,) or (rows<=8, M)."""
    return _matmul(N.KERNEL_GEMV, w, x, out_dtype, launch)


def vq_gemv_rmsnorm(w: DeviceVQTensor, x, residual: torch.Tensor, weight: torch.Tensor, eps: float,
                    residual_out: torch.Tensor = None, out_dtype=torch.float16, launch=None,
                    swiglu: bool = False) -> torch.Tensor:
    """Batch-1 decode GEMV with the residual add + RMSNorm fused into its prologue:
    h = residual + x (x may be None), residual_out = h, y = (weight * rmsnorm(h)) @ W.
    The same result as ``rmsnorm`` followed by ``vq_gemv``, one launch instead of two;
    ``residual_out`` must be a different buffer from ``residual`` (every CTA reads it)."""
    if residual_out is not None and residual_out.data_ptr() == residual.data_ptr():
        raise ConfigError("residual_out must not alias residual")
    mode = N.XF_RMSNORM | (N.XF_SWIGLU_OUT if swiglu else 0)
    return _gemv_xf(w, x, mode, residual, residual_out, weight, eps, out_dtype, launch)


def vq_gemv_silu(w: DeviceVQTensor, gate_up: torch.Tensor, out_dtype=torch.float16, launch=None) -> torch.Tensor:
    """Batch-1 decode GEMV of silu(gate) * up for a fused [gate | up] input, the SiLU
    gating computed in the GEMV's prologue (``silu_mul`` + ``vq_gemv`` in one launch)."""
    return _gemv_xf(w, gate_up, N.XF_SILU_MUL, None, None, None, 0.0, out_dtype, launch)


def _gemv_xf(w, x, mode, res_in, res_out, weight, eps, out_dtype, launch):
    if len(w.shape) != 2:
        raise ShapeError(f"quantized weight must be 2-D, got {w.shape}")
    m, n = w.shape
    swiglu = bool(mode & N.XF_SWIGLU_OUT)
    want = 2 * m if (mode & ~N.XF_SWIGLU_OUT) == N.XF_SILU_MUL else m
    for t in (x, res_in, res_out, weight):
        if t is not None and (t.numel() != (want if t is x else m) or t.dtype != torch.float16):
            raise ShapeError(f"fused-activation GEMV operand of {t.numel()} {t.dtype} values, expected fp16 "
                             f"rows of {want if t is x else m}")
    od = torch_dtype(out_dtype or torch.float16)
    y = torch.empty((1, n // 2 if swiglu else n), dtype=od, device=w.device)
    L = launch if launch is not None else N.VqbLaunch()
    lib = N.lib()
    s = w.struct()
    need = N.check(lib.vqb_workspace_bytes(N.KERNEL_GEMV, s, 1, L))
    ws = workspace(need, w.device)
    for t in (x, res_in, res_out, weight):
        if t is not None and not t.is_contiguous():
            raise ConfigError("fused-activation GEMV operands must be contiguous")
    ptr = lambda t: t.data_ptr() if t is not None else None
    N.check(lib.vqb_gemv_xf(s, ptr(x), N.F16, mode, ptr(res_in), ptr(res_out), ptr(weight), float(eps),
                            y.data_ptr(), dtype_enum(od), L, ws.data_ptr(), ws.numel(), _stream(w.device)))
    return y


def vq_gemm(w: DeviceVQTensor, x: torch.Tensor, out_dtype=None, launch=None) -> torch.Tensor:
    """Prefill GEMM y = X @ dequant(W) for X of shape (rows, M)."""
    return _matmul(N.KERNEL_GEMM, w, x, out_dtype, launch)


def vq_attention(k: DeviceVQTensor, v: DeviceVQTensor, q: torch.Tensor, out_dtype=None,
                 launch=None, length: int = None, d_len: torch.Tensor = None) -> torch.Tensor:
    """Decode attention softmax(q K^T / sqrt(C)) V over a VQ KV cache, q (B, H, C).

    ``length`` attends to the first tokens of a cache whose capacity is K's T axis;
    ``d_len`` (a device int32) supplies that length on the device instead, so a
    decode step can replay as a CUDA graph while the cache grows."""
    if len(k.shape) != 4:
        raise ShapeError(f"quantized K must be (B, H, T, C), got {k.shape}")
    b, h, t, c = k.shape
    if tuple(q.shape) != (b, h, c):
        raise ShapeError(f"query shape {tuple(q.shape)} != {(b, h, c)}")
    q = q.contiguous()
    od = torch_dtype(out_dtype or torch.float32)
    out = torch.empty((b, h, c), dtype=od, device=k.device)
    L = launch if launch is not None else N.VqbLaunch()
    lib = N.lib()
    ks, vs = k.struct(), v.struct()
    need = N.check(lib.vqb_workspace_bytes(N.KERNEL_ATTN, ks, b * h, L))
    ws = workspace(need, k.device)
    n = t if length is None else int(length)
    N.check(lib.vqb_attn_decode_len(ks, vs, q.data_ptr(), dtype_enum(q.dtype), b, h, n, c,
                                    d_len.data_ptr() if d_len is not None else None, out.data_ptr(),
                                    dtype_enum(od), L, ws.data_ptr(), ws.numel(), _stream(k.device)))
    return out


def rmsnorm(x, residual: torch.Tensor, weight: torch.Tensor, eps: float = 1e-5, out=None) -> torch.Tensor:
    """Llama RMSNorm with the residual add fused: residual += x (in place, fp16;
    x may be None), returns weight * rmsnorm(residual)."""
    rows, dim = residual.shape
    out = torch.empty_like(residual) if out is None else out
    N.check(N.lib().vqb_rmsnorm(x.data_ptr() if x is not None else None, residual.data_ptr(), weight.data_ptr(),
                                out.data_ptr(), rows, dim, float(eps), _stream(residual.device)))
    return out


def qkv_rope(qkv: torch.Tensor, heads: int, head_dim: int, d_len: torch.Tensor, theta: float = 10000.0,
             q_out=None) -> torch.Tensor:
    """RoPE at position d_len[0]-1 on the q/k thirds of a fused qkv row block; returns q."""
    b = qkv.shape[0]
    q_out = torch.empty((b, heads, head_dim), dtype=qkv.dtype, device=qkv.device) if q_out is None else q_out
    N.check(N.lib().vqb_qkv_rope(qkv.data_ptr(), q_out.data_ptr(), b, heads, head_dim, d_len.data_ptr(),
                                 float(theta), _stream(qkv.device)))
    return q_out


def qkv_rope_append(qkv: torch.Tensor, k_cache: DeviceVQTensor, v_cache: DeviceVQTensor, d_len: torch.Tensor,
                    theta: float = 10000.0, q_out=None) -> torch.Tensor:
    """Fused qkv_rope + online quantization of the roped k and v rows into the caches
    at position d_len[0]-1; returns the roped q (B, H, C)."""
    b, h, _, c = k_cache.shape
    q_out = torch.empty((b, h, c), dtype=qkv.dtype, device=qkv.device) if q_out is None else q_out
    N.check(N.lib().vqb_qkv_rope_append(qkv.data_ptr(), q_out.data_ptr(), k_cache.struct(), v_cache.struct(), b, h, c,
                                        d_len.data_ptr(), float(theta), _stream(qkv.device)))
    return q_out


def vq_attention_append(k_cache: DeviceVQTensor, v_cache: DeviceVQTensor, qkv: torch.Tensor, d_len: torch.Tensor,
                        theta: float = 10000.0, out_dtype=torch.float16, launch=None) -> torch.Tensor:
    """One launch for ``qkv_rope_append`` + ``vq_attention(..., d_len=d_len)``: the
    attention kernel ropes q, and the CTA covering the new token of each (b, h) ropes k,
    quantizes the new K / V rows against the books it already holds and writes the codes
    before attending (CQ-4 caches). Same results as the two-kernel form."""
    b, h, t, c = k_cache.shape
    if qkv.shape != (b, 3 * h * c) or qkv.dtype != torch.float16 or not qkv.is_contiguous():
        raise ShapeError(f"fused qkv {tuple(qkv.shape)} {qkv.dtype} does not match (B, 3*H*C) = {(b, 3 * h * c)} fp16")
    od = torch_dtype(out_dtype or torch.float16)
    out = torch.empty((b, h, c), dtype=od, device=k_cache.device)
    L = launch if launch is not None else N.VqbLaunch()
    lib = N.lib()
    ks, vs = k_cache.struct(), v_cache.struct()
    need = N.check(lib.vqb_workspace_bytes(N.KERNEL_ATTN, ks, b * h, L))
    ws = workspace(need, k_cache.device)
    N.check(lib.vqb_attn_decode_append(ks, vs, qkv.data_ptr(), b, h, c, d_len.data_ptr(), float(theta), out.data_ptr(),
                                       dtype_enum(od), L, ws.data_ptr(), ws.numel(), _stream(k_cache.device)))
    return out


def silu_mul(gate_up: torch.Tensor, out=None) -> torch.Tensor:
    rows, f2 = gate_up.shape
    out = torch.empty((rows, f2 // 2), dtype=gate_up.dtype, device=gate_up.device) if out is None else out
    N.check(N.lib().vqb_silu_mul(gate_up.data_ptr(), out.data_ptr(), rows, f2 // 2, _stream(gate_up.device)))
    return out


def sample(logits: torch.Tensor, temperature: float = 0.0, top_k: int = 0, seed: int = 0,
           d_step: torch.Tensor = None, out: torch.Tensor = None, top_p: float = 1.0) -> torch.Tensor:
    """Next tokens (B,) int64 from logits (B, vocab) fp16/fp32: a Gumbel-max draw from
    softmax(logits / temperature) over the top_k largest logits (0 = all; ties at the
    k-th value kept) and then the top_p nucleus (1.0 = off), noise hashed from
    (seed, d_step[0], row, index); temperature 0 is greedy argmax (lowest index on ties,
    like torch.argmax)."""
    if logits.dim() != 2 or logits.dtype not in (torch.float16, torch.float32) or not logits.is_contiguous():
        raise ShapeError(f"logits {tuple(logits.shape)} {logits.dtype} must be a contiguous (B, vocab) fp16/fp32 tensor")
    b, v = logits.shape
    out = torch.empty(b, dtype=torch.int64, device=logits.device) if out is None else out
    if out.dtype != torch.int64 or out.numel() != b or not out.is_contiguous():
        raise ShapeError("sample writes a contiguous (B,) int64 tensor")
    if d_step is not None and (d_step.dtype != torch.int32 or d_step.device != logits.device):
        raise ShapeError("d_step must be a device int32 tensor")
    N.check(N.lib().vqb_sample(logits.data_ptr(), dtype_enum(logits.dtype), b, v, float(temperature), int(top_k),
                               float(top_p), int(seed) & 0xFFFFFFFFFFFFFFFF, None if d_step is None else d_step.data_ptr(),
                               out.data_ptr(), _stream(logits.device)))
    return out


def add_len(d_len: torch.Tensor, delta: int = 1) -> None:
    N.check(N.lib().vqb_add_len(d_len.data_ptr(), int(delta), _stream(d_len.device)))


def vq_quantize_kv(cache: DeviceVQTensor, x: torch.Tensor, tok0: int = 0, d_len: torch.Tensor = None) -> None:
    """Online KV quantization (reference quantize, codec.py:367-389) of new rows
    x (B, H, n_tok, C) into the cache at tokens [tok0, tok0 + n_tok) — or ending at
    d_len[0] (a device int32) when given, for graph-replayed decode steps. Any strides
    with contiguous channels are accepted."""
    if len(cache.shape) != 4:
        raise ShapeError(f"KV cache must be (B, H, T, C), got {cache.shape}")
    b, h, _, c = cache.shape
    if x.dim() != 4 or x.shape[0] != b or x.shape[1] != h or x.shape[3] != c or x.stride(3) != 1:
        raise ShapeError(f"rows {tuple(x.shape)} do not match cache {cache.shape}")
    if x.dtype not in (torch.float16, torch.float32):
        raise ConfigError("KV rows must be fp16 or fp32")
    ptr = d_len.data_ptr() if d_len is not None else None
    N.check(N.lib().vqb_cq_quantize(cache.struct(), x.data_ptr(), dtype_enum(x.dtype), x.stride(0), x.stride(1),
                                    x.stride(2), x.shape[2], int(tok0), ptr, _stream(cache.device)))


def vq_codes_regions(w: DeviceVQTensor):
    """(codes (R, S) int64, region id per sub-vector (S,) int64), both on the device.

    Codes come from the GPU repack to the plain layout; region ids restate
    region_layout (pkg/src/vqforge/codec.py:135-177) with torch index arithmetic.
    """
    cfg = w.config
    plain = w.relayout("plain")
    s = w.n_subvectors
    if cfg.log2_entries <= 8:
        codes = plain.codes[: cfg.residuals * s].view(cfg.residuals, s).to(torch.int64)
    else:
        codes = plain.codes[: 2 * cfg.residuals * s].view(torch.int16).view(cfg.residuals, s)
        codes = codes.to(torch.int64) & 0xFFFF
    shape = w.shape
    v = cfg.vector_size
    per_row = shape[-1] // v
    idx = torch.arange(s, device=w.device, dtype=torch.int64)
    row, col = idx // per_row, (idx % per_row) * v
    sh = cfg.sharing
    if sh.kind == "whole":
        regions = torch.zeros_like(idx)
    elif sh.kind == "channel_group":
        grp = col // sh.group_width
        regions = (((row // shape[2]) % shape[1]) * (shape[-1] // sh.group_width) + grp
                   if len(shape) == 4 else grp)
    else:
        n_tc = -(-shape[-1] // sh.tile_cols)
        regions = ((row % shape[-2]) // sh.tile_rows) * n_tc + col // sh.tile_cols
    return codes, regions
