"""ctypes binding of the C ABI in include/vqb.h (libvqb.so, built in-tree).

There is deliberately no fallback: if the shared library is missing every call
raises, so a test or benchmark can never silently run on a CPU path.
"""

import ctypes
import os
import threading

from .errors import (CapacityError, CodeRangeError, ConfigError, ForgeError, KernelError,
                     MappingError, ShapeError)

LIB_NAME = "libvqb.so"
# VQB_LIB_PATH: load another build of the same ABI (A/B timing of kernel revisions)
LIB_PATH = os.environ.get("VQB_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

# status codes / enums (vqb.h)
OK, ESHAPE, ECONFIG, ECODERANGE, ECAPACITY, EMAPPING, ECUDA = 0, -1, -2, -3, -4, -5, -10
F32, F16, BF16 = 0, 1, 2
SHARE = {"whole": 0, "tile": 1, "channel_group": 2}
LAYOUT_PACKED, LAYOUT_GEMV_IL, LAYOUT_KV_IL, LAYOUT_PLAIN = 0, 1, 2, 3
KERNEL_DEQUANT, KERNEL_GEMV, KERNEL_GEMM, KERNEL_ATTN = 0, 1, 2, 3
FLAG_FORCE_GENERIC = 1
FLAG_NO_MMA = 16  # GEMV batch 4-8 on CUDA-core FMAs instead of mma.sync
FLAG_COOPERATIVE = 64
FLAG_NO_PAIR = 128  # GEMM: one-CTA tcgen05 kernel instead of the CTA-pair kernel
FLAG_PAIR_N128 = 256  # GEMM: CTA-pair kernel with 256 x 128 tiles
FLAG_GEMM_FUSED = 512  # GEMM: fused producers at prefill sizes
FLAG_GEMM_TWO_PHASE = 1024  # GEMM: dequantise to an fp16 scratch, then the dense pair GEMM
FLAG_GEMV_TC = 2048  # GEMV: the tcgen05 decode GEMV below its default batch range
FLAG_NO_GEMV_TC = 4096  # GEMV: never the tcgen05 decode GEMV
FLAG_NO_COLSPLIT = 8192  # GEMV batch 1: stream-K instead of the column-split kernel

_ERRORS = {
    ESHAPE: ShapeError,
    ECONFIG: ConfigError,
    ECODERANGE: CodeRangeError,
    ECAPACITY: CapacityError,
    EMAPPING: MappingError,
    ECUDA: KernelError,
}

# every symbol include/vqb.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "vqb_abi_version", "vqb_last_error", "vqb_last_kernel", "vqb_last_launch", "vqb_dequant", "vqb_workspace_bytes", "vqb_gemv",
    "vqb_gemm", "vqb_attn_decode", "vqb_layout_bytes", "vqb_repack", "vqb_query_usage",
    "vqb_debug_smem_base", "vqb_attn_decode_len", "vqb_cq_quantize", "vqb_rmsnorm", "vqb_qkv_rope",
    "vqb_silu_mul", "vqb_add_len", "vqb_qkv_rope_append", "vqb_take_device_error", "vqb_gemv_grouped",
    "vqb_tp_buffer_bytes", "vqb_ipc_get_handle", "vqb_ipc_open_handle", "vqb_ipc_close_handle", "vqb_gemv_tp",
    "vqb_tp_finish", "vqb_tp_take_error", "vqb_gemv_xf", "vqb_attn_decode_append", "vqb_sample",
)
XF_RMSNORM, XF_SILU_MUL, XF_SWIGLU_OUT = 1, 2, 4


class VqbTensor(ctypes.Structure):
    _fields_ = [
        ("vector_size", ctypes.c_int32),
        ("log2_entries", ctypes.c_int32),
        ("residuals", ctypes.c_int32),
        ("sharing", ctypes.c_int32),
        ("tile_rows", ctypes.c_int32),
        ("tile_cols", ctypes.c_int32),
        ("group_width", ctypes.c_int32),
        ("ndim", ctypes.c_int32),
        ("dims", ctypes.c_int64 * 4),
        ("n_regions", ctypes.c_int32),
        ("layout", ctypes.c_int32),
        ("d_codes", ctypes.c_void_p),
        ("codes_bytes", ctypes.c_int64),
        ("codebook_dtype", ctypes.c_int32),
        ("d_codebooks", ctypes.c_void_p),
        ("max_code", ctypes.c_int32),
        ("d_codebooks_t", ctypes.c_void_p),
    ]


class VqbLaunch(ctypes.Structure):
    _fields_ = [
        ("n_reg", ctypes.c_int32),
        ("n_shared", ctypes.c_int32),
        ("split_axis", ctypes.c_int32),
        ("split_factor", ctypes.c_int32),
        ("fusion_level", ctypes.c_int32),
        ("grid_limit", ctypes.c_int32),
        ("flags", ctypes.c_int32),
    ]


TP_MAX_WORLD = 8
TP_ALLREDUCE, TP_ALLGATHER = 0, 1


class VqbPeerComm(ctypes.Structure):
    """include/vqb.h VqbPeerComm: every rank's symmetric buffer as mapped here."""
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("d_peer", ctypes.c_void_p * TP_MAX_WORLD), ("slot_elems", ctypes.c_int64)]


class VqbUsage(ctypes.Structure):
    _fields_ = [
        ("shared_bytes", ctypes.c_int32),
        ("regs_per_thread", ctypes.c_int32),
        ("threads_per_block", ctypes.c_int32),
        ("max_blocks_per_sm", ctypes.c_int32),
        ("sm_count", ctypes.c_int32),
    ]


_lib = None
_lock = threading.Lock()


def lib():
    """Load libvqb.so once; raise (never fall back) if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build the CUDA extension first "
                    "(python -c 'import __graft_entry__ as g; g.build()')")
            L = ctypes.CDLL(LIB_PATH)
            P = ctypes.POINTER
            vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
            T, La = P(VqbTensor), P(VqbLaunch)
            L.vqb_abi_version.restype = ctypes.c_int
            L.vqb_last_error.restype = ctypes.c_char_p
            L.vqb_last_kernel.restype = ctypes.c_char_p
            L.vqb_last_launch.argtypes = [P(i32)]
            L.vqb_dequant.argtypes = [T, vp, i32, vp]
            L.vqb_workspace_bytes.argtypes = [i32, T, i64, La]
            L.vqb_workspace_bytes.restype = i64
            L.vqb_gemv.argtypes = [T, vp, i32, i32, vp, i32, La, vp, sz, vp]
            L.vqb_gemm.argtypes = [T, vp, i32, i32, vp, i32, La, vp, sz, vp]
            L.vqb_gemv_grouped.argtypes = [vp, i32, vp, i32, i32, vp, i32, La, vp, sz, vp]
            L.vqb_attn_decode.argtypes = [T, T, vp, i32, i32, i32, i32, i32, vp, i32, La, vp, sz, vp]
            L.vqb_attn_decode_len.argtypes = [T, T, vp, i32, i32, i32, i32, i32, vp, vp, i32, La, vp, sz, vp]
            f32 = ctypes.c_float
            L.vqb_rmsnorm.argtypes = [vp, vp, vp, vp, i32, i32, f32, vp]
            L.vqb_qkv_rope.argtypes = [vp, vp, i32, i32, i32, vp, f32, vp]
            L.vqb_silu_mul.argtypes = [vp, vp, i32, i32, vp]
            L.vqb_qkv_rope_append.argtypes = [vp, vp, T, T, i32, i32, i32, vp, f32, vp]
            L.vqb_add_len.argtypes = [vp, i32, vp]
            L.vqb_sample.argtypes = [vp, i32, i32, i32, f32, i32, f32, ctypes.c_uint64, vp, vp, vp]
            L.vqb_take_device_error.argtypes = [P(i32)]
            L.vqb_cq_quantize.argtypes = [T, vp, i32, i64, i64, i64, i32, i32, vp, vp]
            L.vqb_layout_bytes.argtypes = [T, i32]
            L.vqb_layout_bytes.restype = i64
            L.vqb_repack.argtypes = [T, i32, vp, i64, vp]
            L.vqb_query_usage.argtypes = [i32, T, P(VqbUsage)]
            C = P(VqbPeerComm)
            L.vqb_tp_buffer_bytes.argtypes = [i32, i64]
            L.vqb_tp_buffer_bytes.restype = i64
            L.vqb_ipc_get_handle.argtypes = [vp, vp, P(i64)]
            L.vqb_ipc_open_handle.argtypes = [vp, i64, P(vp)]
            L.vqb_ipc_close_handle.argtypes = [vp]
            L.vqb_gemv_tp.argtypes = [T, vp, i32, i32, i32, C, La, vp, sz, vp]
            L.vqb_gemv_xf.argtypes = [T, vp, i32, i32, vp, vp, vp, f32, vp, i32, La, vp, sz, vp]
            L.vqb_attn_decode_append.argtypes = [T, T, vp, i32, i32, i32, vp, f32, vp, i32, La, vp, sz, vp]
            L.vqb_tp_finish.argtypes = [C, i32, i32, i32, vp, i32, vp]
            L.vqb_tp_take_error.argtypes = [C, P(i32)]
            L.vqb_debug_smem_base.argtypes = [vp, vp]
            L.vqb_debug_smem_base.restype = ctypes.c_int
            for name in ("vqb_dequant", "vqb_gemv", "vqb_gemm", "vqb_attn_decode", "vqb_repack",
                         "vqb_query_usage", "vqb_attn_decode_len", "vqb_rmsnorm", "vqb_qkv_rope",
                         "vqb_silu_mul", "vqb_add_len", "vqb_cq_quantize", "vqb_qkv_rope_append",
                         "vqb_take_device_error", "vqb_gemv_grouped", "vqb_ipc_get_handle",
                         "vqb_ipc_open_handle", "vqb_ipc_close_handle", "vqb_gemv_tp", "vqb_tp_finish",
                         "vqb_tp_take_error", "vqb_gemv_xf", "vqb_attn_decode_append", "vqb_sample"):
                getattr(L, name).restype = ctypes.c_int
            _lib = L
    return _lib


def last_error() -> str:
    msg = lib().vqb_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def last_kernel() -> str:
    """Name of the last kernel launched by this thread (proves which path ran)."""
    k = lib().vqb_last_kernel()
    return k.decode() if k else ""


def take_device_error() -> int:
    """Read and clear the device error word (bit 0: a KV append out of capacity)."""
    v = ctypes.c_int32(0)
    check(lib().vqb_take_device_error(ctypes.byref(v)))
    return int(v.value)


def last_launch() -> dict:
    """grid / threads / shared-tier / register-tier entries of the last fused launch."""
    out = (ctypes.c_int32 * 4)()
    lib().vqb_last_launch(out)
    return {"grid": out[0], "threads": out[1], "n_shared": out[2], "n_reg": out[3]}


def check(status: int) -> int:
    """Raise the exception class the status maps to; return non-negative values."""
    if status >= 0:
        return status
    cls = _ERRORS.get(int(status), ForgeError)
    raise cls(last_error() or f"vqb status {status}")
