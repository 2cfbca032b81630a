"""ctypes wrapper of oracle/liboracle.so — TEST INFRASTRUCTURE / CPU BASELINE ONLY.

Built by __graft_entry__.build() (gcc -O2 -fopenmp). Used by tests/test_oracle_c.py
(cross-check against the numpy oracle) and by bench.py's CPU legs.
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "vq_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")
_lib = None


def build():
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", LIB, SRC, "-lm"], check=True)


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        P = ctypes.c_void_p
        L.vqo_threads.restype = ctypes.c_int
        L.vqo_set_threads.argtypes = [ctypes.c_int]
        L.vqo_dequant.argtypes = [P, ctypes.c_int, ctypes.c_int64, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P]
        L.vqo_gemv.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, ctypes.c_int,
                               ctypes.c_int, P, P, ctypes.c_int, P]
        L.vqo_attention.argtypes = [P, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def threads() -> int:
    return int(lib().vqo_threads())


def set_threads(n: int) -> None:
    lib().vqo_set_threads(int(n))


def dequantize(codes, books, shape, v, n_regions, regions):
    codes = np.ascontiguousarray(codes, np.int32)
    books = np.ascontiguousarray(books, np.float32)
    regions = np.ascontiguousarray(regions, np.int32)
    out = np.empty(int(np.prod(shape)), np.float32)
    st = lib().vqo_dequant(_p(codes), codes.shape[0], codes.shape[1], _p(books), books.shape[1], v, n_regions,
                           _p(regions), _p(out))
    if st:
        raise ValueError("code out of range")
    return out.reshape(shape)


def gemv(codes, books, shape, v, n_regions, regions, x):
    codes = np.ascontiguousarray(codes, np.int32)
    books = np.ascontiguousarray(books, np.float32)
    regions = np.ascontiguousarray(regions, np.int32)
    x2 = np.ascontiguousarray(np.atleast_2d(x), np.float32)
    m, n = shape
    y = np.empty((x2.shape[0], n), np.float32)
    st = lib().vqo_gemv(_p(codes), codes.shape[0], m, n, v, _p(books), books.shape[1], n_regions, _p(regions),
                        _p(x2), x2.shape[0], _p(y))
    if st:
        raise ValueError(f"vqo_gemv status {st}")
    return y[0] if np.ndim(x) == 1 else y


def attention(q, k, v):
    q = np.ascontiguousarray(q, np.float32)
    k = np.ascontiguousarray(k, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    b, h, t, c = k.shape
    out = np.empty((b, h, c), np.float32)
    lib().vqo_attention(_p(q), _p(k), _p(v), b, h, t, c, _p(out))
    return out
