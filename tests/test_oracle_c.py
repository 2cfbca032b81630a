"""The C (OpenMP) oracle agrees with the numpy oracle: bit-exact dequantization,
reference tolerance for the dense ops."""

import hashlib

import numpy as np
import pytest
from conftest import ATTENTION_CASES, CASES, Case, O

from oracle import c_oracle as C


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", sorted(CASES))
def test_c_dequant_bit_exact(name, meta):
    c = Case(name)
    out = C.dequantize(c.codes, c.books, c.shape, c.v, c.n_regions, c.regions)
    assert sha(out) == meta["dequant"][name]["dequant_sha"]


@pytest.mark.parametrize("name", ["gptvq2", "quip2", "aqlm2x8", "aqlm3"])
def test_c_gemv(name):
    c = Case(name)
    x = O.synthetic_tensor((3, c.shape[0]), 4)
    y = C.gemv(c.codes, c.books, c.shape, c.v, c.n_regions, c.regions, x)
    assert O.rel_err(y, O.matmul_ref(x, c.dense())) <= 1e-5


@pytest.mark.parametrize("name,base", ATTENTION_CASES)
def test_c_attention(name, base, arrays):
    k, v = Case(base), Case(base, seed_offset=1)
    b, h, t, ch = k.shape
    q = O.synthetic_tensor((b, h, ch), k.seed + 2)
    out = C.attention(q, k.dense(), v.dense())
    assert O.rel_err(out, arrays[f"at_ref_{name}"]) <= 1e-5


def test_c_code_range():
    c = Case("cq2")
    codes = c.codes.copy()
    codes[0, 5] = 999
    with pytest.raises(ValueError, match="code out of range"):
        C.dequantize(codes, c.books, c.shape, c.v, c.n_regions, c.regions)
