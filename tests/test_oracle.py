"""Pin the CPU oracle against golden vectors produced by the real reference."""

import hashlib

import numpy as np
import pytest
from conftest import ATTENTION_CASES, CASES, MATMUL_CASES, QUANTIZE_CASES, Case, O


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", sorted(CASES))
def test_synth_reproduces_reference_inputs(name, meta):
    c = Case(name)
    g = meta["dequant"][name]
    assert c.n_regions == g["n_regions"]
    assert sha(c.codes) == g["codes_sha"]
    assert sha(c.books) == g["books_sha"]
    assert sha(c.regions.astype(np.int64)) == g["region_sha"]


@pytest.mark.parametrize("name", sorted(CASES))
def test_dequant_bit_exact(name, meta, arrays):
    c = Case(name)
    out = c.dense()
    assert out.dtype == np.float32 and out.shape == c.shape
    assert sha(out) == meta["dequant"][name]["dequant_sha"]
    idx = arrays[f"deq_idx_{name}"]
    assert np.array_equal(out.reshape(-1)[idx], arrays[f"deq_val_{name}"])
    c16 = Case(name, books_f16=True)
    assert sha(c16.dense()) == meta["dequant"][name]["dequant16_sha"]


@pytest.mark.parametrize("name,base,kind,extra", MATMUL_CASES)
def test_matmul_oracle(name, base, kind, extra, arrays):
    c = Case(name=base)
    m = c.shape[0]
    act = O.synthetic_tensor((m,) if kind == "gemv" else (extra["rows"], m), c.seed + 2)
    ref = O.matmul_ref(act, c.dense())
    assert O.rel_err(ref, arrays[f"mm_ref_{name}"]) <= 1e-6
    # the reference's own fused template agrees within its 1e-4 contract
    assert O.rel_err(arrays[f"mm_sim_{name}"], ref) <= 1e-4


@pytest.mark.parametrize("name,base", ATTENTION_CASES)
def test_attention_oracle(name, base, meta, arrays):
    k = Case(base)
    v = Case(base, seed_offset=1)
    assert sha(v.codes) == meta["attention"][name]["v_codes_sha"]
    b, h, t, ch = k.shape
    q = O.synthetic_tensor((b, h, ch), k.seed + 2)
    assert sha(q) == meta["attention"][name]["query_sha"]
    ref = O.attention_ref(q, k.dense(), v.dense())
    assert O.rel_err(ref, arrays[f"at_ref_{name}"]) <= 1e-6
    assert O.rel_err(arrays[f"at_sim_{name}"], ref) <= 1e-4


def test_attention_known_answers():
    # T = 1: softmax weight is 1, output is the V row (T/test_sim.py:91-98)
    k = np.ones((1, 1, 1, 4), np.float32)
    v = np.arange(4, dtype=np.float32).reshape(1, 1, 1, 4)
    q = np.ones((1, 1, 4), np.float32)
    assert np.allclose(O.attention_ref(q, k, v)[0, 0], v[0, 0, 0])
    # [[1,2]] @ [[3,0],[4,1]] = [[11,2]] (T/test_sim.py:85-90)
    out = O.matmul_ref(np.array([[1.0, 2.0]], np.float32), np.array([[3, 0], [4, 1]], np.float32))
    assert out.tolist() == [[11.0, 2.0]]


def test_dequant_signed_zero_becomes_positive():
    books = np.array([[[-0.0, 1.0], [2.0, -0.0]]], np.float32)
    codes = np.array([[0, 1]], np.int32)
    out = O.dequantize(codes, books, (1, 4), 2, 1, np.zeros(2, np.int64))
    assert not np.signbit(out).any()


@pytest.mark.parametrize("name,base,dseed", QUANTIZE_CASES)
def test_quantize_matches_reference(name, base, dseed, meta, arrays):
    """Online KV quantization oracle vs the reference's quantize() (fp16-rounded books)."""
    c = Case(base, books_f16=True)
    data = O.round_f16(O.synthetic_tensor(c.shape, dseed))
    assert sha(data) == meta["quantize"][name]["data_sha"]
    codes = O.quantize(data, c.books, c.shape, c.v, c.n_regions, c.regions, c.R)
    assert np.array_equal(codes, arrays[f"qz_codes_{name}"])
