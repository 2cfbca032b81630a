"""Parity at the BASELINE configs' full sizes, where the CPU oracle would take
minutes: the reference for a fused op is the GPU's dequantization (bit-exact with
the reference, proven on the golden cases) followed by a plain fp32 torch matmul /
attention; plus size-independent properties (linearity, determinism, quantize ->
dequantize round trips)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    return torch.device("cuda", 0)


def _mods():
    from paper_2503_02236_b200 import _native as N
    from paper_2503_02236_b200 import ops
    from paper_2503_02236_b200.codec import Sharing, VQConfig, region_count
    from paper_2503_02236_b200.device import DeviceVQTensor
    return N, ops, Sharing, VQConfig, region_count, DeviceVQTensor


def _weight(dev, shape, v, bits, r, sharing, work=None, seed=0):
    N, ops, Sharing, VQConfig, region_count, DeviceVQTensor = _mods()
    sh = Sharing.per_tile(256, 256) if sharing == "tile" else Sharing.whole_tensor()
    cfg = VQConfig(v, bits, r, sh)
    g = torch.Generator(device=dev).manual_seed(seed)
    m, n = shape
    nreg = region_count(shape, cfg)
    codes = torch.randint(0, work or cfg.n_entries, (r, m * n // v), generator=g, device=dev, dtype=torch.int32)
    books = (torch.randn((r * nreg, cfg.n_entries, v), generator=g, device=dev) * 0.1).half()
    return DeviceVQTensor.from_device_codes(codes, shape, cfg, books).relayout("gemv")


def _rel(a, b):
    return ((a.float() - b.float()).abs().max() / b.float().abs().max()).item()


FULL_GEMV = [
    ("C1 gptvq2 q_proj", (4096, 4096), 4, 8, 1, "tile", None),
    ("C2 quip2 qkv", (4096, 12288), 8, 16, 1, "whole", 256),
    ("C2 quip2 down", (11008, 4096), 8, 16, 1, "whole", 256),
    ("C3 aqlm2x8 65B q", (8192, 8192), 8, 8, 2, "whole", None),
]


@pytest.mark.parametrize("label,shape,v,bits,r,sharing,work", FULL_GEMV)
def test_full_size_gemv(label, shape, v, bits, r, sharing, work, dev):
    N, ops, *_ = _mods()
    w = _weight(dev, shape, v, bits, r, sharing, work)
    dense = ops.vq_dequantize(w)  # fp32, bit-exact
    g = torch.Generator(device=dev).manual_seed(1)
    x = torch.randn((1, shape[0]), generator=g, device=dev).half()
    y = ops.vq_gemv(w, x, out_dtype=torch.float32)
    assert N.last_kernel() in ("gemv_fast", "gemv_cs")  # column-split for 16-block outputs
    ref = x.float() @ dense
    assert _rel(y, ref) <= 1e-3, label
    # determinism of the split reduction and linearity in the activation
    assert torch.equal(y, ops.vq_gemv(w, x, out_dtype=torch.float32))
    x2 = torch.randn((1, shape[0]), generator=g, device=dev).half()
    y2 = ops.vq_gemv(w, x2, out_dtype=torch.float32)
    y12 = ops.vq_gemv(w, (x.float() + x2.float()).half(), out_dtype=torch.float32)
    assert _rel(y12, (x.float() + x2.float()).half().float() @ dense) <= 1e-3
    assert _rel(y + y2, y12) <= 2e-3


@pytest.mark.parametrize("rows,n", [(16, 12288), (1024, 12288), (16, 22016), (64, 22016), (1024, 4096)])
def test_full_size_gemm(rows, n, dev):
    """qkv and gate_up shapes: split-K below one wave of tiles (96 tiles) and between
    one and two waves (172 tiles), no split at prefill size."""
    N, ops, *_ = _mods()
    w = _weight(dev, (4096, n), 8, 16, 1, "whole", 256, seed=2)
    dense = ops.vq_dequantize(w)
    g = torch.Generator(device=dev).manual_seed(3)
    x = torch.randn((rows, 4096), generator=g, device=dev).half()
    y = ops.vq_gemm(w, x, out_dtype=torch.float32)
    assert N.last_kernel() == ("gemm_tc2" if rows > 256 and n % 256 == 0 else "gemm_tc")
    ref = x.float() @ dense.half().float()  # the tensor cores consume the fp16-rounded W
    assert _rel(y, ref) <= 2e-3


def test_full_size_attention_c4(dev):
    """C4: CQ-4 KV cache, B16 H32 T4096 C128, against fp32 attention over the
    bit-exact dequantized cache."""
    N, ops, Sharing, VQConfig, region_count, DeviceVQTensor = _mods()
    B, H, T, C = 16, 32, 4096, 128
    cfg = VQConfig(2, 8, 1, Sharing.per_channel_group(2))
    g = torch.Generator(device=dev).manual_seed(4)
    kv = []
    for _ in range(2):
        codes = torch.randint(0, 256, (1, B * H * T * C // 2), generator=g, device=dev, dtype=torch.int32)
        books = (torch.randn((H * 64, 256, 2), generator=g, device=dev) * 0.1).half()
        kv.append(DeviceVQTensor.from_device_codes(codes, (B, H, T, C), cfg, books).relayout("kv"))
    q = torch.randn((B, H, C), generator=g, device=dev).half()
    out = ops.vq_attention(kv[0], kv[1], q, out_dtype=torch.float32)
    assert N.last_kernel() == "attn_cq"
    k = ops.vq_dequantize(kv[0])
    v = ops.vq_dequantize(kv[1])
    logits = torch.einsum("bhc,bhtc->bht", q.float(), k) / C ** 0.5
    ref = torch.einsum("bht,bhtc->bhc", torch.softmax(logits, -1), v)
    assert _rel(out, ref) <= 2e-3
    assert torch.equal(out, ops.vq_attention(kv[0], kv[1], q, out_dtype=torch.float32))


def test_quantize_dequantize_round_trip_full_cache(dev):
    """Rows that are codebook entries quantize to codes whose dequantization gives
    the rows back (a full C4-sized layer cache, 134M sub-vectors per tensor)."""
    N, ops, Sharing, VQConfig, region_count, DeviceVQTensor = _mods()
    B, H, T, C = 16, 32, 4096, 128
    cfg = VQConfig(2, 8, 1, Sharing.per_channel_group(2))
    g = torch.Generator(device=dev).manual_seed(5)
    codes = torch.randint(0, 256, (1, B * H * T * C // 2), generator=g, device=dev, dtype=torch.int32)
    books = torch.randn((H * 64, 256, 2), generator=g, device=dev).half()
    src = DeviceVQTensor.from_device_codes(codes, (B, H, T, C), cfg, books).relayout("kv")
    rows = ops.vq_dequantize(src)
    cache = DeviceVQTensor.empty_cache((B, H, T, C), cfg, books)
    ops.vq_quantize_kv(cache, rows.half(), tok0=0)
    back = ops.vq_dequantize(cache)
    assert torch.equal(back, rows)
