"""GPU parity of the decode-step additions: online KV quantization (bit-exact
against the reference's quantize() golden codes), attention over a valid prefix of
a KV cache (host and device-resident length, partial 32-token batches), and the
Llama glue kernels against plain fp32 references."""

import numpy as np
import pytest
from conftest import QUANTIZE_CASES, Case, O

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOL_ATTN = 2e-3


@pytest.fixture(scope="module")
def dev():
    return torch.device("cuda", 0)


def _mods():
    from paper_2503_02236_b200 import _native as N
    from paper_2503_02236_b200 import ops
    from paper_2503_02236_b200.device import DeviceVQTensor
    return N, DeviceVQTensor, ops


def _cache(c, dev, layout):
    _, DeviceVQTensor, _ = _mods()
    books = torch.from_numpy(c.books).to(dev).half()
    return DeviceVQTensor.empty_cache(c.shape, c.config(), books, layout=layout)


def _codes(cache):
    plain = cache.relayout("plain")
    cfg = cache.config
    s = int(np.prod(cache.shape)) // cfg.vector_size
    return plain.codes[: cfg.residuals * s].cpu().numpy().reshape(cfg.residuals, s).astype(np.int32)


@pytest.mark.parametrize("name,base,dseed", QUANTIZE_CASES)
def test_cq_quantize_bit_exact(name, base, dseed, dev, arrays):
    N, _, ops = _mods()
    c = Case(base, books_f16=True)
    data = O.round_f16(O.synthetic_tensor(c.shape, dseed))
    layout = "kv" if (c.shape[3] // c.v) in (32, 64) else "plain"
    cache = _cache(c, dev, layout)
    x = torch.from_numpy(data).to(dev).half()
    ops.vq_quantize_kv(cache, x, tok0=0)
    assert N.last_kernel() == "cq_quantize"
    assert np.array_equal(_codes(cache), arrays[f"qz_codes_{name}"])


@pytest.mark.parametrize("name,base,dseed", QUANTIZE_CASES[:2])
def test_cq_quantize_token_by_token(name, base, dseed, dev, arrays):
    """Decode-style appends (one token per call, position read on the device) give
    the same cache as one bulk quantization."""
    _, _, ops = _mods()
    c = Case(base, books_f16=True)
    data = O.round_f16(O.synthetic_tensor(c.shape, dseed))
    cache = _cache(c, dev, "kv")
    x = torch.from_numpy(data).to(dev).half()
    d_len = torch.zeros(1, dtype=torch.int32, device=dev)
    for t in range(c.shape[2]):
        d_len.fill_(t + 1)
        ops.vq_quantize_kv(cache, x[:, :, t:t + 1], d_len=d_len)
    assert np.array_equal(_codes(cache), arrays[f"qz_codes_{name}"])


@pytest.mark.parametrize("T", [1, 17, 32, 100, 511, 513, 1000])
def test_attention_valid_prefix(T, dev):
    """Attention over the first T tokens of a 1024-token cache; T not a multiple of 32
    exercises the masked partial batch. Host length and device length agree."""
    from paper_2503_02236_b200.codec import Codebook, QuantizedTensor, Sharing, VQConfig
    N, DeviceVQTensor, ops = _mods()
    B, H, Tc, C, v = 2, 4, 1024, 128, 2
    cfg = VQConfig(v, 8, 1, Sharing.per_channel_group(v))
    shape = (B, H, Tc, C)
    nreg = O.n_regions_of(shape, v, "channel_group", group_width=v)
    regs = O.region_ids(shape, v, "channel_group", group_width=v)
    kc, kb = O.synthetic_codes_books(shape, v, 8, 1, nreg, 31)
    vc, vb = O.synthetic_codes_books(shape, v, 8, 1, nreg, 32)
    kb, vb = O.round_f16(kb), O.round_f16(vb)

    def qt(codes, books):
        cbs = [Codebook(books[i], 0, i) for i in range(books.shape[0])]
        return QuantizedTensor(codes, shape, cfg, cbs, nreg)

    kd = DeviceVQTensor.from_quantized(qt(kc, kb), device=dev)
    vd = DeviceVQTensor.from_quantized(qt(vc, vb), device=dev)
    q = O.synthetic_tensor((B, H, C), 33)
    kdense = O.dequantize(kc, kb, shape, v, nreg, regs)[:, :, :T]
    vdense = O.dequantize(vc, vb, shape, v, nreg, regs)[:, :, :T]
    ref = O.attention_ref(q, kdense, vdense)
    qt_ = torch.from_numpy(q).to(dev)
    out = ops.vq_attention(kd, vd, qt_, length=T)
    assert N.last_kernel() == "attn_cq"
    assert O.rel_err(out.cpu().numpy(), ref) <= TOL_ATTN
    d_len = torch.full((1,), T, dtype=torch.int32, device=dev)
    out2 = ops.vq_attention(kd, vd, qt_, d_len=d_len)
    assert torch.equal(out, out2)


def test_rmsnorm_rope_silu(dev):
    N, _, ops = _mods()
    g = torch.Generator(device=dev).manual_seed(5)
    B, D = 3, 512
    x = torch.randn(B, D, generator=g, device=dev).half()
    res = torch.randn(B, D, generator=g, device=dev).half()
    w = (1 + 0.1 * torch.randn(D, generator=g, device=dev)).half()
    res0 = res.clone()
    out = ops.rmsnorm(x, res, w, eps=1e-5)
    h = (x.float() + res0.float()).half()
    assert torch.equal(res, h)
    hf = h.float()
    ref = w.float() * (hf * torch.rsqrt(hf.pow(2).mean(-1, keepdim=True) + 1e-5)).half().float()
    assert (out.float() - ref).abs().max().item() <= 2e-3 * ref.abs().max().item()

    H, C = 4, 64
    qkv = torch.randn(B, 3 * H * C, generator=g, device=dev).half()
    orig = qkv.clone()
    d_len = torch.full((1,), 7, dtype=torch.int32, device=dev)
    q = ops.qkv_rope(qkv, H, C, d_len, theta=10000.0)
    pos = 6
    inv = 1.0 / (10000.0 ** (torch.arange(0, C, 2, device=dev).float() / C))
    ang = pos * inv
    cos, sin = torch.cat([ang.cos(), ang.cos()]), torch.cat([ang.sin(), ang.sin()])

    def rope(t):
        t = t.float().view(B, H, C)
        rot = torch.cat([-t[..., C // 2:], t[..., : C // 2]], dim=-1)
        return t * cos + rot * sin

    assert (q.float() - rope(orig[:, : H * C])).abs().max().item() <= 4e-3
    assert (qkv[:, H * C: 2 * H * C].float().view(B, H, C) - rope(orig[:, H * C: 2 * H * C])).abs().max().item() <= 4e-3
    assert torch.equal(qkv[:, 2 * H * C:], orig[:, 2 * H * C:])

    F = 96
    gu = torch.randn(B, 2 * F, generator=g, device=dev).half()
    hmid = ops.silu_mul(gu)
    ref = torch.nn.functional.silu(gu[:, :F].float()) * gu[:, F:].float()
    assert (hmid.float() - ref).abs().max().item() <= 4e-3 * max(1.0, ref.abs().max().item())
