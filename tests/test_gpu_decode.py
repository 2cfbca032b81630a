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


# ---- end-to-end decode (C5) against a numpy restatement of the same model ------------------------

def _tiny_model(dev, batch, capacity):
    from paper_2503_02236_b200.codec import Codebook, QuantizedTensor
    from paper_2503_02236_b200.decode import KV_CFG, WEIGHT_CFG, DecoderLayer, LlamaShape, VQLlamaDecoder
    _, DeviceVQTensor, _ = _mods()
    sh = LlamaShape(hidden=256, heads=4, head_dim=64, ffn=512, layers=2, vocab=512)
    d, f = sh.hidden, sh.ffn
    rng = np.random.default_rng(0)
    host = {}

    def weight(name, m, n, seed):
        codes, books = O.synthetic_codes_books((m, n), 8, 16, 1, 1, seed, working_entries=256)
        books = O.round_f16(books * (0.5 / m ** 0.5 / 0.1))
        q = QuantizedTensor(codes, (m, n), WEIGHT_CFG, [Codebook(books[0], 0, 0)], 1)
        host[name] = O.dequantize(codes, books, (m, n), 8, 1, np.zeros(m * n // 8, np.int64))
        return DeviceVQTensor.from_quantized(q, device=dev)

    layers, kv_books = [], []
    for li in range(sh.layers):
        kb = O.round_f16(rng.standard_normal((sh.heads * sh.head_dim // 2, 256, 2)).astype(np.float32))
        vb = O.round_f16(rng.standard_normal((sh.heads * sh.head_dim // 2, 256, 2)).astype(np.float32))
        kv_books.append((kb, vb))
        cache = lambda books: DeviceVQTensor.empty_cache((batch, sh.heads, capacity, sh.head_dim), KV_CFG,
                                                         torch.from_numpy(books).to(dev).half())
        an = O.round_f16(1 + 0.1 * rng.standard_normal(d).astype(np.float32))
        fn = O.round_f16(1 + 0.1 * rng.standard_normal(d).astype(np.float32))
        host[f"an{li}"], host[f"fn{li}"] = an, fn
        layers.append(DecoderLayer(weight(f"qkv{li}", d, 3 * d, 100 + li), weight(f"o{li}", d, d, 200 + li),
                                   weight(f"gu{li}", d, 2 * f, 300 + li), weight(f"down{li}", f, d, 400 + li),
                                   torch.from_numpy(an).to(dev).half(), torch.from_numpy(fn).to(dev).half(),
                                   cache(kb), cache(vb)))
    embed = O.round_f16(rng.standard_normal((sh.vocab, d)).astype(np.float32))
    head = O.round_f16((rng.standard_normal((d, sh.vocab)) / d ** 0.5).astype(np.float32))
    fin = O.round_f16(1 + 0.1 * rng.standard_normal(d).astype(np.float32))
    host.update(embed=embed, head=head, fin=fin, kv_books=kv_books)
    dec = VQLlamaDecoder(sh, layers, torch.from_numpy(embed).to(dev).half(), torch.from_numpy(fin).to(dev).half(),
                         torch.from_numpy(head).to(dev).half(), batch)
    return sh, dec, host


def _np_decode(sh, host, tokens, steps, capacity):
    """fp32 restatement of VQLlamaDecoder.step with fp16 rounding where the device
    stores fp16 tensors; KV rows quantized with the oracle's quantize (nearest)."""
    r16 = O.round_f16
    b = len(tokens)
    d, hh, c, f = sh.hidden, sh.heads, sh.head_dim, sh.ffn
    kv_codes = [[[] for _ in range(2)] for _ in range(sh.layers)]  # per layer: K/V rows (b, h, t, c) dense
    toks, logits_all = np.array(tokens), []

    def rms(x, w):
        x = x.astype(np.float32)
        inv = 1.0 / np.sqrt((x * x).mean(-1, keepdims=True) + sh.eps)
        return r16(w * r16(x * inv))

    def nearest_rows(rows, books):  # rows (b, h, c) -> dequantized via nearest entry per group
        out = np.empty_like(rows)
        for hi in range(hh):
            for gi in range(c // 2):
                bk = books[hi * (c // 2) + gi]
                idx = O.nearest(rows[:, hi, 2 * gi:2 * gi + 2], bk)
                out[:, hi, 2 * gi:2 * gi + 2] = bk[idx]
        return out

    for t in range(steps):
        pos = t
        inv_freq = 1.0 / (sh.rope_theta ** (np.arange(0, c, 2, dtype=np.float32) / c))
        ang = pos * inv_freq
        cos, sin = np.cos(ang), np.sin(ang)
        res = host["embed"][toks].astype(np.float32)
        x = None
        for li in range(sh.layers):
            if x is not None:
                res = r16(res + x)
            xn = rms(res, host[f"an{li}"])
            qkv = r16(xn @ host[f"qkv{li}"]).reshape(b, 3, hh, c)

            def rope(v):
                v0, v1 = v[..., : c // 2], v[..., c // 2:]
                return r16(np.concatenate([v0 * cos - v1 * sin, v1 * cos + v0 * sin], -1))

            q, k, v = rope(qkv[:, 0]), rope(qkv[:, 1]), qkv[:, 2]
            kb, vb = host["kv_books"][li]
            kv_codes[li][0].append(nearest_rows(k, kb))
            kv_codes[li][1].append(nearest_rows(v, vb))
            kd = np.stack(kv_codes[li][0], axis=2)
            vd = np.stack(kv_codes[li][1], axis=2)
            a = r16(O.attention_ref(q, kd, vd)).reshape(b, d)
            o = r16(a @ host[f"o{li}"])
            res = r16(res + o)
            xn = rms(res, host[f"fn{li}"])
            gu = r16(xn @ host[f"gu{li}"])
            s = r16(gu[:, :f] / (1 + np.exp(-gu[:, :f])))
            x = r16(r16(s * gu[:, f:]) @ host[f"down{li}"])
        res = r16(res + x)
        logits = rms(res, host["fin"]) @ host["head"]
        logits_all.append(logits)
        toks = logits.argmax(-1)
    return logits_all


@pytest.mark.parametrize("batch", [1, 2, 4, 8, 16, 24])  # 4-8: mma.sync GEMV, 16-24: tcgen05 GEMV
def test_decode_matches_numpy_model(batch, dev):
    capacity, steps = 64, 6
    sh, dec, host = _tiny_model(dev, batch, capacity)
    tokens = list(range(3, 3 + batch))
    dec.tokens.copy_(torch.tensor(tokens, device=dev))
    ref = _np_decode(sh, host, tokens, steps, capacity)
    for t in range(steps):
        dec.step()
        got = dec.logits.float().cpu().numpy()
        assert O.rel_err(got, ref[t]) <= 3e-2, (t, O.rel_err(got, ref[t]))
        assert int(dec.d_len.item()) == t + 1


def test_decode_graph_replay_matches_eager(dev):
    capacity, steps = 64, 5
    sh, dec, host = _tiny_model(dev, 1, capacity)
    dec.tokens.fill_(7)
    eager = []
    for _ in range(steps):
        dec.step()
        eager.append(dec.logits.float().clone())
    sh2, dec2, _ = _tiny_model(dev, 1, capacity)
    dec2.tokens.fill_(7)
    dec2.capture()
    for t in range(steps):
        dec2.replay()
        assert torch.equal(dec2.logits.float(), eager[t]), t
    assert int(dec2.d_len.item()) == steps


@pytest.mark.parametrize("B", [2, 5, 16, 64])  # lanes per row 16 / 4 / 2 / 1 (two passes)
def test_qkv_rope_append_matches_separate_kernels(B, dev):
    """The fused front end (rope + K/V quantization in one launch) writes the same
    codes and q as qkv_rope followed by two vq_quantize_kv calls."""
    from paper_2503_02236_b200.decode import KV_CFG
    _, DeviceVQTensor, ops = _mods()
    H, C, T = 4, 128, 64
    g = torch.Generator(device=dev).manual_seed(9)
    books = [torch.randn((H * C // 2, 256, 2), generator=g, device=dev).half() for _ in range(2)]
    caches = [[DeviceVQTensor.empty_cache((B, H, T, C), KV_CFG, bk) for bk in books] for _ in range(2)]
    d_len = torch.full((1,), 37, dtype=torch.int32, device=dev)
    qkv = torch.randn((B, 3 * H * C), generator=g, device=dev).half()
    q1 = ops.qkv_rope_append(qkv.clone(), caches[0][0], caches[0][1], d_len)
    qkv2 = qkv.clone()
    q2 = ops.qkv_rope(qkv2, H, C, d_len)
    kv = qkv2.view(B, 3, H, 1, C)
    ops.vq_quantize_kv(caches[1][0], kv[:, 1], d_len=d_len)
    ops.vq_quantize_kv(caches[1][1], kv[:, 2], d_len=d_len)
    assert torch.equal(q1, q2)
    for i in range(2):
        assert torch.equal(caches[0][i].codes, caches[1][i].codes)


@pytest.mark.parametrize("mode", ["bulk", "token"])
def test_cq_quantize_near_ties(mode, dev):
    """Adversarial KV rows for the nearest-centroid screen (V/codec.py:239-253):
    fp16 midpoints of two entries (exact float64 ties -> lowest index), midpoints
    nudged by one fp16 ulp either way, rows equal to a duplicated entry, and rows a
    hair away from an entry. Codes must equal the float64 oracle bit for bit."""
    N, DeviceVQTensor, ops = _mods()
    from paper_2503_02236_b200.codec import Sharing, VQConfig
    B, H, T, C, v = 2, 4, 64, 128, 2
    G = C // v
    rng = np.random.default_rng(123)
    books = O.round_f16(rng.normal(0, 1, (H * G, 256, v)).astype(np.float32))
    books[:, 200] = books[:, 17]  # exact duplicates: the lower index must win
    pts = np.empty((B, H, T, G, v), np.float32)
    for h in range(H):
        for g in range(G):
            bk = books[h * G + g]
            for b in range(B):
                for t in range(T):
                    kind = (b * T + t + g) % 5
                    i, j = rng.choice(256, 2, replace=False)
                    if kind == 0:
                        p = (bk[i].astype(np.float64) + bk[j]) / 2
                    elif kind in (1, 2):
                        p = np.nextafter(((bk[i] + bk[j]) / 2).astype(np.float16),
                                         np.float16(np.inf if kind == 1 else -np.inf)).astype(np.float64)
                    elif kind == 3:
                        p = bk[17].astype(np.float64)
                    else:
                        p = np.nextafter(bk[i].astype(np.float16), np.float16(np.inf)).astype(np.float64)
                    pts[b, h, t, g] = p
    data = O.round_f16(pts.reshape(B, H, T, C))
    regions = O.region_ids((B, H, T, C), v, "channel_group", group_width=v)
    ref = O.quantize(data, books, (B, H, T, C), v, H * G, regions, 1)
    cfg = VQConfig(v, 8, 1, Sharing.per_channel_group(v))
    cache = DeviceVQTensor.empty_cache((B, H, T, C), cfg, torch.from_numpy(books).to(dev).half())
    x = torch.from_numpy(data).to(dev).half()
    if mode == "bulk":
        ops.vq_quantize_kv(cache, x, tok0=0)
    else:
        d_len = torch.zeros(1, dtype=torch.int32, device=dev)
        for t in range(T):
            d_len.fill_(t + 1)
            ops.vq_quantize_kv(cache, x[:, :, t:t + 1], d_len=d_len)
    got = _codes(cache)
    assert np.array_equal(got, ref), int((got != ref).sum())


def test_fused_norm_and_silu_gemv_match_separate_kernels(dev):
    """vqb_gemv_xf: the RMSNorm (with residual add) and the SiLU gate computed in the
    GEMV prologue give bit-identical results to rmsnorm/silu_mul + vq_gemv."""
    N, DeviceVQTensor, ops = _mods()
    from paper_2503_02236_b200.decode import WEIGHT_CFG
    g = torch.Generator(device=dev).manual_seed(17)

    def weight(m, n):
        codes = torch.randint(0, 256, (1, m * n // 8), generator=g, device=dev, dtype=torch.int32)
        books = (torch.randn((1, 65536, 8), generator=g, device=dev) * 0.05).half()
        return DeviceVQTensor.from_device_codes(codes, (m, n), WEIGHT_CFG, books).relayout("gemv")

    for m, n in ((4096, 12288), (1024, 768)):
        w = weight(m, n)
        res = torch.randn((1, m), generator=g, device=dev).half()
        x = torch.randn((1, m), generator=g, device=dev).half()
        nw = (1 + 0.1 * torch.randn(m, generator=g, device=dev)).half()
        for add in (x, None):
            r1 = res.clone()
            xn = ops.rmsnorm(add, r1, nw, 1e-5)
            ref = ops.vq_gemv(w, xn, out_dtype=torch.float16)
            r_out = torch.empty_like(res)
            y = ops.vq_gemv_rmsnorm(w, add, res, nw, 1e-5, residual_out=r_out)
            assert N.last_kernel() == "gemv_rmsnorm"
            assert torch.equal(y, ref) and torch.equal(r_out, r1)
        gu = torch.randn((1, 2 * m), generator=g, device=dev).half()
        ref = ops.vq_gemv(w, ops.silu_mul(gu), out_dtype=torch.float16)
        y = ops.vq_gemv_silu(w, gu)
        assert N.last_kernel() == "gemv_silu"
        assert torch.equal(y, ref)


def test_fused_decode_step_bit_identical(dev):
    """The batch-1 decode step with the norms / SiLU fused into the GEMVs produces
    the unfused step's logits bit for bit, eagerly and as a replayed CUDA graph."""
    from paper_2503_02236_b200.decode import LlamaShape, VQLlamaDecoder
    sh = LlamaShape(hidden=512, heads=4, head_dim=128, ffn=1024, layers=2, vocab=256)
    a = VQLlamaDecoder.synthetic(sh, 1, 64, dev, seed=8)
    b = VQLlamaDecoder.synthetic(sh, 1, 64, dev, seed=8)
    b.fuse_norms = False
    for d in (a, b):
        d.tokens.fill_(7)
    for _ in range(3):
        a.run_step()
        b.run_step()
        assert torch.equal(a.logits, b.logits)
    a.capture()
    b.capture()
    for _ in range(3):
        a.replay()
        b.replay()
        assert torch.equal(a.logits, b.logits)


@pytest.mark.parametrize("batch", [1, 3, 8])
def test_fused_append_attention_bit_identical(batch, dev):
    """vqb_attn_decode_append (RoPE + KV append inside the attention kernel) gives the
    two-kernel step's logits and KV-cache codes bit for bit, eagerly and replayed."""
    from paper_2503_02236_b200.decode import LlamaShape, VQLlamaDecoder
    sh = LlamaShape(hidden=512, heads=4, head_dim=128, ffn=1024, layers=2, vocab=256)
    a = VQLlamaDecoder.synthetic(sh, batch, 96, dev, seed=12)
    b = VQLlamaDecoder.synthetic(sh, batch, 96, dev, seed=12)
    b.fuse_append = False
    for d in (a, b):
        d.tokens.copy_(torch.arange(5, 5 + batch, device=dev))
        d.set_length(29)  # the new tokens cross a 32-token batch boundary
    from paper_2503_02236_b200 import _native as N
    for _ in range(4):
        a.run_step()
        assert N.last_kernel() != "qkv_rope_append"
        b.run_step()
        assert torch.equal(a.logits, b.logits)
    for La, Lb in zip(a.layers, b.layers):
        assert torch.equal(La.k_cache.codes, Lb.k_cache.codes) and torch.equal(La.v_cache.codes, Lb.v_cache.codes)
    a.capture()
    b.capture()
    for _ in range(3):
        a.replay()
        b.replay()
        assert torch.equal(a.logits, b.logits)


def test_swiglu_epilogue_matches_separate_kernels(dev):
    """VQB_XF_SWIGLU_OUT: the gate_up GEMV stored [gate 128 | up 128] per 256-column
    block emits silu(gate) * up from its epilogue — bit-identical to the fp16 gate_up
    output followed by silu_mul, whole and split column blocks alike."""
    N, DeviceVQTensor, ops = _mods()
    from paper_2503_02236_b200.decode import WEIGHT_CFG
    g = torch.Generator(device=dev).manual_seed(23)
    for m, n in ((4096, 22016), (512, 1024)):
        codes = torch.randint(0, 256, (1, m * n // 8), generator=g, device=dev, dtype=torch.int32)
        books = (torch.randn((1, 65536, 8), generator=g, device=dev) * 0.05).half()
        w = DeviceVQTensor.from_device_codes(codes, (m, n), WEIGHT_CFG, books).relayout("gemv")
        res = torch.randn((1, m), generator=g, device=dev).half()
        x = torch.randn((1, m), generator=g, device=dev).half()
        nw = (1 + 0.1 * torch.randn(m, generator=g, device=dev)).half()
        r_a, r_b = torch.empty_like(res), torch.empty_like(res)
        gu = ops.vq_gemv_rmsnorm(w, x, res, nw, 1e-5, residual_out=r_a)
        gu = gu.view(1, n // 256, 2, 128).permute(0, 2, 1, 3).reshape(1, n).contiguous()
        ref = ops.silu_mul(gu)
        h = ops.vq_gemv_rmsnorm(w, x, res, nw, 1e-5, residual_out=r_b, swiglu=True)
        assert h.shape == (1, n // 2)
        assert torch.equal(h, ref) and torch.equal(r_a, r_b)


def test_decode_sampling_replay_matches_eager(dev):
    """Temperature / top-k sampling inside the decode step: a replayed graph draws
    the eager step's tokens (the noise is keyed on the device length), every token is
    in the top-k set of its logits, and the draw is the oracle's Gumbel-max choice."""
    from oracle import sample_oracle as SO
    from paper_2503_02236_b200.decode import LlamaShape, VQLlamaDecoder
    sh = LlamaShape(hidden=512, heads=4, head_dim=128, ffn=1024, layers=2, vocab=256)
    a = VQLlamaDecoder.synthetic(sh, 4, 64, dev, seed=8)
    b = VQLlamaDecoder.synthetic(sh, 4, 64, dev, seed=8)
    for d in (a, b):
        d.set_sampling(temperature=0.8, top_k=20, seed=77, top_p=0.9)
        d.tokens.fill_(7)
    b.capture()
    for _ in range(4):
        tok = a.run_step().clone()
        b.replay()
        assert torch.equal(tok, b.tokens)
        lg = a.logits.float().cpu().numpy()
        sc = SO.scores(lg, 0.8, 20, 77, int(a.d_len.item()), top_p=0.9 + 2e-3)
        t = tok.cpu().numpy()
        got = sc[np.arange(4), t]
        assert np.all(np.isfinite(got)) and np.all(got >= sc.max(axis=1) - 1e-4 * np.maximum(1, np.abs(sc.max(axis=1))))
