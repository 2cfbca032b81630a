"""Robustness of the device-length and append paths:

* attention with a device-resident length much shorter than the capacity the grid
  was sized for (B=1, H=32, T_cap=4096): fewer work units than CTAs must neither
  hang the split-T finisher nor change the result;
* KV appends whose device position falls outside [0, capacity) skip the write and
  raise the device error word; the decoder refuses to step past its capacity.
"""

import numpy as np
import pytest
from conftest import O

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOL_ATTN = 2e-3


@pytest.fixture(scope="module")
def dev():
    return torch.device("cuda", 0)


@pytest.fixture(scope="module")
def long_cache(dev):
    from paper_2503_02236_b200.codec import Codebook, QuantizedTensor, Sharing, VQConfig
    from paper_2503_02236_b200.device import DeviceVQTensor
    B, H, Tc, C, v = 1, 32, 4096, 128, 2
    cfg = VQConfig(v, 8, 1, Sharing.per_channel_group(v))
    shape = (B, H, Tc, C)
    nreg = O.n_regions_of(shape, v, "channel_group", group_width=v)
    regs = O.region_ids(shape, v, "channel_group", group_width=v)
    kc, kb = O.synthetic_codes_books(shape, v, 8, 1, nreg, 41)
    vc, vb = O.synthetic_codes_books(shape, v, 8, 1, nreg, 42)
    kb, vb = O.round_f16(kb), O.round_f16(vb)

    def qt(codes, books):
        return QuantizedTensor(codes, shape, cfg, [Codebook(books[i], 0, i) for i in range(books.shape[0])], nreg)

    kd = DeviceVQTensor.from_quantized(qt(kc, kb), device=dev)
    vd = DeviceVQTensor.from_quantized(qt(vc, vb), device=dev)
    kdense = O.dequantize(kc, kb, shape, v, nreg, regs)
    vdense = O.dequantize(vc, vb, shape, v, nreg, regs)
    return kd, vd, kdense, vdense


@pytest.mark.parametrize("T", [600, 2000, 4000])
def test_device_length_shorter_than_capacity(T, dev, long_cache):
    from paper_2503_02236_b200 import _native as N
    from paper_2503_02236_b200 import ops
    kd, vd, kdense, vdense = long_cache
    q = O.synthetic_tensor((1, 32, 128), 43)
    qt = torch.from_numpy(q).to(dev)
    d_len = torch.full((1,), T, dtype=torch.int32, device=dev)
    out_dev = ops.vq_attention(kd, vd, qt, d_len=d_len)
    assert N.last_kernel() == "attn_cq"
    torch.cuda.synchronize()
    out_host = ops.vq_attention(kd, vd, qt, length=T)
    assert torch.equal(out_dev, out_host)
    ref = O.attention_ref(q, kdense[:, :, :T], vdense[:, :, :T])
    assert O.rel_err(out_dev.cpu().numpy(), ref) <= TOL_ATTN


def test_kv_append_out_of_capacity_is_skipped_and_flagged(dev):
    from paper_2503_02236_b200 import _native as N
    from paper_2503_02236_b200 import ops
    from paper_2503_02236_b200.decode import KV_CFG
    from paper_2503_02236_b200.device import DeviceVQTensor
    B, H, C, T = 2, 4, 128, 64
    g = torch.Generator(device=dev).manual_seed(3)
    books = [torch.randn((H * C // 2, 256, 2), generator=g, device=dev).half() for _ in range(2)]
    k, v = (DeviceVQTensor.empty_cache((B, H, T, C), KV_CFG, bk) for bk in books)
    before = (k.codes.clone(), v.codes.clone())
    N.take_device_error()
    qkv = torch.randn((B, 3 * H * C), generator=g, device=dev).half()
    for bad in (T + 1, 0):  # position T (one past the end) and -1
        d_len = torch.full((1,), bad, dtype=torch.int32, device=dev)
        ops.qkv_rope_append(qkv, k, v, d_len)
        assert N.take_device_error() & 1, bad
        x = torch.randn((B, H, 1, C), generator=g, device=dev).half()
        ops.vq_quantize_kv(k, x, d_len=d_len)
        assert N.take_device_error() & 1, bad
    assert torch.equal(k.codes, before[0]) and torch.equal(v.codes, before[1])
    d_len = torch.full((1,), T, dtype=torch.int32, device=dev)  # the last slot: valid
    ops.qkv_rope_append(qkv, k, v, d_len)
    assert N.take_device_error() == 0


def test_decoder_refuses_to_step_past_capacity(dev):
    from paper_2503_02236_b200.decode import LlamaShape, VQLlamaDecoder
    from paper_2503_02236_b200.errors import CapacityError
    sh = LlamaShape(hidden=256, heads=2, head_dim=128, ffn=512, layers=1, vocab=64)
    dec = VQLlamaDecoder.synthetic(sh, 1, 64, dev, seed=1)
    with pytest.raises(CapacityError):
        dec.set_length(64)
    dec.set_length(62)
    dec.capture()
    dec.replay()
    dec.replay()  # position 63, the last slot
    with pytest.raises(CapacityError):
        dec.replay()
    dec.check_device_errors()
    assert int(dec.d_len.item()) == 64


def _quip_weight(dev, m=4096, n=12288, seed=3):
    from paper_2503_02236_b200.codec import VQConfig
    from paper_2503_02236_b200.device import DeviceVQTensor
    g = torch.Generator(device=dev).manual_seed(seed)
    codes = torch.randint(0, 256, (1, m * n // 8), generator=g, device=dev, dtype=torch.int32)
    books = (torch.randn((1, 1 << 16, 8), generator=g, device=dev) * 0.1).half()
    return DeviceVQTensor.from_device_codes(codes, (m, n), VQConfig(8, 16, 1), books).relayout("gemv")


def test_cooperative_launch_matches_default(dev, long_cache):
    """VQB_FLAG_COOPERATIVE (driver-guaranteed co-residency of the persistent grid)
    gives the same results as the default PDL launch."""
    from paper_2503_02236_b200 import _native as N
    from paper_2503_02236_b200 import ops
    w = _quip_weight(dev)
    x = torch.randn((1, 4096), device=dev).half()
    coop = ops.launch_struct()
    coop.flags |= N.FLAG_COOPERATIVE
    assert torch.equal(ops.vq_gemv(w, x), ops.vq_gemv(w, x, launch=coop))
    kd, vd, _, _ = long_cache
    q = torch.randn((1, 32, 128), device=dev).half()
    assert torch.equal(ops.vq_attention(kd, vd, q), ops.vq_attention(kd, vd, q, launch=coop))


def test_concurrent_stream_holding_sms(dev, long_cache):
    """The persistent kernels' finishers wait on later CTAs: with another stream's
    kernels holding SMs they must still complete (the other work is finite) and
    give the same results."""
    from paper_2503_02236_b200 import ops
    w = _quip_weight(dev)
    kd, vd, _, _ = long_cache
    x = torch.randn((1, 4096), device=dev).half()
    q = torch.randn((1, 32, 128), device=dev).half()
    y0, a0 = ops.vq_gemv(w, x), ops.vq_attention(kd, vd, q)
    torch.cuda.synchronize()
    side = torch.cuda.Stream(dev)
    big = torch.randn((8192, 8192), device=dev).half()
    with torch.cuda.stream(side):
        for _ in range(12):
            big = (big @ big).clamp_(-1, 1)
    ys, as_ = [], []
    for _ in range(30):
        ys.append(ops.vq_gemv(w, x))
        as_.append(ops.vq_attention(kd, vd, q))
    torch.cuda.synchronize()
    assert all(torch.equal(y, y0) for y in ys)
    assert all(torch.equal(a, a0) for a in as_)
