"""Full-size parity against the independent CPU oracle (oracle/vq_oracle.c, the
C/OpenMP restatement of V/codec.py:391-408 dequantize + V/sim.py:133-155
reference_compute), not against the GPU's own dequantization: the BASELINE
configs' real shapes (C1 GPTVQ 4096^2, C2 QuiP# qkv / down, C3 AQLM 2x8 at the
65B q shape, the C2 prefill GEMM at rows 1024, C4 attention B16 H32 T4096 C128
sampled over batch rows). Tolerances: 1e-3 rel-to-max for fp16 I/O with fp32
accumulation, 2e-3 for the tcgen05 GEMM and attention."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import c_oracle as CO  # noqa: E402
from oracle import vq_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    return torch.device("cuda", 0)


def _weight(dev, shape, v, bits, r, sharing, work=None, seed=0):
    from paper_2503_02236_b200.codec import Sharing, VQConfig, region_count
    from paper_2503_02236_b200.device import DeviceVQTensor
    sh = Sharing.per_tile(256, 256) if sharing == "tile" else Sharing.whole_tensor()
    cfg = VQConfig(v, bits, r, sh)
    g = torch.Generator(device=dev).manual_seed(seed)
    m, n = shape
    nreg = region_count(shape, cfg)
    codes = torch.randint(0, work or cfg.n_entries, (r, m * n // v), generator=g, device=dev, dtype=torch.int32)
    books = (torch.randn((r * nreg, cfg.n_entries, v), generator=g, device=dev) * 0.1).half()
    w = DeviceVQTensor.from_device_codes(codes, shape, cfg, books).relayout("gemv")
    regions = O.region_ids(shape, v, sharing, (256, 256), 0)
    return w, codes.cpu().numpy(), books.float().cpu().numpy(), nreg, regions


def _rel(y, ref):
    y = y.float().cpu().numpy() if torch.is_tensor(y) else y
    return float(np.abs(y - ref).max() / np.abs(ref).max())


FULL_GEMV = [
    ("C1 gptvq2 q_proj", (4096, 4096), 4, 8, 1, "tile", None),
    ("C2 quip2 qkv", (4096, 12288), 8, 16, 1, "whole", 256),
    ("C2 quip2 down", (11008, 4096), 8, 16, 1, "whole", 256),
    ("C3 aqlm2x8 65B q", (8192, 8192), 8, 8, 2, "whole", None),
]


@pytest.mark.parametrize("label,shape,v,bits,r,sharing,work", FULL_GEMV)
@pytest.mark.parametrize("rows", [1, 8, 16])
def test_full_size_gemv_vs_c_oracle(label, shape, v, bits, r, sharing, work, rows, dev):
    from paper_2503_02236_b200 import _native as N
    from paper_2503_02236_b200 import ops
    w, codes, books, nreg, regions = _weight(dev, shape, v, bits, r, sharing, work)
    x = O.round_f16(O.synthetic_tensor((rows, shape[0]), 7))
    y = ops.vq_gemv(w, torch.from_numpy(x).to(dev).half(), out_dtype=torch.float32)
    colsplit = rows == 1 and sharing == "whole" and r == 1 and 111 <= shape[1] // 256 * 8 <= 148
    want = ("gemv_cs" if colsplit else "gemv_fast") if rows <= 4 or (rows <= 8 and sharing != "whole") \
        else "gemv_tc" if sharing == "whole" else "gemv_generic"
    assert N.last_kernel() == want, label
    ref = CO.gemv(codes, books, shape, v, nreg, regions, x)
    assert _rel(y, ref) <= 1e-3, label


def test_full_size_prefill_gemm_vs_c_oracle(dev):
    """C2 q_proj prefill, rows 1024 (tcgen05 CTA-pair GEMM) vs the C oracle on the
    fp16-rounded dequantized weight the tensor cores consume."""
    from paper_2503_02236_b200 import _native as N
    from paper_2503_02236_b200 import ops
    shape = (4096, 4096)
    w, codes, books, nreg, regions = _weight(dev, shape, 8, 16, 1, "whole", 256, seed=3)
    x = O.round_f16(O.synthetic_tensor((1024, 4096), 8))
    y = ops.vq_gemm(w, torch.from_numpy(x).to(dev).half(), out_dtype=torch.float32)
    assert N.last_kernel() == "gemm_tc2"
    # the books are fp16 already and R == 1, so dequant(W) is exactly fp16-representable
    ref = CO.gemv(codes, books, shape, 8, nreg, regions, x)
    assert _rel(y, ref) <= 2e-3


def test_full_size_attention_c4_vs_c_oracle(dev):
    """C4 CQ-4 cache at full size on the GPU; the C oracle recomputes batch rows
    0, 7 and 15 (all 32 heads, 4096 tokens) from the same codes and books."""
    from paper_2503_02236_b200 import _native as N
    from paper_2503_02236_b200 import ops
    from paper_2503_02236_b200.codec import Sharing, VQConfig
    from paper_2503_02236_b200.device import DeviceVQTensor
    B, H, T, C = 16, 32, 4096, 128
    cfg = VQConfig(2, 8, 1, Sharing.per_channel_group(2))
    g = torch.Generator(device=dev).manual_seed(9)
    per_b = H * T * C // 2
    host = []
    kv = []
    for _ in range(2):
        codes = torch.randint(0, 256, (1, B * per_b), generator=g, device=dev, dtype=torch.int32)
        books = (torch.randn((H * 64, 256, 2), generator=g, device=dev) * 0.1).half()
        kv.append(DeviceVQTensor.from_device_codes(codes, (B, H, T, C), cfg, books).relayout("kv"))
        host.append((codes.cpu().numpy(), books.float().cpu().numpy()))
    q = O.round_f16(O.synthetic_tensor((B, H, C), 10))
    out = ops.vq_attention(kv[0], kv[1], torch.from_numpy(q).to(dev).half(), out_dtype=torch.float32)
    assert N.last_kernel() == "attn_cq"
    out = out.cpu().numpy()
    regions = O.region_ids((1, H, T, C), 2, "channel_group", group_width=2)
    for b in (0, 7, 15):
        dense = [CO.dequantize(c[:, b * per_b:(b + 1) * per_b], bk, (1, H, T, C), 2, H * 64, regions)
                 for c, bk in host]
        ref = CO.attention(q[b:b + 1], dense[0], dense[1])
        assert _rel(out[b:b + 1], ref) <= 2e-3, b
