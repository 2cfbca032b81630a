"""Column-split batch 1/2/4 GEMV (csrc/gemv_cs.cu): every CTA owns a 32-column slice of a
256-column block for all M rows, so there is no cross-CTA split reduction. Parity
against the C oracle (oracle/vq_oracle.c, V/codec.py:391-408 + V/sim.py:133-155) at the
Llama-7B o / down shapes and a TP2 o shard, fp16 and fp32 outputs, a 65536-entry book
with a 256-entry working set, against the stream-K kernel (VQB_FLAG_NO_COLSPLIT), and
deterministic replays. Tolerance 1e-3 rel-to-max (fp16 I/O, fp32 accumulation)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import c_oracle as CO  # noqa: E402
from oracle import vq_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    return torch.device("cuda", 0)


def _weight(dev, shape, entries, work, seed):
    from paper_2503_02236_b200.codec import Sharing, VQConfig
    from paper_2503_02236_b200.device import DeviceVQTensor
    cfg = VQConfig(8, 16, 1, Sharing.whole_tensor())
    g = torch.Generator(device=dev).manual_seed(seed)
    m, n = shape
    codes = torch.randint(0, work, (1, m * n // 8), generator=g, device=dev, dtype=torch.int32)
    books = (torch.randn((1, entries, 8), generator=g, device=dev) * 0.1).half()
    w = DeviceVQTensor.from_device_codes(codes, shape, cfg, books).relayout("gemv")
    return w, codes.cpu().numpy(), books.float().cpu().numpy()


@pytest.mark.parametrize("shape", [(4096, 4096), (11008, 4096), (2048, 4096)])
@pytest.mark.parametrize("out", ["f16", "f32"])
@pytest.mark.parametrize("rows", [1, 2, 4])
def test_colsplit_gemv_vs_c_oracle(shape, out, rows, dev):
    from paper_2503_02236_b200 import _native as N
    from paper_2503_02236_b200 import ops
    w, codes, books, = _weight(dev, shape, 65536, 256, seed=shape[0] % 97)
    x = O.round_f16(O.synthetic_tensor((rows, shape[0]), 3))
    od = torch.float16 if out == "f16" else torch.float32
    y = ops.vq_gemv(w, torch.from_numpy(x).to(dev).half(), out_dtype=od)
    assert N.last_kernel() == "gemv_cs"
    regions = O.region_ids(shape, 8, "whole", (256, 256), 0)
    ref = CO.gemv(codes, books, shape, 8, 1, regions, x)
    got = y.float().cpu().numpy()
    assert float(np.abs(got - ref).max() / np.abs(ref).max()) <= 1e-3
    # deterministic (no atomics, no cross-CTA order)
    assert torch.equal(y, ops.vq_gemv(w, torch.from_numpy(x).to(dev).half(), out_dtype=od))


def test_colsplit_matches_stream_k(dev):
    from paper_2503_02236_b200 import _native as N
    from paper_2503_02236_b200 import ops
    w, _, _ = _weight(dev, (4096, 4096), 256, 256, seed=5)
    g = torch.Generator(device=dev).manual_seed(6)
    x = torch.randn((1, 4096), generator=g, device=dev).half()
    a = ops.vq_gemv(w, x, out_dtype=torch.float32)
    assert N.last_kernel() == "gemv_cs"
    L = ops.launch_struct()
    L.flags |= N.FLAG_NO_COLSPLIT
    b = ops.vq_gemv(w, x, out_dtype=torch.float32, launch=L)
    assert N.last_kernel() == "gemv_fast"
    assert float((a - b).abs().max() / b.abs().max()) <= 1e-3


def test_colsplit_not_taken_outside_its_shapes(dev):
    from paper_2503_02236_b200 import _native as N
    from paper_2503_02236_b200 import ops
    w, _, _ = _weight(dev, (4096, 12288), 256, 256, seed=7)  # 48 blocks: stream-K
    ops.vq_gemv(w, torch.randn((1, 4096), device=dev).half())
    assert N.last_kernel() == "gemv_fast"
    w, _, _ = _weight(dev, (4096, 4096), 65536, 65536, seed=8)  # codes beyond 256: global tier
    ops.vq_gemv(w, torch.randn((1, 4096), device=dev).half())
    assert N.last_kernel() != "gemv_cs"


@pytest.mark.parametrize("m", [4104, 1032, 8])  # row groups not a multiple of the 128 row lanes
@pytest.mark.parametrize("rows", [1, 4])
def test_colsplit_ragged_rows(m, rows, dev):
    from paper_2503_02236_b200 import _native as N
    from paper_2503_02236_b200 import ops
    shape = (m, 4096)
    w, codes, books = _weight(dev, shape, 256, 256, seed=m)
    x = O.round_f16(O.synthetic_tensor((rows, m), 4))
    y = ops.vq_gemv(w, torch.from_numpy(x).to(dev).half(), out_dtype=torch.float32)
    assert N.last_kernel() == "gemv_cs"
    regions = O.region_ids(shape, 8, "whole", (256, 256), 0)
    ref = CO.gemv(codes, books, shape, 8, 1, regions, x)
    got = y.float().cpu().numpy()
    assert float(np.abs(got - ref).max() / np.abs(ref).max()) <= 1e-3
