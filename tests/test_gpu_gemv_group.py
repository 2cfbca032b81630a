"""Fast GEMV beyond whole 256-column blocks and the grouped (multi-linear) launch.

* TP shards of Llama widths are not multiples of 256 columns (22016 / 4 = 5504,
  22016 / 8 = 2752): the fast kernel handles the narrower last column block of
  the GEMV_IL layout instead of falling back to the generic kernel.
* vqb_gemv_grouped runs a list of independent GEMVs as one persistent launch; per
  problem the result matches the oracle (dequantize + fp32 matmul, V/sim.py:136-144)
  within the fp16 tolerance and the single-launch kernel to fp32 rounding.
"""

import numpy as np
import pytest
from conftest import O

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOL_F16 = 1e-3


@pytest.fixture(scope="module")
def dev():
    return torch.device("cuda", 0)


def _weight(m, n, seed, dev, bits=16, work=256, r=1):
    from paper_2503_02236_b200.codec import Codebook, QuantizedTensor, VQConfig
    from paper_2503_02236_b200.device import DeviceVQTensor
    cfg = VQConfig(8, bits, r)
    codes, books = O.synthetic_codes_books((m, n), 8, bits, r, 1, seed, working_entries=work)
    books = O.round_f16(books)
    q = QuantizedTensor(codes, (m, n), cfg, [Codebook(books[i], i, 0) for i in range(r)], 1)
    w = DeviceVQTensor.from_quantized(q, device=dev)
    assert w.layout == "gemv"
    dense = O.dequantize(codes, books, (m, n), 8, 1, np.zeros(m * n // 8, np.int32))
    return w, dense


@pytest.mark.parametrize("rows", [1, 2, 4, 8])
@pytest.mark.parametrize("shape", [(4096, 5504), (1024, 2752), (2752, 1024), (512, 264)])
def test_partial_column_block_stays_fast(shape, rows, dev):
    from paper_2503_02236_b200 import _native as N
    from paper_2503_02236_b200.ops import vq_gemv
    m, n = shape
    w, dense = _weight(m, n, 5 + rows, dev)
    x = O.round_f16(O.synthetic_tensor((rows, m), 7))
    y = vq_gemv(w, torch.from_numpy(x).to(dev).half(), out_dtype=torch.float32)
    # never the generic kernel: the decode GEMV families (tcgen05 from 5 rows where N % 256 == 0)
    assert N.last_kernel() in ("gemv_fast", "gemv_tc")
    assert O.rel_err(y.cpu().numpy(), O.matmul_ref(x, dense)) <= TOL_F16


def test_partial_column_block_aqlm(dev):
    """AQLM 2x8 (two u8 levels) at the TP8 up-projection shard width."""
    from paper_2503_02236_b200 import _native as N
    from paper_2503_02236_b200.ops import vq_gemv
    w, dense = _weight(1024, 2752, 9, dev, bits=8, work=None, r=2)
    x = O.round_f16(O.synthetic_tensor((1024,), 3))
    y = vq_gemv(w, torch.from_numpy(x).to(dev).half(), out_dtype=torch.float32)
    assert N.last_kernel() == "gemv_fast"
    assert O.rel_err(y.cpu().numpy(), O.matmul_ref(x, dense)) <= TOL_F16


@pytest.mark.parametrize("rows", [1, 2, 4, 8])
def test_grouped_matches_oracle_and_single_launches(rows, dev):
    from paper_2503_02236_b200 import _native as N
    from paper_2503_02236_b200.stack import VQLinearStack
    shapes = [(1024, 3072), (1024, 1024), (1024, 5504), (2752, 1024), (512, 264), (4096, 256), (1024, 2048)]
    ws, dense = zip(*[_weight(m, n, 20 + i, dev) for i, (m, n) in enumerate(shapes)])
    grouped = VQLinearStack(ws, rows=rows, out_dtype=torch.float32, grouped=True)
    single = VQLinearStack(ws, rows=rows, out_dtype=torch.float32)
    assert grouped.n_launches == 1 and single.n_launches == len(shapes)
    g = torch.Generator(device=dev).manual_seed(1)
    grouped.x.copy_(torch.randn(grouped.x.shape, generator=g, device=dev).half())
    single.x.copy_(grouped.x)
    grouped.launch_all()
    assert N.last_kernel() == "gemv_group"
    single.launch_all()
    torch.cuda.synchronize()
    for i, d in enumerate(dense):
        x = grouped.input_view(i).float().cpu().numpy()
        yg = grouped.output_view(i).cpu().numpy()
        ys = single.output_view(i).cpu().numpy()
        assert O.rel_err(yg, O.matmul_ref(x, d)) <= TOL_F16, i
        assert O.rel_err(yg, ys) <= 1e-5, i


def test_grouped_graph_replay_is_deterministic(dev):
    from paper_2503_02236_b200.stack import VQLinearStack
    shapes = [(2048, 3072), (2048, 1024), (1024, 5504)] * 3
    ws, _ = zip(*[_weight(m, n, 40 + i, dev) for i, (m, n) in enumerate(shapes)])
    st = VQLinearStack(ws, rows=1, grouped=True)
    st.x.copy_(torch.randn(st.x.shape, device=dev).half())
    st.capture()
    st.replay()
    torch.cuda.synchronize()
    first = st.y.clone()
    for _ in range(5):
        st.replay()
    torch.cuda.synchronize()
    assert torch.equal(first, st.y)


def test_grouped_rejects_mixed_configs(dev):
    from paper_2503_02236_b200.errors import ConfigError
    from paper_2503_02236_b200.stack import VQLinearStack
    a, _ = _weight(512, 512, 1, dev)
    b, _ = _weight(512, 512, 2, dev, bits=8, work=None, r=2)
    st = VQLinearStack([a, b], rows=1, grouped=True)
    with pytest.raises(ConfigError, match="grouped GEMV"):
        st.launch_all()


def test_stack_pipeline_matches_serial_runs(dev):
    """StackPipeline (double-buffered sets, H2D / D2H on their own streams) returns, per
    step, exactly what the serial VQLinearStack.run returns for that step's input."""
    from paper_2503_02236_b200.stack import StackPipeline, VQLinearStack
    shapes = [(1024, 3072), (1024, 1024), (2752, 1024)]
    ws, _ = zip(*[_weight(m, n, 60 + i, dev) for i, (m, n) in enumerate(shapes)])
    st = VQLinearStack(ws, rows=1, grouped=True)
    ref = VQLinearStack(ws, rows=1, grouped=True)
    steps = 5
    g = torch.Generator().manual_seed(3)
    hxs = [torch.randn(st.x.shape, generator=g).half().pin_memory() for _ in range(steps)]
    hys = [torch.empty(st.y.shape, dtype=st.y.dtype).pin_memory() for _ in range(steps)]
    StackPipeline(st).run(hxs, hys)
    torch.cuda.synchronize()
    for hx, hy in zip(hxs, hys):
        out = torch.empty_like(hy).pin_memory()
        ref.run(hx, out)
        torch.cuda.synchronize()
        assert torch.equal(hy, out)
