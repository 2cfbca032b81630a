"""Parity of the CUDA kernels (through the C ABI) against the CPU oracle and the
reference's golden vectors. Bit-exact for dequantization; the fused ops within
the stated tolerances:

  * fp32 codebooks + fp32 activations (parity mode, generic kernel): 1e-4
    rel-to-max — the reference's own contract (verify.py:212-213)
  * fp16 codebooks + fp16 activations, fp32 accumulation (fast kernels): 1e-3
    against the oracle run on the same fp16-rounded inputs
  * attention with fp16 probabilities in the V accumulation: 2e-3
"""

import hashlib

import numpy as np
import pytest
from conftest import ATTENTION_CASES, CASES, MATMUL_CASES, Case, O

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOL_PARITY = 1e-4
TOL_F16 = 1e-3
TOL_ATTN = 2e-3


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def dev():
    return torch.device("cuda", 0)


def _mods():
    from paper_2503_02236_b200 import _native as N
    from paper_2503_02236_b200.device import DeviceVQTensor
    from paper_2503_02236_b200 import ops
    return N, DeviceVQTensor, ops


# ---- dequantization: bit-exact -----------------------------------------------------------------

@pytest.mark.parametrize("layout", ["plain", "packed", "auto"])
@pytest.mark.parametrize("name", sorted(CASES))
def test_dequant_bit_exact_fp32(name, layout, dev, meta):
    N, DeviceVQTensor, ops = _mods()
    c = Case(name)
    q = c.quantized()
    if layout == "packed":
        d = DeviceVQTensor.from_packed(q.packed_codes(), q.shape, q.config, q.codebooks, device=dev,
                                       codebook_dtype="float32")
    else:
        d = DeviceVQTensor.from_quantized(q, device=dev, codebook_dtype="float32", layout=layout)
    out = ops.vq_dequantize(d).cpu().numpy()
    assert N.last_kernel() == "dequant"
    assert sha(out) == meta["dequant"][name]["dequant_sha"]


@pytest.mark.parametrize("name", sorted(CASES))
def test_dequant_fp16_books_and_casts(name, dev, meta):
    N, DeviceVQTensor, ops = _mods()
    c = Case(name, books_f16=True)
    d = DeviceVQTensor.from_quantized(c.quantized(), device=dev, codebook_dtype="float16")
    out = ops.vq_dequantize(d).cpu().numpy()
    assert sha(out) == meta["dequant"][name]["dequant16_sha"]
    ref = c.dense()
    h = ops.vq_dequantize(d, out_dtype=torch.float16).cpu()
    assert torch.equal(h, torch.from_numpy(ref).half())
    b = ops.vq_dequantize(d, out_dtype=torch.bfloat16).cpu()
    assert torch.equal(b, torch.from_numpy(ref).bfloat16())


def test_dequant_module_api_matches_reference(meta):
    from paper_2503_02236_b200.codec import dequantize
    c = Case("aqlm3")
    out = dequantize(c.quantized())
    assert isinstance(out, np.ndarray) and out.dtype == np.float32
    assert sha(out) == meta["dequant"]["aqlm3"]["dequant_sha"]


def test_dequant_code_out_of_range(dev):
    from paper_2503_02236_b200.errors import CodeRangeError
    _, DeviceVQTensor, _ = _mods()
    c = Case("cq2")
    q = c.quantized()
    q.codes[0, 3] = q.config.n_entries + 7
    with pytest.raises(CodeRangeError, match="code out of range"):
        DeviceVQTensor.from_quantized(q, device=dev)


def test_dequant_negative_zero(dev):
    from paper_2503_02236_b200.codec import Codebook, QuantizedTensor, VQConfig
    _, DeviceVQTensor, ops = _mods()
    books = [Codebook(np.array([[-0.0, 1.0], [2.0, -0.0]], np.float32), 0, 0),
             Codebook(np.array([[-0.0, -0.0], [0.5, -0.0]], np.float32), 1, 0)]
    q = QuantizedTensor(np.array([[0, 1], [0, 0]], np.int32), (1, 4), VQConfig(2, 1, 2), books, 1)
    out = ops.vq_dequantize(DeviceVQTensor.from_quantized(q, device=dev, codebook_dtype="float32"))
    assert not torch.signbit(out).any()


# ---- fused GEMV / GEMM ----------------------------------------------------------------------------

def _act(c, kind, extra):
    m = c.shape[0]
    return O.synthetic_tensor((m,) if kind == "gemv" else (extra["rows"], m), c.seed + 2)


@pytest.mark.parametrize("name,base,kind,extra", MATMUL_CASES)
def test_matmul_parity_mode(name, base, kind, extra, dev, arrays):
    """fp32 books + fp32 activations: within the reference's 1e-4 of its own golden output."""
    N, DeviceVQTensor, ops = _mods()
    c = Case(base)
    d = DeviceVQTensor.from_quantized(c.quantized(), device=dev, codebook_dtype="float32")
    a = torch.from_numpy(_act(c, kind, extra)).to(dev)
    fn = ops.vq_gemv if kind == "gemv" else ops.vq_gemm
    y = fn(d, a).cpu().numpy()
    assert O.rel_err(y, arrays[f"mm_ref_{name}"]) <= TOL_PARITY


def _big_weight(shape, v, bits, r, sharing="whole", tile=(0, 0), work=None, seed=0):
    nreg = O.n_regions_of(shape, v, sharing, tile)
    codes, books = O.synthetic_codes_books(shape, v, bits, r, nreg, seed, working_entries=work)
    books = O.round_f16(books)
    dense = O.dequantize(codes, books, shape, v, nreg, O.region_ids(shape, v, sharing, tile))
    return codes, books, nreg, dense


def _qt(codes, books, nreg, shape, cfg):
    from paper_2503_02236_b200.codec import Codebook, QuantizedTensor
    cbs = [Codebook(books[i], i // nreg, i % nreg) for i in range(books.shape[0])]
    return QuantizedTensor(codes, shape, cfg, cbs, nreg)


FAST_GEMV = [
    # (label, shape, v, bits, R, sharing, tile, working set)
    ("C2_quip2_q_proj", (4096, 4096), 8, 16, 1, "whole", (0, 0), 256),
    ("C1_gptvq2_q_proj", (4096, 4096), 4, 8, 1, "tile", (256, 256), None),
    ("C3_aqlm2x8", (4096, 2048), 8, 8, 2, "whole", (0, 0), None),
    ("C2_quip2_down", (11008, 1024), 8, 16, 1, "whole", (0, 0), 256),
    ("quip2_full_table", (512, 1024), 8, 16, 1, "whole", (0, 0), None),  # global tier hits
]


@pytest.mark.parametrize("rows", [1, 2, 4, 8])
@pytest.mark.parametrize("label,shape,v,bits,r,sharing,tile,work", FAST_GEMV)
def test_gemv_fast_kernel(label, shape, v, bits, r, sharing, tile, work, rows, dev):
    from paper_2503_02236_b200.codec import Sharing, VQConfig
    N, DeviceVQTensor, ops = _mods()
    sh = Sharing.per_tile(*tile) if sharing == "tile" else Sharing.whole_tensor()
    cfg = VQConfig(v, bits, r, sh)
    codes, books, nreg, dense = _big_weight(shape, v, bits, r, sharing, tile, work)
    d = DeviceVQTensor.from_quantized(_qt(codes, books, nreg, shape, cfg), device=dev)
    assert d.layout == "gemv"
    x = O.round_f16(O.synthetic_tensor((rows, shape[0]), 7))
    L = ops.launch_struct()
    L.flags |= N.FLAG_NO_GEMV_TC | N.FLAG_NO_COLSPLIT  # this kernel family (batch 8 defaults to the
    y = ops.vq_gemv(d, torch.from_numpy(x).to(dev).half(), launch=L)  # tcgen05 GEMV, batch 1 at N = 4096
    assert N.last_kernel() == "gemv_fast"
    ref = O.matmul_ref(x, dense)
    assert O.rel_err(y.cpu().numpy(), ref) <= TOL_F16
    # second launch reuses the self-reset split counters
    y2 = ops.vq_gemv(d, torch.from_numpy(x).to(dev).half(), launch=L)
    assert torch.equal(y, y2), "split reduction must be deterministic"


@pytest.mark.parametrize("label,shape,v,bits,r,sharing,tile,work", FAST_GEMV)
def test_gemv_batch16(label, shape, v, bits, r, sharing, tile, work, dev):
    """Batch 16: the tcgen05 decode GEMV where every code is in the shared tier and
    N % 256 == 0 (the mma.sync kernel with two n8 batch tiles under VQB_FLAG_NO_GEMV_TC);
    tile-shared and global-tier configurations take the generic kernel, equally exact."""
    from paper_2503_02236_b200.codec import Sharing, VQConfig
    N, DeviceVQTensor, ops = _mods()
    sh = Sharing.per_tile(*tile) if sharing == "tile" else Sharing.whole_tensor()
    cfg = VQConfig(v, bits, r, sh)
    codes, books, nreg, dense = _big_weight(shape, v, bits, r, sharing, tile, work)
    d = DeviceVQTensor.from_quantized(_qt(codes, books, nreg, shape, cfg), device=dev)
    x = O.round_f16(O.synthetic_tensor((16, shape[0]), 9))
    y = ops.vq_gemv(d, torch.from_numpy(x).to(dev).half())
    fast = v == 8 and sharing == "whole" and (work is not None or bits == 8)
    assert N.last_kernel() == ("gemv_tc" if fast else "gemv_generic"), label
    assert O.rel_err(y.cpu().numpy(), O.matmul_ref(x, dense)) <= TOL_F16
    assert torch.equal(y, ops.vq_gemv(d, torch.from_numpy(x).to(dev).half()))


@pytest.mark.parametrize("rows", [4, 8])
@pytest.mark.parametrize("label,shape,v,bits,r,sharing,tile,work", [c for c in FAST_GEMV if c[2] == 8 and c[5] == "whole"])
def test_gemv_cuda_core_path_at_mma_batches(label, shape, v, bits, r, sharing, tile, work, rows, dev):
    """Batch 4-8 default to the tensor-core inner product; VQB_FLAG_NO_MMA keeps the
    CUDA-core path reachable and equally exact."""
    from paper_2503_02236_b200.codec import Sharing, VQConfig
    N, DeviceVQTensor, ops = _mods()
    cfg = VQConfig(v, bits, r, Sharing.whole_tensor())
    codes, books, nreg, dense = _big_weight(shape, v, bits, r, sharing, tile, work)
    d = DeviceVQTensor.from_quantized(_qt(codes, books, nreg, shape, cfg), device=dev)
    x = torch.from_numpy(O.round_f16(O.synthetic_tensor((rows, shape[0]), 7))).to(dev).half()
    ref = O.matmul_ref(x.float().cpu().numpy(), dense)
    L = ops.launch_struct()
    L.flags = N.FLAG_NO_MMA | N.FLAG_NO_GEMV_TC | N.FLAG_NO_COLSPLIT
    y_fma = ops.vq_gemv(d, x, launch=L)
    L2 = ops.launch_struct()
    L2.flags = N.FLAG_NO_GEMV_TC | N.FLAG_NO_COLSPLIT
    y_mma = ops.vq_gemv(d, x, launch=L2)
    assert N.last_kernel() == "gemv_fast"
    assert O.rel_err(y_fma.cpu().numpy(), ref) <= TOL_F16
    assert O.rel_err(y_mma.cpu().numpy(), ref) <= TOL_F16


def test_gemv_fast_fp16_output_and_plans(dev):
    from paper_2503_02236_b200.codec import VQConfig
    N, DeviceVQTensor, ops = _mods()
    shape = (2048, 2048)
    codes, books, nreg, dense = _big_weight(shape, 8, 16, 1, work=256, seed=3)
    d = DeviceVQTensor.from_quantized(_qt(codes, books, nreg, shape, VQConfig(8, 16, 1)), device=dev)
    x = O.round_f16(O.synthetic_tensor((shape[0],), 9))
    xt = torch.from_numpy(x).to(dev).half()
    ref = O.matmul_ref(x, dense)
    for grid in (0, 5, 37):
        for n_sh in (0, 64, 256, 1024):
            for flags in (0, 4, 8):  # default / no PDL / exact fp32 accumulation
                L = ops.launch_struct(n_shared=n_sh if n_sh else None, grid_limit=grid)
                L.flags = flags
                y = ops.vq_gemv(d, xt, out_dtype=torch.float16, launch=L)
                assert N.last_kernel() == "gemv_fast"
                assert O.rel_err(y.float().cpu().numpy(), ref) <= 2e-3, (grid, n_sh, flags)


# ---- attention ------------------------------------------------------------------------------------

@pytest.mark.parametrize("name,base", ATTENTION_CASES)
def test_attention_parity_mode(name, base, dev, arrays):
    N, DeviceVQTensor, ops = _mods()
    k, v = Case(base), Case(base, seed_offset=1)
    kd = DeviceVQTensor.from_quantized(k.quantized(), device=dev, codebook_dtype="float32")
    vd = DeviceVQTensor.from_quantized(v.quantized(), device=dev, codebook_dtype="float32")
    b, h, t, c = k.shape
    q = torch.from_numpy(O.synthetic_tensor((b, h, c), k.seed + 2)).to(dev)
    out = ops.vq_attention(kd, vd, q).cpu().numpy()
    assert N.last_kernel() == "attn_generic"
    assert O.rel_err(out, arrays[f"at_ref_{name}"]) <= TOL_PARITY


ATTN_SHAPES = [
    # (v, gw, shape): CQ-4 / CQ-2 at several contexts, incl. multi-chunk splits
    (2, 2, (2, 4, 64, 128)),
    (2, 2, (2, 3, 4096, 128)),
    (2, 2, (1, 2, 1000 // 32 * 32, 128)),
    (4, 4, (2, 4, 512, 128)),
    (4, 4, (3, 2, 2048, 128)),
    (2, 2, (2, 2, 256, 64)),
]


@pytest.mark.parametrize("v,gw,shape", ATTN_SHAPES)
def test_attention_fast_kernel(v, gw, shape, dev):
    from paper_2503_02236_b200.codec import Sharing, VQConfig
    N, DeviceVQTensor, ops = _mods()
    cfg = VQConfig(v, 8, 1, Sharing.per_channel_group(gw))
    nreg = O.n_regions_of(shape, v, "channel_group", group_width=gw)
    regs = O.region_ids(shape, v, "channel_group", group_width=gw)
    dense = []
    devs = []
    for s in (11, 12):
        codes, books = O.synthetic_codes_books(shape, v, 8, 1, nreg, s)
        books = O.round_f16(books)
        dense.append(O.dequantize(codes, books, shape, v, nreg, regs))
        devs.append(DeviceVQTensor.from_quantized(_qt(codes, books, nreg, shape, cfg), device=dev))
    assert devs[0].layout == "kv"
    b, h, t, c = shape
    q = O.synthetic_tensor((b, h, c), 13)
    ref = O.attention_ref(q, dense[0], dense[1])
    for grid in (0, 7):
        L = ops.launch_struct(grid_limit=grid)
        out = ops.vq_attention(devs[0], devs[1], torch.from_numpy(q).to(dev), launch=L)
        assert N.last_kernel() == "attn_cq"
        assert O.rel_err(out.cpu().numpy(), ref) <= TOL_ATTN, grid


def test_attention_known_answer_single_token(dev):
    """T = 1 (generic path): the output is the V row (T/test_sim.py:91-98)."""
    from paper_2503_02236_b200.codec import Codebook, QuantizedTensor, Sharing, VQConfig
    _, DeviceVQTensor, ops = _mods()
    cfg = VQConfig(2, 1, 1, Sharing.per_channel_group(2))
    kb = [Codebook(np.ones((2, 2), np.float32), 0, g) for g in range(2)]
    vb = [Codebook(np.array([[0, 1], [2, 3]], np.float32) + 4 * g, 0, g) for g in range(2)]
    codes = np.zeros((1, 2), np.int32)
    kq = QuantizedTensor(codes, (1, 1, 1, 4), cfg, kb, 2)
    vq = QuantizedTensor(codes, (1, 1, 1, 4), cfg, vb, 2)
    out = ops.vq_attention(DeviceVQTensor.from_quantized(kq, device=dev, codebook_dtype="float32"),
                           DeviceVQTensor.from_quantized(vq, device=dev, codebook_dtype="float32"),
                           torch.ones((1, 1, 4), device=dev))
    assert torch.allclose(out.cpu()[0, 0], torch.tensor([0.0, 1.0, 4.0, 5.0]))


def test_shape_errors(dev):
    from paper_2503_02236_b200.errors import ShapeError
    N, DeviceVQTensor, ops = _mods()
    c = Case("quip2")
    d = DeviceVQTensor.from_quantized(c.quantized(), device=dev)
    with pytest.raises(ShapeError):
        ops.vq_gemv(d, torch.zeros(c.shape[0] + 1, device=dev, dtype=torch.float16))


# ---- prefill GEMM on tcgen05 --------------------------------------------------------------------

GEMM_CASES = [
    # (label, shape (M, N), v, bits, R, working set, rows)
    ("C2_quip2", (1024, 512), 8, 16, 1, 256, 256),
    ("C2_quip2_ragged_rows", (512, 384), 8, 16, 1, 256, 100),
    ("C2_quip2_full_table", (256, 256), 8, 16, 1, None, 64),   # codes beyond the shared tier
    ("C3_aqlm2x8", (1024, 256), 8, 8, 2, None, 300),
    ("aqlm1x8", (768, 640), 8, 8, 1, None, 512),
    ("C2_quip2_prefill_pair", (1024, 768), 8, 16, 1, 256, 600),  # CTA-pair kernel, 256 x 128 tiles
    ("C3_aqlm2x8_prefill", (1024, 512), 8, 8, 2, None, 700),  # two-phase (dequantise + dense pair GEMM)
    ("C2_quip2_prefill_wide", (512, 512), 8, 16, 1, 256, 520),  # 256 x 256 pair tiles, partial row tile
]


@pytest.mark.parametrize("dtype", ["float16", "bfloat16"])
@pytest.mark.parametrize("label,shape,v,bits,r,work,rows", GEMM_CASES)
def test_gemm_tcgen05(label, shape, v, bits, r, work, rows, dtype, dev):
    from paper_2503_02236_b200.codec import VQConfig
    N, DeviceVQTensor, ops = _mods()
    tdt = getattr(torch, dtype)
    cfg = VQConfig(v, bits, r)
    nreg = 1
    codes, books = O.synthetic_codes_books(shape, v, bits, r, nreg, 21, working_entries=work)
    # the device codebook dtype is the operand dtype; the oracle sees the same rounding
    books = torch.from_numpy(books).to(tdt).float().numpy()
    dense = O.dequantize(codes, books, shape, v, nreg, O.region_ids(shape, v, "whole"))
    d = DeviceVQTensor.from_quantized(_qt(codes, books, nreg, shape, cfg), device=dev, codebook_dtype=dtype)
    x = torch.from_numpy(O.synthetic_tensor((rows, shape[0]), 22)).to(tdt)
    ref = O.matmul_ref(x.float().numpy(), dense)
    # prefill sizes (> 256 rows) run the CTA-pair (cta_group::2) kernel; VQB_FLAG_NO_PAIR
    # pins the one-CTA kernel, which also serves the split-K decode sizes
    no_pair = ops.launch_struct()
    no_pair.flags |= N.FLAG_NO_PAIR
    for out_dtype in (torch.float32, tdt):
        n128 = ops.launch_struct()
        n128.flags |= N.FLAG_PAIR_N128
        pair_default = rows > 256 and shape[1] % 256 == 0
        two_phase = pair_default and r == 2 and rows >= 512
        for L, kerns in ((None, ("gemm_2phase",) if two_phase else ("gemm_tc2",) if pair_default
                          else ("gemm_tc", "gemm_tc2")),
                         (no_pair, ("gemm_tc",)), (n128, ("gemm_tc2",) if rows > 256 else ("gemm_tc", "gemm_tc2"))):
            y = ops.vq_gemm(d, x.to(dev), out_dtype=out_dtype, launch=L)
            assert N.last_kernel() in kerns, (N.last_kernel(), kerns)
            tol = 2e-3 if dtype == "float16" else 1.6e-2
            assert O.rel_err(y.float().cpu().numpy(), ref) <= tol, (label, out_dtype, kern)


@pytest.mark.parametrize("dtype", ["float16", "bfloat16"])
@pytest.mark.parametrize("label,shape,v,bits,r,work,rows", [c for c in GEMM_CASES if c[6] > 256 and c[1][1] % 256 == 0])
def test_gemm_two_phase_matches_fused(label, shape, v, bits, r, work, rows, dtype, dev):
    """Prefill sizes through both paths: the fused CTA-pair kernel (VQB_FLAG_GEMM_FUSED)
    and the two-phase path (dequantise to the fp16 scratch, dense tcgen05 pair GEMM,
    VQB_FLAG_GEMM_TWO_PHASE), each against the oracle."""
    from paper_2503_02236_b200.codec import VQConfig
    N, DeviceVQTensor, ops = _mods()
    tdt = getattr(torch, dtype)
    cfg = VQConfig(v, bits, r)
    codes, books = O.synthetic_codes_books(shape, v, bits, r, 1, 23, working_entries=work)
    books = torch.from_numpy(books).to(tdt).float().numpy()
    dense = O.dequantize(codes, books, shape, v, 1, O.region_ids(shape, v, "whole"))
    d = DeviceVQTensor.from_quantized(_qt(codes, books, 1, shape, cfg), device=dev, codebook_dtype=dtype)
    x = torch.from_numpy(O.synthetic_tensor((rows, shape[0]), 24)).to(tdt)
    # the two-phase path rounds the summed levels once (fp32 -> fp16/bf16); the oracle
    # applies the same rounding to the dense weight the tensor cores consume
    w16 = torch.from_numpy(dense).to(tdt).float().numpy()
    ref = O.matmul_ref(x.float().numpy(), w16)
    tol = 2e-3 if dtype == "float16" else 1.6e-2
    for flag, kern in ((N.FLAG_GEMM_FUSED, "gemm_tc2"), (N.FLAG_GEMM_TWO_PHASE, "gemm_2phase")):
        L = ops.launch_struct()
        L.flags |= flag
        for out_dtype in (torch.float32, tdt):
            y = ops.vq_gemm(d, x.to(dev), out_dtype=out_dtype, launch=L)
            assert N.last_kernel() == kern, (N.last_kernel(), kern)
            assert O.rel_err(y.float().cpu().numpy(), ref) <= tol, (label, kern, out_dtype)


@pytest.mark.parametrize("rows", [3, 9, 16, 33, 64])
@pytest.mark.parametrize("label,shape,v,bits,r,sharing,tile,work", [c for c in FAST_GEMV if c[5] == "whole" and (c[7] is not None or c[3] == 8)])
def test_gemv_tcgen05(label, shape, v, bits, r, sharing, tile, work, rows, dev):
    """The tcgen05 decode GEMV (batch = UMMA N, padded to 8..64; split-K partials reduced
    in order): oracle parity, determinism, and the mma.sync kernel at 16 rows agrees."""
    from paper_2503_02236_b200.codec import Sharing, VQConfig
    N, DeviceVQTensor, ops = _mods()
    cfg = VQConfig(v, bits, r, Sharing.whole_tensor())
    codes, books, nreg, dense = _big_weight(shape, v, bits, r, sharing, tile, work)
    d = DeviceVQTensor.from_quantized(_qt(codes, books, nreg, shape, cfg), device=dev)
    x = O.round_f16(O.synthetic_tensor((rows, shape[0]), 11))
    xt = torch.from_numpy(x).to(dev).half()
    y = ops.vq_gemv(d, xt, out_dtype=torch.float32)
    assert N.last_kernel() == "gemv_tc", label
    assert O.rel_err(y.cpu().numpy(), O.matmul_ref(x, dense)) <= TOL_F16
    assert torch.equal(y, ops.vq_gemv(d, xt, out_dtype=torch.float32))
    if rows == 16:
        L = ops.launch_struct()
        L.flags |= N.FLAG_NO_GEMV_TC
        y2 = ops.vq_gemv(d, xt, out_dtype=torch.float32, launch=L)
        assert N.last_kernel() == "gemv_fast"
        assert O.rel_err(y2.cpu().numpy(), O.matmul_ref(x, dense)) <= TOL_F16
