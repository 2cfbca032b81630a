"""Host side of the drop-in: vqforge's own objects go through the upload
conversion unchanged (no GPU needed). Runs only where the reference is mounted
(the build container); the GPU-side counterpart is test_gpu_reference_api.py."""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")


@pytest.fixture(scope="module")
def vq():
    if REF not in sys.path:
        sys.path.append(REF)
    import vqforge.codec as codec
    import vqforge.synth as synth
    return codec, synth


@pytest.mark.parametrize("spec", [(8, 12, 2, "whole"), (4, 8, 1, "tile"), (2, 8, 1, "cg")])
def test_upload_conversion_accepts_vqforge_objects(vq, spec):
    from paper_2503_02236_b200.device import host_codes, stack_codebooks
    codec, synth = vq
    v, bits, r, kind = spec
    sh = {"whole": codec.Sharing.whole_tensor(), "tile": codec.Sharing.per_tile(256, 256),
          "cg": codec.Sharing.per_channel_group(2)}[kind]
    shape = (2, 2, 64, 128) if kind == "cg" else (512, 512)
    q = synth.synthetic_quantized(shape, codec.VQConfig(v, bits, r, sh), 3)
    books = stack_codebooks(q)
    assert books.shape == (r * q.n_regions, 1 << bits, v) and books.dtype == np.float32
    for i, cb in enumerate(q.codebooks):
        assert np.array_equal(books[i], cb.entries)
    raw, hi = host_codes(q)
    narrow = np.uint8 if bits <= 8 else np.uint16
    assert np.array_equal(raw.view(narrow).reshape(q.codes.shape), q.codes)
    assert hi == int(q.codes.max())


def test_code_range_error_on_vqforge_object(vq):
    from paper_2503_02236_b200.device import host_codes
    from paper_2503_02236_b200.errors import CodeRangeError
    codec, synth = vq
    q = synth.synthetic_quantized((64, 64), codec.VQConfig(4, 8, 1), 0)
    q.codes[0, 5] = 300
    with pytest.raises(CodeRangeError, match="code out of range"):
        host_codes(q)


def test_plans_from_vqforge_config_match_reference(vq):
    """plan_kernel fed vqforge's VQConfig / ComputeOp reproduces vqforge's plans."""
    codec, _ = vq
    import vqforge.dataflow as rdf
    import vqforge.gpumodel as rgm
    import vqforge.sim as rsim
    from paper_2503_02236_b200.gpumodel import load_gpu_model
    from paper_2503_02236_b200.machine import plan_kernel
    cfg = codec.VQConfig(4, 8, 1, codec.Sharing.per_channel_group(4))
    for op in (rdf.ComputeOp.attention_decode(16, 32, 4096, 128), rdf.ComputeOp.gemv(4096, 4096)):
        ref = rsim.plan_kernel(cfg, op, rgm.load_gpu_model("rtx4090"))
        ours = plan_kernel(cfg, op, load_gpu_model("rtx4090"))
        assert (ours.cache_plan.n_reg, ours.cache_plan.n_shared) == (ref.cache_plan.n_reg, ref.cache_plan.n_shared)
        assert (ours.dataflow_plan.split_axis, ours.dataflow_plan.split_factor) == (
            ref.dataflow_plan.split_axis, ref.dataflow_plan.split_factor)
        assert ours.fusion_level == ref.fusion_level
