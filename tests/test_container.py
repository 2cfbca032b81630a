"""VQLF container (V/container.py:25-94): the writer is byte-identical to the
reference's dump_quantized; the reader parses reference blobs; the device ingest
(packed stream unpacked and interleaved on the GPU) dequantizes bit-exactly."""

import hashlib

import numpy as np
import pytest
from conftest import Case

NAMES = ("aqlm3", "gptvq2_edge", "cg2d", "v16r3")


@pytest.mark.parametrize("name", NAMES)
def test_dump_is_byte_identical_to_reference(name, meta):
    from paper_2503_02236_b200.container import dump_vqlf
    blob = dump_vqlf(Case(name).quantized())
    assert hashlib.sha256(blob).hexdigest() == meta["vqlf"][name]["sha"]
    assert len(blob) == meta["vqlf"][name]["len"]


@pytest.mark.parametrize("name", NAMES)
def test_parse_reference_blob(name, arrays):
    from paper_2503_02236_b200.container import parse_header
    c = Case(name)
    cfg, shape, n_regions, books, levels, regions, bits, off = parse_header(arrays[f"vqlf_{name}"].tobytes())
    assert shape == c.shape and n_regions == c.n_regions
    assert (cfg.vector_size, cfg.log2_entries, cfg.residuals, cfg.sharing.kind) == (c.v, c.bits, c.R, c.sharing)
    order = np.argsort(levels * n_regions + regions, kind="stable")
    assert np.array_equal(books[order], c.books)
    assert bits == c.codes.size * c.bits


def test_bad_magic_and_version(arrays):
    from paper_2503_02236_b200.container import parse_header
    from paper_2503_02236_b200.errors import ConfigError
    blob = bytearray(arrays["vqlf_v16r3"].tobytes())
    with pytest.raises(ConfigError, match="bad magic"):
        parse_header(b"XXXX" + bytes(blob[4:]))
    blob[4] = 9
    with pytest.raises(ConfigError, match="unsupported container version"):
        parse_header(bytes(blob))


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_device_ingest_dequant_bit_exact(name, arrays, meta):
    torch = pytest.importorskip("torch")
    from paper_2503_02236_b200 import ops
    from paper_2503_02236_b200.container import load_vqlf
    d = load_vqlf(arrays[f"vqlf_{name}"].tobytes(), device=torch.device("cuda", 0), codebook_dtype="float32")
    out = ops.vq_dequantize(d).cpu().numpy()
    assert hashlib.sha256(np.ascontiguousarray(out).tobytes()).hexdigest() == meta["dequant"][name]["dequant_sha"]
