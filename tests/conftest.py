import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, GOLDEN):
    if p not in sys.path:
        sys.path.insert(0, p)

from cases import ATTENTION_CASES, DEQUANT_CASES, MATMUL_CASES, QUANTIZE_CASES  # noqa: E402
from oracle import vq_oracle as O  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libvqb.so")
    config.addinivalue_line("markers", "slow: long-running full-size parity checks")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def golden_meta():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


def golden_arrays():
    return np.load(os.path.join(GOLDEN, "golden.npz"))


CASES = {c[0]: c for c in DEQUANT_CASES}


class Case:
    """One golden case rebuilt with the oracle's seeded generator."""

    def __init__(self, name, seed_offset=0, books_f16=False):
        (self.name, shape, v, bits, r, sharing, tile, gw, seed, work) = CASES[name]
        self.shape, self.v, self.bits, self.R = tuple(shape), v, bits, r
        self.sharing, self.tile, self.gw, self.seed, self.work = sharing, tile, gw, seed + seed_offset, work
        self.n_regions = O.n_regions_of(self.shape, v, sharing, tile, gw)
        self.codes, self.books = O.synthetic_codes_books(self.shape, v, bits, r, self.n_regions,
                                                         self.seed, working_entries=work)
        if books_f16:
            self.books = O.round_f16(self.books)
        self.regions = O.region_ids(self.shape, v, sharing, tile, gw)

    def dense(self):
        return O.dequantize(self.codes, self.books, self.shape, self.v, self.n_regions, self.regions)

    def config(self):
        from paper_2503_02236_b200.codec import Sharing, VQConfig
        if self.sharing == "tile":
            sh = Sharing.per_tile(*self.tile)
        elif self.sharing == "channel_group":
            sh = Sharing.per_channel_group(self.gw)
        else:
            sh = Sharing.whole_tensor()
        return VQConfig(self.v, self.bits, self.R, sh)

    def quantized(self):
        from paper_2503_02236_b200.codec import Codebook, QuantizedTensor
        nreg = self.n_regions
        books = [Codebook(self.books[i], residual_level=i // nreg, region_id=i % nreg)
                 for i in range(self.books.shape[0])]
        return QuantizedTensor(codes=self.codes, shape=self.shape, config=self.config(),
                               codebooks=books, n_regions=nreg)


@pytest.fixture(scope="session")
def meta():
    return golden_meta()


@pytest.fixture(scope="session")
def arrays():
    return golden_arrays()
