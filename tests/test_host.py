"""Host-side mirror of the reference API (no GPU): containers, bitpack, planner,
profiling, fusion schedules — checked against the reference's golden outputs
and its own known-answer tests."""

import hashlib

import numpy as np
import pytest
from conftest import CASES, Case
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2503_02236_b200 import bitpack
from paper_2503_02236_b200.cacheplan import (CachePlan, b200_shared_entries, cache_access,
                                             cache_access_bulk, cache_load, cache_switch, compute_slack,
                                             plan_cache)
from paper_2503_02236_b200.codec import (Codebook, QuantizedTensor, Sharing, VQConfig, compression_ratio,
                                         region_layout)
from paper_2503_02236_b200.dataflow import ComputeOp, build_dataflow, solve_split_factor
from paper_2503_02236_b200.errors import CodeRangeError, ConfigError, ShapeError
from paper_2503_02236_b200.fusion import (STYLE_MMA, STYLE_STRIDED, LayoutPair, build_shuffle_schedule,
                                          dequant_register_file, expected_compute_ownership,
                                          run_shuffle_steps, shuffle_count)
from paper_2503_02236_b200.gpumodel import KernelUsage, load_gpu_model
from paper_2503_02236_b200.machine import KERNEL_USAGE, plan_kernel
from paper_2503_02236_b200.presets import PRESET_ORDER, PRESETS, load_preset
from paper_2503_02236_b200.profiling import AccessHistogram, profile_accesses, reorder_all


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---- containers ---------------------------------------------------------------------------------

@pytest.mark.parametrize("name", sorted(CASES))
def test_region_layout_matches_reference(name, meta):
    c = Case(name)
    n, ids = region_layout(c.shape, c.config())
    assert n == meta["dequant"][name]["n_regions"]
    assert sha(ids.astype(np.int64)) == meta["dequant"][name]["region_sha"]


@pytest.mark.parametrize("name", sorted(CASES))
def test_packed_stream_matches_reference(name, meta):
    q = Case(name).quantized()
    stream = q.packed_codes()
    assert len(stream) == meta["dequant"][name]["packed_len"]
    assert hashlib.sha256(stream).hexdigest() == meta["dequant"][name]["packed_sha"]
    back = bitpack.unpack_indices(stream, q.config.log2_entries, q.codes.size)
    assert np.array_equal(back.reshape(q.codes.shape), q.codes)


def test_bitpack_known_answers(meta):
    assert bitpack.packed_length(2, 12) == 3
    assert list(bitpack.pack_indices(np.array([0xABC, 0x123]), 12)) == meta["kat"]["pack_12"]
    assert list(bitpack.pack_indices(np.array([1, 2, 3, 4, 5, 6, 7, 0]), 3)) == meta["kat"]["pack_3"]
    with pytest.raises(CodeRangeError):
        bitpack.pack_indices(np.array([16]), 4)
    with pytest.raises(ValueError, match="truncated"):
        bitpack.unpack_indices(b"\x01", 12, 2)


@given(st.integers(1, 16), st.lists(st.integers(0, 2 ** 16 - 1), max_size=200))
@settings(max_examples=60, deadline=None)
def test_bitpack_roundtrip(bits, vals):
    vals = np.array([v % (1 << bits) for v in vals], dtype=np.int64)
    data = bitpack.pack_indices(vals, bits)
    assert len(data) == bitpack.packed_length(vals.size, bits)
    assert np.array_equal(bitpack.unpack_indices(data, bits, vals.size), vals)


def test_config_validation():
    with pytest.raises(ConfigError):
        VQConfig(3, 8, 1)
    with pytest.raises(ConfigError):
        VQConfig(4, 0, 1)
    with pytest.raises(ConfigError):
        VQConfig(4, 8, 1, Sharing.per_channel_group(6))
    with pytest.raises(ConfigError):
        Sharing("diagonal")
    with pytest.raises(ShapeError):
        region_layout((4, 6), VQConfig(4, 8, 1))
    with pytest.raises(ShapeError):
        QuantizedTensor(np.zeros((1, 3), np.int32), (4, 4), VQConfig(4, 2, 1),
                        [Codebook(np.zeros((4, 4)), 0, 0)], 1)


def test_compression_ratios():
    want = [("quip4", 0.25), ("aqlm3", 0.1875), ("gptvq2", 0.125), ("cq4", 0.25), ("cq2", 0.125)]
    assert [(n, compression_ratio(PRESETS[n].config)) for n, _ in want] == want
    assert compression_ratio(load_preset("quip2").config) == 0.125
    assert compression_ratio(load_preset("aqlm2x8").config) == 0.125


# ---- planner: identical to the reference on its own GPU models --------------------------------------

def _configs():
    out = {p: PRESETS[p].config for p in PRESET_ORDER}
    out["quip2"] = load_preset("quip2").config
    out["aqlm2x8"] = load_preset("aqlm2x8").config
    return out


OPS = {
    "gemm": lambda cfg: ComputeOp.gemm(4096, 4096, 256, residuals=cfg.residuals),
    "gemv": lambda cfg: ComputeOp.gemv(4096, 4096, residuals=cfg.residuals),
    "attention_decode": lambda cfg: ComputeOp.attention_decode(16, 32, 4096, 128, residuals=cfg.residuals),
}


@pytest.mark.parametrize("model", ["rtx4090", "a40"])
def test_plan_kernel_matches_reference(model, meta):
    m = load_gpu_model(model)
    for pname, cfg in _configs().items():
        for kind, mk in OPS.items():
            want = meta["plans"][f"{model}/{pname}/{kind}"]
            p = plan_kernel(cfg, mk(cfg), m)
            fp = p.dataflow_plan
            got = {"n_reg": p.cache_plan.n_reg, "n_shared": p.cache_plan.n_shared,
                   "split_axis": fp.split_axis, "split_factor": fp.split_factor,
                   "switch_axes": list(fp.switch_axes), "region_tasks": fp.region_tasks,
                   "base_tiles": fp.base_tiles, "temporal_axes": list(fp.temporal_axes),
                   "fusion_level": p.fusion_level,
                   "n_shuffle": p.schedule.n_shuffle if p.schedule else None}
            assert got == want, (model, pname, kind)


def test_b200_plans_fit_and_are_conflict_free_layout():
    b200 = load_gpu_model("b200")
    for pname, cfg in _configs().items():
        for kind, mk in OPS.items():
            p = plan_kernel(cfg, mk(cfg), b200)
            assert p.cache_plan.n_reg == 0
            assert 0 <= p.cache_plan.n_shared <= cfg.n_entries
    # the replicated layout: 128 B per resident entry (<= 16-byte entries)
    assert b200_shared_entries(32768, 8, 65536) == 256
    assert b200_shared_entries(32768, 4, 256) == 256
    assert b200_shared_entries(65536, 16, 65536) == 256


@given(st.integers(1, 10 ** 6), st.integers(1, 10 ** 9), st.sampled_from([1, 2, 4, 12, 16, 64, 96, 256]))
@settings(max_examples=80, deadline=None)
def test_split_factor_is_optimal(out, cb, extent):
    f = solve_split_factor(out, cb, extent)
    divs = [d for d in range(1, extent + 1) if extent % d == 0]
    cost = {d: d * out + cb / d for d in divs}
    best = min(cost.values())
    assert abs(cost[f] - best) <= 1e-9 * max(1.0, best)
    assert f == min(d for d in divs if abs(cost[d] - best) <= 1e-9 * max(1.0, best))


def test_dataflow_examples():
    gptvq = PRESETS["gptvq2"].config
    # the paper's GPTVQ GeMM: every two naive blocks load the same 256-col book
    flow = build_dataflow(gptvq, ComputeOp.gemm(512, 512, 8))
    assert flow.switch_axes == ("M", "N")
    with pytest.raises(ShapeError):
        build_dataflow(gptvq, ComputeOp.gemv(4096, 4096), split_factor=3)


def test_slack_and_occupancy():
    m = load_gpu_model("rtx4090")
    u = KERNEL_USAGE["gemv"]
    s = compute_slack(u, m)
    occ = m.occupancy_of(u)
    assert m.occupancy(u.shared_bytes + s[0], u.regs_per_thread + s[1] // 4, u.threads_per_block) == occ
    assert m.occupancy(0, 0, 4096) == 0
    b200 = load_gpu_model("b200")
    assert b200.occupancy(200 * 1024, 128, 512) == 1


def test_cache_primitives():
    book = Codebook(np.arange(32, dtype=np.float32).reshape(8, 4), 0, 0)
    plan = CachePlan(2, 6, 8, 8)
    h = cache_load(book, plan)
    assert h.counters.global_to_shared_bytes == 32 and h.counters.global_bytes == 16
    assert cache_access(h, 1)[1] == "reg" and cache_access(h, 3)[1] == "shared"
    assert cache_access(h, 7)[1] == "global"
    cache_access_bulk(h, [0, 2, 6, 7])
    with pytest.raises(ConfigError):
        cache_access(h, 8)
    h2 = cache_switch(h, Codebook(np.zeros((8, 4)), 0, 1))
    assert h2.counters is h.counters
    with pytest.raises(ConfigError):
        plan_cache(book, AccessHistogram(np.arange(8)), (0, 0))


# ---- fusion: the reference's exhaustive ownership oracle ------------------------------------------

def test_shuffle_counts_table():
    table = {(8, 2): 3, (8, 1): 7, (4, 2): 1, (4, 1): 3, (2, 1): 1}
    for (v, dst), want in table.items():
        assert shuffle_count(v, dst) == want


def test_schedules_deliver_compute_layout():
    checked = 0
    for src in (2, 4, 8):
        for dst in (1, 2, 4):
            if src < dst:
                continue
            styles = [STYLE_STRIDED] + ([STYLE_MMA] if dst == 2 and src >= 4 else [])
            for style in styles:
                sch = build_shuffle_schedule(LayoutPair(src, dst), style)
                got = run_shuffle_steps(sch, dequant_register_file(sch))
                assert np.array_equal(got, expected_compute_ownership(sch)), (src, dst, style)
                checked += 1
    assert checked >= 8
    sch = build_shuffle_schedule(LayoutPair(8, 2), STYLE_MMA)
    assert sch.offsets == (1, 2, 3)


# ---- profiling: pure relabelling -------------------------------------------------------------------

def test_reorder_is_relabelling_and_sorted():
    from oracle import vq_oracle as O
    c = Case("cq2")
    q = c.quantized()
    # skew the codes
    q.codes[0] = O.zipf_codes(q.codes.shape[1], 256, seed=3)
    q2, perms = reorder_all(q)
    for h in profile_accesses(q2):
        assert (np.diff(h.counts) <= 0).all()
    regs = O.region_ids(q.shape, q.config.vector_size, "channel_group", group_width=4)
    books = np.stack([cb.entries for cb in q.codebooks])
    books2 = np.stack([cb.entries for cb in q2.codebooks])
    d1 = O.dequantize(q.codes, books, q.shape, 4, q.n_regions, regs)
    d2 = O.dequantize(q2.codes, books2, q.shape, 4, q.n_regions, regs)
    assert np.array_equal(d1, d2)
    h = AccessHistogram(np.array([100] + [1] * 63))
    assert h.hot_set().tolist() == [0]
