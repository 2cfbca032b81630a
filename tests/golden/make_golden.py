"""Generate tests/golden/golden.npz + golden.json by running the REAL reference.

Needs /root/reference (read-only) — run in the build container only:

    python tests/golden/make_golden.py

Nothing on the GPU box reads /root/reference; the tests consume the committed
fixtures. For every case the script records, straight from vqforge:
  * sha256 of codes / codebooks from synthetic_quantized (pins the oracle's RNG restatement)
  * sha256 + samples of dequantize() output (bit-exact target)
  * sha256 of QuantizedTensor.packed_codes() (bitpack format)
  * reference_compute() outputs and SimMachine.run_fused_kernel() outputs for the
    fused-op cases
  * plan_kernel() results for every preset x op x shipped GPU model
"""

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, HERE)

from cases import ATTENTION_CASES, DEQUANT_CASES, MATMUL_CASES, PRESETS_FOR_PLANS, QUANTIZE_CASES  # noqa: E402
from vqforge.codec import Sharing, VQConfig, dequantize, quantize  # noqa: E402
from vqforge.dataflow import ComputeOp  # noqa: E402
from vqforge.gpumodel import load_gpu_model  # noqa: E402
from vqforge.presets import PRESETS  # noqa: E402
from vqforge.sim import SimMachine, plan_kernel, reference_compute  # noqa: E402
from vqforge.synth import synthetic_quantized, synthetic_tensor  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make_cfg(v, bits, r, sharing, tile, gw):
    if sharing == "tile":
        sh = Sharing.per_tile(*tile)
    elif sharing == "channel_group":
        sh = Sharing.per_channel_group(gw)
    else:
        sh = Sharing.whole_tensor()
    return VQConfig(v, bits, r, sh)


def main():
    arrays, meta = {}, {"dequant": {}, "matmul": {}, "attention": {}, "plans": {}, "kat": {}, "quantize": {}}
    qts = {}
    for (name, shape, v, bits, r, sharing, tile, gw, seed, work) in DEQUANT_CASES:
        cfg = make_cfg(v, bits, r, sharing, tile, gw)
        q = synthetic_quantized(shape, cfg, seed, working_entries=work)
        qts[name] = (q, cfg, seed, work)
        books = np.stack([cb.entries for cb in q.codebooks])
        deq = dequantize(q)
        # fp16-rounded books (the device's default codebook dtype)
        q16 = synthetic_quantized(shape, cfg, seed, working_entries=work)
        for cb in q16.codebooks:
            cb.entries = cb.entries.astype(np.float16).astype(np.float32)
        deq16 = dequantize(q16)
        rng = np.random.default_rng(0)
        idx = rng.integers(0, deq.size, size=64)
        meta["dequant"][name] = {
            "n_regions": int(q.n_regions),
            "codes_sha": sha(q.codes), "books_sha": sha(books),
            "region_sha": sha(q.region_ids.astype(np.int64)),
            "dequant_sha": sha(deq), "dequant16_sha": sha(deq16),
            "packed_sha": hashlib.sha256(q.packed_codes()).hexdigest(),
            "packed_len": len(q.packed_codes()),
        }
        arrays[f"deq_idx_{name}"] = idx
        arrays[f"deq_val_{name}"] = deq.reshape(-1)[idx]

    for (name, base, kind, extra) in MATMUL_CASES:
        q, cfg, seed, work = qts[base]
        m, n = q.shape
        if kind == "gemv":
            op = ComputeOp.gemv(m, n, residuals=cfg.residuals)
            act = synthetic_tensor((m,), seed + 2)
        else:
            rows = extra["rows"]
            op = ComputeOp.gemm(m, n, rows, residuals=cfg.residuals)
            act = synthetic_tensor((rows, m), seed + 2)
        ref = reference_compute(op, {"activation": act, "weight": dequantize(q)})
        model = load_gpu_model("rtx4090")
        plans = plan_kernel(cfg, op, model)
        fused, rep = SimMachine(model).run_fused_kernel(q, plans, op, {"activation": act})
        arrays[f"mm_ref_{name}"] = ref
        arrays[f"mm_sim_{name}"] = fused
        meta["matmul"][name] = {"act_sha": sha(act), "reduce_bytes": int(rep.reduce_bytes)}

    for (name, base) in ATTENTION_CASES:
        kq, cfg, seed, work = qts[base]
        vq = synthetic_quantized(kq.shape, cfg, seed + 1, working_entries=work)
        b, h, t, c = kq.shape
        query = synthetic_tensor((b, h, c), seed + 2)
        op = ComputeOp.attention_decode(b, h, t, c, residuals=cfg.residuals)
        ref = reference_compute(op, {"query": query, "k": dequantize(kq), "v": dequantize(vq)})
        model = load_gpu_model("rtx4090")
        plans = plan_kernel(cfg, op, model)
        fused, _ = SimMachine(model).run_fused_kernel({"k": kq, "v": vq}, plans, op, {"query": query})
        arrays[f"at_ref_{name}"] = ref
        arrays[f"at_sim_{name}"] = fused
        meta["attention"][name] = {"v_codes_sha": sha(vq.codes), "query_sha": sha(query)}

    # online quantization: the reference's nearest-centroid quantize() with the
    # fp16-rounded codebooks the device holds
    for (name, base, dseed) in QUANTIZE_CASES:
        q, cfg, seed, work = qts[base]
        q16 = synthetic_quantized(q.shape, cfg, seed, working_entries=work)
        for cb in q16.codebooks:
            cb.entries = cb.entries.astype(np.float16).astype(np.float32)
        data = synthetic_tensor(q.shape, dseed).astype(np.float16).astype(np.float32)
        qq = quantize(data, q16.codebooks, cfg)
        arrays[f"qz_codes_{name}"] = qq.codes.astype(np.int32)
        meta["quantize"][name] = {"data_sha": sha(data), "codes_sha": sha(qq.codes.astype(np.int32))}

    # VQLF containers (V/container.py:25-49) of a few cases, byte for byte
    from vqforge.container import dump_quantized
    meta["vqlf"] = {}
    for name in ("aqlm3", "gptvq2_edge", "cg2d", "v16r3"):
        q, cfg, seed, work = qts[name]
        blob = dump_quantized(q)
        arrays[f"vqlf_{name}"] = np.frombuffer(blob, dtype=np.uint8)
        meta["vqlf"][name] = {"sha": hashlib.sha256(blob).hexdigest(), "len": len(blob)}

    # planner outputs at the reference's own configs and the BASELINE configs
    ops = {
        "gemm": lambda cfg: ComputeOp.gemm(4096, 4096, 256, residuals=cfg.residuals),
        "gemv": lambda cfg: ComputeOp.gemv(4096, 4096, residuals=cfg.residuals),
        "attention_decode": lambda cfg: ComputeOp.attention_decode(16, 32, 4096, 128,
                                                                   residuals=cfg.residuals),
    }
    configs = {p: PRESETS[p].config for p in PRESETS_FOR_PLANS}
    configs["quip2"] = VQConfig(8, 16, 1)
    configs["aqlm2x8"] = VQConfig(8, 8, 2)
    for model_name in ("rtx4090", "a40"):
        model = load_gpu_model(model_name)
        for pname, cfg in configs.items():
            for kind, mk in ops.items():
                op = mk(cfg)
                p = plan_kernel(cfg, op, model)
                fp = p.dataflow_plan
                meta["plans"][f"{model_name}/{pname}/{kind}"] = {
                    "n_reg": p.cache_plan.n_reg, "n_shared": p.cache_plan.n_shared,
                    "split_axis": fp.split_axis, "split_factor": fp.split_factor,
                    "switch_axes": list(fp.switch_axes), "region_tasks": fp.region_tasks,
                    "base_tiles": fp.base_tiles, "temporal_axes": list(fp.temporal_axes),
                    "fusion_level": p.fusion_level,
                    "n_shuffle": (p.schedule.n_shuffle if p.schedule else None),
                }

    # known-answer vectors (T/test_bitpack.py:10-46, T/test_sim.py:85-98)
    from vqforge.bitpack import pack_indices
    meta["kat"]["pack_12"] = list(pack_indices(np.array([0xABC, 0x123]), 12))
    meta["kat"]["pack_3"] = list(pack_indices(np.array([1, 2, 3, 4, 5, 6, 7, 0]), 3))
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print(f"wrote {len(arrays)} arrays, {sum(len(v) for v in meta.values())} records")


if __name__ == "__main__":
    main()
