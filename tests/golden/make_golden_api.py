"""Generate tests/golden/golden_api.{npz,json}: the reference's own operator-API
numeric test bodies, run through the REAL vqforge (needs /root/reference; run in
the build container only):

    python tests/golden/make_golden_api.py

For every cell of cases.API_CELLS it records, straight from vqforge:
  * sha256 of the weight / K / V codes and books and of the operand (the GPU-side
    tests rebuild the inputs with the oracle's seeded generator and must hit these)
  * reference_compute() on the dequantized operands (the oracle output the B200
    executor is held to, 1e-4 rel-to-max in fp32 parity mode)
  * SimMachine.run_fused_kernel() output and the FusedPlans summary for rtx4090
Nothing on the GPU box reads /root/reference.
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

from cases import API_CELLS, API_VARIANT_CELLS  # noqa: E402
from vqforge.codec import Sharing, VQConfig, dequantize  # noqa: E402
from vqforge.dataflow import ComputeOp  # noqa: E402
from vqforge.gpumodel import load_gpu_model  # noqa: E402
from vqforge.sim import SimMachine, plan_kernel, reference_compute  # noqa: E402
from vqforge.synth import synthetic_quantized, synthetic_tensor  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make_cfg(spec):
    v, bits, r, sharing, tile, gw = spec
    if sharing == "tile":
        sh = Sharing.per_tile(*tile)
    elif sharing == "channel_group":
        sh = Sharing.per_channel_group(gw)
    else:
        sh = Sharing.whole_tensor()
    return VQConfig(v, bits, r, sh)


def build(cell):
    name, spec, kind, dims, seed, work = cell
    cfg = make_cfg(spec)
    if kind == "attention_decode":
        b, h, t, c = dims
        op = ComputeOp.attention_decode(b, h, t, c, residuals=cfg.residuals)
        kq = synthetic_quantized((b, h, t, c), cfg, seed, working_entries=work)
        vq = synthetic_quantized((b, h, t, c), cfg, seed + 1, working_entries=work)
        operands = {"query": synthetic_tensor((b, h, c), seed + 2)}
        dense = {"query": operands["query"], "k": dequantize(kq), "v": dequantize(vq)}
        return cfg, op, {"k": kq, "v": vq}, operands, dense
    m, n, rows = dims
    if kind == "gemm":
        op = ComputeOp.gemm(m, n, rows, residuals=cfg.residuals)
        act = synthetic_tensor((rows, m), seed + 2)
    else:
        op = ComputeOp.gemv(m, n, residuals=cfg.residuals)
        act = synthetic_tensor((m,), seed + 2)
    wq = synthetic_quantized((m, n), cfg, seed, working_entries=work)
    return cfg, op, wq, {"activation": act}, {"activation": act, "weight": dequantize(wq)}


def main():
    model = load_gpu_model("rtx4090")
    machine = SimMachine(model)
    arrays, meta = {}, {}
    for cell in API_CELLS:
        name = cell[0]
        cfg, op, quantized, operands, dense = build(cell)
        ref = reference_compute(op, dense)
        plans = plan_kernel(cfg, op, model)
        sim, _ = machine.run_fused_kernel(quantized, plans, op, operands)
        qs = quantized if isinstance(quantized, dict) else {"weight": quantized}
        rec = {
            "codes_sha": {k: sha(q.codes) for k, q in qs.items()},
            "books_sha": {k: sha(np.stack([cb.entries for cb in q.codebooks])) for k, q in qs.items()},
            "operand_sha": {k: sha(v) for k, v in operands.items()},
            "plans": {"n_reg": plans.cache_plan.n_reg, "n_shared": plans.cache_plan.n_shared,
                      "split_axis": plans.dataflow_plan.split_axis,
                      "split_factor": plans.dataflow_plan.split_factor,
                      "fusion_level": plans.fusion_level},
            "sim_rel": float(np.abs(sim - ref).max() / max(np.abs(ref).max(), 1e-12)),
        }
        if name in API_VARIANT_CELLS:
            rec["variants_rel"] = {}
            for var in ("gc", "sc", "o1", "o2", "o3", "o4"):
                out, _ = machine.run_variant(var, quantized, op, operands, plans)
                rec["variants_rel"][var] = float(np.abs(out - ref).max() / np.abs(ref).max())
        arrays[f"ref_{name}"] = ref.astype(np.float32)
        meta[name] = rec
        print(name, rec["sim_rel"], flush=True)
    np.savez_compressed(os.path.join(HERE, "golden_api.npz"), **arrays)
    with open(os.path.join(HERE, "golden_api.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print(f"wrote {len(arrays)} arrays")


if __name__ == "__main__":
    main()
