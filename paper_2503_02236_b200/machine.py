"""B200 executor with the reference's fused-kernel operator API.

``B200Machine.run_fused_kernel(quantized, plans, op, operands) -> (out, SimReport)``
has the contract of ``SimMachine.run_fused_kernel`` (pkg/src/vqforge/sim.py:297-316):
same argument meaning, same output shapes (fp32 ndarray for ndarray inputs), same
errors (plan/op mismatch -> ConfigError, shape mismatch -> ShapeError, corrupt
codes -> CodeRangeError). The work runs in the sm_100a kernels behind the C ABI;
the SimReport carries the launch's algorithmic traffic and, in ``meta``, the
kernel that ran and (``measure=True``) its CUDA-event time.

``plan_kernel`` keeps the reference signature (sim.py:255-269). For the shipped
rtx4090 / a40 models it reproduces the reference plans exactly; for ``b200`` it
feeds compute_slack with the *measured* kernel usage (vqb_query_usage on the
loaded cubin, sim.py:53-57 used constants) and sizes the shared tier for the
kernels' replicated, conflict-free layout.
"""

import weakref
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .cacheplan import CachePlan, compute_slack, plan_b200_tiers, plan_cache
from .codec import Codebook, QuantizedTensor, VQConfig
from .dataflow import ATTENTION, GEMM, GEMV, ComputeOp, DataflowPlan, b200_split, build_dataflow
from .errors import CapacityError, ConfigError, ShapeError
from .fusion import (B200_GEMV_MAX_ROWS, B200_GEMV_TC_MAX_ROWS, STYLE_MMA, STYLE_STRIDED, THRES_SHUFFLE, LayoutPair, MappingError,
                     ShuffleSchedule, b200_fusion, build_shuffle_schedule, choose_fusion_level)
from .gpumodel import GpuModel, KernelUsage, load_gpu_model
from .report import SimReport

# the reference's modelled per-kernel usage (sim.py:53-57), used for non-B200 models
KERNEL_USAGE = {
    GEMM: KernelUsage(shared_bytes=32768, regs_per_thread=64, threads_per_block=256),
    GEMV: KernelUsage(shared_bytes=8192, regs_per_thread=40, threads_per_block=256),
    ATTENTION: KernelUsage(shared_bytes=8192, regs_per_thread=32, threads_per_block=256),
}
# B200 kernels without their codebook span (used when no GPU is visible to query)
B200_KERNEL_USAGE = {
    GEMM: KernelUsage(shared_bytes=131072, regs_per_thread=128, threads_per_block=256),
    GEMV: KernelUsage(shared_bytes=8192 + 128, regs_per_thread=48, threads_per_block=256),
    ATTENTION: KernelUsage(shared_bytes=8448 + 128, regs_per_thread=128, threads_per_block=512),
}

VARIANTS = ("gc", "sc", "o1", "o2", "o3", "o4")
N_FLAG_NO_SHARED = 2  # VQB_FLAG_NO_SHARED


@dataclass
class FusedPlans:
    cache_plan: CachePlan
    dataflow_plan: DataflowPlan
    fusion_level: str
    schedule: Optional[ShuffleSchedule] = None


def fusion_for(config: VQConfig, op: ComputeOp, thres_shuffle: int = THRES_SHUFFLE):
    layouts = LayoutPair(config.vector_size, op.required_layout)
    level = choose_fusion_level(layouts, thres_shuffle)
    schedule = None
    if level == "register":
        try:
            schedule = build_shuffle_schedule(layouts, STYLE_MMA if op.kind == GEMM else STYLE_STRIDED)
        except MappingError:
            level = "shared"
    return level, schedule


def measured_usage(kind: str) -> Optional[KernelUsage]:
    """Real usage of the B200 kernel family (cudaFuncGetAttributes), minus the codebook span."""
    try:
        import torch
        if not torch.cuda.is_available():
            return None
        from . import _native as N
        u = N.VqbUsage()
        k = {GEMV: N.KERNEL_GEMV, GEMM: N.KERNEL_GEMM, ATTENTION: N.KERNEL_ATTN}[kind]
        N.check(N.lib().vqb_query_usage(k, None, u))
        if u.threads_per_block <= 0:
            return None
        span = {GEMV: 256 * 128, ATTENTION: 2 * 256 * 128 * 2, GEMM: 0}[kind]
        return KernelUsage(max(u.shared_bytes - span, 0), u.regs_per_thread, u.threads_per_block)
    except Exception:
        return None


def _proto(config: VQConfig) -> Codebook:
    return Codebook(np.zeros((config.n_entries, config.vector_size), np.float32), 0, 0)


def plan_kernel(config: VQConfig, op: ComputeOp, model: Optional[GpuModel] = None,
                kernel_usage: Optional[KernelUsage] = None, histogram=None, n_reg: Optional[int] = None,
                n_shared: Optional[int] = None, split_factor: Optional[int] = None,
                thres_shuffle: int = THRES_SHUFFLE) -> FusedPlans:
    """FusedPlans for (config, op, model), the reference signature (sim.py:255-269).

    Reference models (rtx4090, a40) get the reference's plans exactly. The b200
    model gets the plan the sm_100a kernels launch with: tiers from the real
    cubin's shared-memory slack and (if given) a measured access histogram
    (cacheplan.plan_b200_tiers), the persistent kernels' split granularity
    (dataflow.b200_split) and the kernel family's fusion level (fusion.b200_fusion).
    ``run_fused_kernel`` turns every field into a launch parameter."""
    model = model or load_gpu_model("b200")
    if model.name != "b200":
        usage = kernel_usage or KERNEL_USAGE[op.kind]
        cache = plan_cache(_proto(config), histogram, compute_slack(usage, model), n_reg=n_reg, n_shared=n_shared)
        flow = build_dataflow(config, op, model, split_factor=split_factor)
        level, schedule = fusion_for(config, op, thres_shuffle)
        return FusedPlans(cache, flow, level, schedule)
    usage = kernel_usage or measured_usage(op.kind) or B200_KERNEL_USAGE[op.kind]
    shared_slack, _ = compute_slack(usage, model)
    levels = config.residuals if op.kind != ATTENTION else 1
    reg, shared = plan_b200_tiers(config.n_entries, config.vector_size, levels, shared_slack,
                                  histogram=histogram, n_reg=n_reg, n_shared=n_shared)
    cache = CachePlan(reg, shared, config.n_entries, config.entry_bytes)
    axis, f = b200_split(op, model.sm_count)
    if split_factor is not None:
        f = int(split_factor)
    flow = build_dataflow(config, op, model, split_factor=None)
    from .cacheplan import hot_register_slots
    flow = DataflowPlan(flow.op_kind, flow.switch_axes, flow.global_reduce_axes, axis, f,
                        dict(flow.region_tasks, **{axis: max(f, 1)}), flow.base_tiles, flow.temporal_axes,
                        meta={"model": "b200", "split": "persistent-kernel granularity (dataflow.b200_split)",
                              "hot_entries": (int(histogram.hot_set().size) if histogram is not None else None),
                              "hot_register_slots": hot_register_slots(histogram)})
    level = b200_fusion(op.kind, op.activation_rows)
    schedule = None
    if level == "register":
        _, schedule = fusion_for(config, op, thres_shuffle)
    return FusedPlans(cache, flow, level, schedule)


def launch_of(plans: FusedPlans, op: ComputeOp):
    """VqbLaunch carrying every field of the plan the kernels read: n_reg (register
    slots), n_shared (shared span; codes beyond it use the global tier),
    split_axis/split_factor (M for the GEMV's stream-K granularity, T for the
    attention's span split; splits over other axes are not a launch parameter of
    these kernels and are dropped)."""
    from .ops import launch_struct
    L = launch_struct(plans)
    ax = plans.dataflow_plan.split_axis
    ok = (op.kind in (GEMV, GEMM) and ax == "M") or (op.kind == ATTENTION and ax == "T")
    if not ok:
        L.split_factor, L.split_axis = 0, 0
    return L


class B200Machine:
    """Drop-in for SimMachine backed by the sm_100a kernels."""

    def __init__(self, model: Optional[GpuModel] = None, thres_shuffle: int = THRES_SHUFFLE,
                 codebook_dtype: str = "float16", activation_dtype: Optional[str] = None,
                 device=None, measure: bool = False):
        import torch

        from .device import default_device, torch_dtype

        self.model = model or load_gpu_model("b200")
        self.thres_shuffle = thres_shuffle
        self.device = default_device(device)
        self.codebook_dtype = torch_dtype(codebook_dtype)
        if activation_dtype is None:
            activation_dtype = "float32" if self.codebook_dtype == torch.float32 else "float16"
        self.activation_dtype = torch_dtype(activation_dtype)
        self.measure = measure
        self._cache = {}

    # -- device residency ---------------------------------------------------------------------

    def to_device(self, q):
        from .device import DeviceVQTensor

        if isinstance(q, DeviceVQTensor):
            return q
        key = id(q)
        hit = self._cache.get(key)
        if hit is not None and hit[0]() is q:
            return hit[1]
        d = DeviceVQTensor.from_quantized(q, device=self.device, codebook_dtype=self.codebook_dtype)
        try:
            ref = weakref.ref(q, lambda _r, k=key: self._cache.pop(k, None))
        except TypeError:
            return d
        self._cache[key] = (ref, d)
        return d

    def _operand(self, x):
        import torch

        if isinstance(x, torch.Tensor):
            return x.to(self.device, self.activation_dtype), False
        return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(
            self.device).to(self.activation_dtype), True

    # -- public entry points ------------------------------------------------------------------

    def run_fused_kernel(self, quantized, plans: FusedPlans, op: ComputeOp, operands: dict):
        if plans.dataflow_plan.op_kind != op.kind:
            raise ConfigError(f"dataflow plan for {plans.dataflow_plan.op_kind} used with {op.kind}")
        cfg = _config_of(quantized)
        if plans.cache_plan.n_entries != cfg.n_entries:
            raise ConfigError(f"cache plan over {plans.cache_plan.n_entries} entries used with "
                              f"{cfg.n_entries}-entry codebooks")
        L = launch_of(plans, op)
        return self._execute(quantized, op, operands, L, plans, variant="o4")

    def run_variant(self, name: str, quantized, op: ComputeOp, operands: dict,
                    plans: Optional[FusedPlans] = None):
        """One rung of the reference's ladder (sim.py:211-226) mapped to launch knobs:
        gc = every lookup from global/L2, sc = whole book in shared memory, o1..o4 = planned."""
        key = name.lower()
        if key not in VARIANTS:
            raise ConfigError(f"unknown variant {name!r}")
        cfg = _config_of(quantized)
        plans = plans or plan_kernel(cfg, op, self.model, thres_shuffle=self.thres_shuffle)
        from .ops import launch_struct

        if key == "gc":
            L = launch_struct()
            L.flags |= N_FLAG_NO_SHARED
        elif key == "sc":
            L = launch_struct(n_shared=min(cfg.n_entries, 1024))
        else:
            L = launch_struct(plans)
            L.split_factor, L.split_axis = 0, 0
        return self._execute(quantized, op, operands, L, plans, variant=key)

    def run_baseline_kernel(self, quantized, variant: str, op: ComputeOp, operands: dict):
        if variant.lower() not in ("gc", "sc"):
            raise ConfigError(f"baseline variant must be GC or SC, got {variant}")
        return self.run_variant(variant, quantized, op, operands)

    def run_dense(self, op: ComputeOp, operands: dict):
        """fp16 dense baseline on the GPU: cuBLAS for GEMM/GEMV, SDPA for attention."""
        import torch

        rep = SimReport(meta={"variant": "fp16"})
        t = {k: torch.from_numpy(np.asarray(v, np.float32)).to(self.device).half() for k, v in operands.items()}
        if op.kind in (GEMM, GEMV):
            a = t["activation"]
            out = (a.view(1, -1) if a.dim() == 1 else a) @ t["weight"]
            out = out[0] if op.kind == GEMV else out
        else:
            q = t["query"].unsqueeze(2)
            out = torch.nn.functional.scaled_dot_product_attention(q, t["k"], t["v"])[:, :, 0]
        rep.global_bytes = 2 * sum(int(np.asarray(v).size) for v in operands.values()) + 2 * out.numel()
        return out.float().cpu().numpy(), rep

    # -- execution ------------------------------------------------------------------------------

    def _execute(self, quantized, op, operands, L, plans, variant):
        import torch

        from . import _native as N
        from .ops import vq_attention, vq_gemm, vq_gemv

        rep = SimReport(meta={"variant": variant})
        cfg = _config_of(quantized)
        ev = None
        if self.measure:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        if op.kind == ATTENTION:
            kq, vq = quantized["k"], quantized["v"]
            shape = tuple(op.axes[a] for a in "BHTC")
            if tuple(kq.shape) != shape or tuple(vq.shape) != shape:
                raise ShapeError(f"quantized KV shape {tuple(kq.shape)} does not match op axes {shape}")
            q = operands["query"]
            qshape = tuple(q.shape)
            if qshape != (shape[0], shape[1], shape[3]):
                raise ShapeError(f"query shape {qshape} != {(shape[0], shape[1], shape[3])}")
            kd, vd = self.to_device(kq), self.to_device(vq)
            qt, host = self._operand(q)
            if ev:
                ev[0].record()
            out = vq_attention(kd, vd, qt, out_dtype=torch.float32, launch=L)
            n_codes = 2 * kd.n_subvectors * cfg.residuals
            code_bytes = 2 * ((kd.n_subvectors * cfg.residuals * cfg.log2_entries + 7) // 8)
            rep.global_bytes = code_bytes + 2 * int(np.prod(qshape)) + 2 * out.numel()
            rep.global_to_shared_bytes = 2 * kd.n_regions * cfg.residuals * min(cfg.n_entries, 256) * cfg.entry_bytes
            nt = -(-shape[2] // 512)
            rep.reduce_bytes = (nt * op.output_bytes()) if nt > 1 else 0
        else:
            w = quantized if not isinstance(quantized, dict) else quantized["weight"]
            m, n = op.axes["M"], op.axes["N"]
            if tuple(w.shape) != (m, n):
                raise ShapeError(f"quantized weight {tuple(w.shape)} != {(m, n)}")
            a = operands["activation"]
            ashape = tuple(a.shape)
            if ashape[-1] != m or len(ashape) > 2:
                raise ShapeError(f"activation {ashape} does not match M={m}")
            wd = self.to_device(w)
            at, host = self._operand(a)
            # fusion level -> kernel family: "register" = lookups feed the consumer's
            # registers (GEMV kernels, rows <= 4); "shared" = dequantized tiles staged
            # in shared memory for tcgen05 (the decode GEMV to 64 rows, then the GEMM). One activation row always takes the
            # GEMV (a 128-row MMA tile would be 1/128 used).
            rows = 1 if at.dim() == 1 else at.shape[0]
            gemv_ok = rows <= B200_GEMV_MAX_ROWS and rows in (1, 2, 4)
            # shared level at 5-64 rows: the tcgen05 decode GEMV (batch = UMMA N)
            tc_gemv = plans.fusion_level == "shared" and B200_GEMV_MAX_ROWS < rows <= B200_GEMV_TC_MAX_ROWS
            use_gemv = op.kind == GEMV or tc_gemv or (gemv_ok and (plans.fusion_level == "register" or rows == 1))
            fn = vq_gemv if use_gemv else vq_gemm
            if ev:
                ev[0].record()
            out = fn(wd, at, out_dtype=torch.float32, launch=L)
            if op.kind == GEMV and out.dim() == 2:
                out = out[0]
            n_codes = wd.n_subvectors * cfg.residuals
            rep.global_bytes = (n_codes * cfg.log2_entries + 7) // 8 + 2 * int(np.prod(ashape)) + 2 * out.numel()
            rep.global_to_shared_bytes = wd.n_regions * cfg.residuals * max(L.n_shared, 0) * cfg.entry_bytes
            if L.split_factor > 1:
                rep.reduce_bytes = L.split_factor * op.output_bytes()
        if ev:
            ev[1].record()
            torch.cuda.synchronize()
            rep.meta["us"] = ev[0].elapsed_time(ev[1]) * 1e3
        rep.meta["kernel"] = N.last_kernel()
        rep.meta["device"] = torch.cuda.get_device_name(self.device)
        rep.occupancy = self._occupancy(op.kind)
        rep.validate()
        return (out.cpu().numpy() if host else out), rep

    def _occupancy(self, kind) -> int:
        u = measured_usage(kind)
        if u is None:
            return 1
        try:
            return max(self.model.occupancy_of(u), 1)
        except Exception:
            return 1


def _config_of(quantized) -> VQConfig:
    if isinstance(quantized, dict):
        return (quantized.get("k") or quantized.get("weight")).config
    return quantized.config
