"""Benchmark of the fused VQ hot path on B200 (driver contract: one JSON line).

Workload (BASELINE.json configs[1], the config the metric is quoted on): the
decode-step linears of Llama-7B under QuiP#-style E8 VQ (VQConfig(8, 16, 1),
whole-tensor 2^16-entry codebook, codes drawn from the 256-entry working set),
batch 1. A step = one fused VQ GEMV over every linear of all 32 layers (q/k/v
fused as one 4096x12288 GEMV, o 4096x4096, gate/up fused 4096x22016, down
11008x4096: 128 launches), replayed as one CUDA graph. The 1.6 GB of codes is
> L2 (126 MB), so no flush is needed between steps.

value      whole-job algorithmic GB/s (codes + working-set codebook + x + y bytes)
e2e        the same through VQLinearStack.run with pinned host buffers (H2D of all
           activations, D2H of all outputs inside the timed region)
roofline   the dominant kernel (gemv_fast) against MEASURED_PEAKS.json hbm_gbs
cpu_baseline  the numpy oracle (dequantize + fp32 matmul) on a bounded sample
extra keys C4 decode attention and C1 GPTVQ GEMV per-call numbers

--impl reference times the reference algorithm's CPU restatement (oracle port)
on the host cores on the same metric.
"""

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused VQ GEMV/attn µs/call & HBM GB/s vs roofline; decode tokens/s Llama-7B"
LLAMA7B = [("qkv", 4096, 12288), ("o", 4096, 4096), ("gate_up", 4096, 22016), ("down", 11008, 4096)]
N_LAYERS = 32
WORK = 256


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def algorithmic_bytes(m, n, rows=1, code_bits=16, v=8, work=WORK):
    codes = (m * n // v) * code_bits // 8
    books = work * v * 2
    return codes + books + rows * m * 2 + rows * n * 2


class Clocks:
    """SM clock and throttle-reason sampling during the timed region (the
    B200_PROFILING.md clocks line): NVML polled every millisecond from a thread —
    the timed regions last tens of milliseconds, too short for nvidia-smi -lms."""

    NAMES = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, gpu_index=0):
        import threading
        self.samples, self.max_mhz, self.reasons = [], None, set()
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self.nv = None
            return
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.NAMES.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.001)

    def stop(self):
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        self._stop.set()
        self.t.join(timeout=2)
        sm = self.samples or [0.0]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples), "source": "nvml 1 ms"}


def ncu_traffic():
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture
    (profiles/ncu_summary.json, written from `ncu --set full`), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        return json.load(f).get("gemv_group")


def roofline(achieved_gbs, peak, src, kern, kernel_us, per_linear):
    """At N=1 the step is ONE gemv_group launch and nothing else, so the kernel's
    achieved bandwidth is algorithmic step bytes / its CUDA-event time; traffic is
    that launch's DRAM bytes from the committed ncu --set full capture."""
    t = ncu_traffic()
    return {"bound": "hbm", "achieved": achieved_gbs, "peak": peak, "unit": "GB/s", "frac": achieved_gbs / peak,
            "traffic": t["dram_bytes"] if t else None,
            "traffic_alg_bytes": t["alg_bytes"] if t else None,
            "traffic_launch": t["launch"] if t else None,
            "kernel": kern, "peak_source": src, "kernel_us_mean": kernel_us}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------------------------------
# CPU legs (oracle port: the reference's algorithm restated, V/codec.py:391-408 + V/sim.py:133-144)

_CPU_CASE = {}


def cpu_sample(seconds_budget=12.0, threads=None):
    """The reference algorithm (dequantize, V/codec.py:391-408, then the fp32 matmul of
    reference_compute, V/sim.py:136-144) restated in C with OpenMP on the host cores
    (all of them, or `threads`), on one 4096x4096 q_proj of the workload config,
    repeated for ~seconds_budget. Returns (GB/s over the same algorithmic bytes,
    sample description, threads)."""
    from oracle import c_oracle as C
    from oracle import vq_oracle as O

    m, n, v = 4096, 4096, 8
    if not _CPU_CASE:
        codes, books = O.synthetic_codes_books((m, n), v, 16, 1, 1, 0, working_entries=WORK)
        _CPU_CASE.update(codes=codes, books=books, regions=np.zeros(m * n // v, dtype=np.int32),
                         x=O.synthetic_tensor((m,), 2), all=C.threads())
    c = _CPU_CASE
    C.set_threads(threads or c["all"])
    reps, t0 = 0, time.perf_counter()
    try:
        while True:
            C.gemv(c["codes"], c["books"], (m, n), v, 1, c["regions"], c["x"])
            reps += 1
            if time.perf_counter() - t0 > seconds_budget or reps >= 2000:
                break
        used = C.threads()
    finally:
        C.set_threads(c["all"])
    dt = (time.perf_counter() - t0) / reps
    gbs = algorithmic_bytes(m, n) / dt / 1e9
    return gbs, (f"C/OpenMP oracle (dequantize + fp32 matmul) of one 4096x4096 quip2 q_proj, {used} thread(s), "
                 f"{reps} reps, {dt*1e3:.2f} ms each"), used


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    step_bytes = sum(algorithmic_bytes(m, n) for _, m, n in LLAMA7B) * N_LAYERS
    for _ in range(args.warmup):
        cpu_sample(seconds_budget=0.5)
    vals = []
    for _ in range(args.steps):
        gbs, sample, cores = cpu_sample(seconds_budget=3.0)
        vals.append(gbs)
    value = float(np.median(vals))
    ms = step_bytes / (value * 1e9) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "llama7b-decode-linears quip2 VQ<8,16,1> ws256 batch1 (sampled on q_proj)"},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cores, "kind": "port", "sample": sample,
                         "host_cpus": os.cpu_count()},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------------

# Megatron-style tensor parallelism of the decode linears: qkv and
# gate_up column-parallel (N / tp, outputs stay local for attention / SiLU), o and
# down row-parallel (M / tp, partial outputs all-reduced)
TP_KIND = {"qkv": "col", "o": "row", "gate_up": "col", "down": "row"}


def shard_shape(name, m, n, world):
    return (m, n // world) if TP_KIND[name] == "col" else (m // world, n)


def build_stack(torch, dev, rank=0, world=1, grouped=True):
    """The step's 32 x 4 linears (this rank's TP shards) as a VQLinearStack;
    grouped=True runs them as one persistent grouped GEMV launch."""
    from paper_2503_02236_b200.codec import VQConfig
    from paper_2503_02236_b200.device import DeviceVQTensor
    from paper_2503_02236_b200.stack import VQLinearStack

    cfg = VQConfig(8, 16, 1)
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    weights, bytes_per, names = [], [], []
    for _layer in range(N_LAYERS):
        for name, m, n in LLAMA7B:
            ms, ns = shard_shape(name, m, n, world)
            codes = torch.randint(0, WORK, (1, ms * ns // 8), generator=g, device=dev, dtype=torch.int32)
            books = (torch.randn((1, 1 << 16, 8), generator=g, device=dev) * 0.1).half()
            w = DeviceVQTensor.from_device_codes(codes, (ms, ns), cfg, books, layout="plain").relayout("gemv")
            weights.append(w)
            names.append(name)
            bytes_per.append(algorithmic_bytes(ms, ns))
    stack = VQLinearStack(weights, rows=1, grouped=grouped)
    stack.x.copy_((torch.randn(stack.x.shape, generator=g, device=dev)).half())
    stack.names = names
    return stack, bytes_per


def graph_time(torch, fn, reps):
    """us per replay of fn captured in a CUDA graph (events on the replaying stream)."""
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            fn()
    torch.cuda.current_stream().wait_stream(st)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def time_attention(torch, dev, ops, N):
    """C4: CQ-4 KV cache decode attention, B16 H32 T4096 C128 (per-call us, GB/s)."""
    from paper_2503_02236_b200.codec import Sharing, VQConfig
    from paper_2503_02236_b200.device import DeviceVQTensor

    B, H, T, C = 16, 32, 4096, 128
    cfg = VQConfig(2, 8, 1, Sharing.per_channel_group(2))
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    s = B * H * T * C // 2
    kv = []
    for _ in range(2):
        codes = torch.randint(0, 256, (1, s), generator=g, device=dev, dtype=torch.int32)
        books = (torch.randn((H * 64, 256, 2), generator=g, device=dev) * 0.1).half()
        kv.append(DeviceVQTensor.from_device_codes(codes, (B, H, T, C), cfg, books).relayout("kv"))
    q = torch.randn((B, H, C), generator=g, device=dev).half()
    for _ in range(3):
        ops.vq_attention(kv[0], kv[1], q, out_dtype=torch.float16)
    kern = N.last_kernel()
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        ops.vq_attention(kv[0], kv[1], q, out_dtype=torch.float16)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    alg = 2 * s + 2 * H * 64 * 256 * 2 * 2 + B * H * C * 2 * 2
    # dense fp16 baseline at equal shape (flash-attn decode), if importable
    dense_us = None
    try:
        from flash_attn import flash_attn_with_kvcache
        kd = torch.randn((B, T, H, C), device=dev, dtype=torch.float16)
        vd = torch.randn((B, T, H, C), device=dev, dtype=torch.float16)
        qd = q.view(B, 1, H, C)
        for _ in range(3):
            flash_attn_with_kvcache(qd, kd, vd)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            flash_attn_with_kvcache(qd, kd, vd)
        e1.record()
        torch.cuda.synchronize()
        dense_us = e0.elapsed_time(e1) * 1e3 / reps
        del kd, vd
    except Exception as ex:  # pragma: no cover - optional baseline
        dense_us = f"unavailable: {type(ex).__name__}"
    return {"config": "C4 cq4 VQ<2,8,1> cg2 B16 H32 T4096 C128", "kernel": kern, "us_per_call": us,
            "alg_bytes": alg, "GB_s": alg / us / 1e3, "fp16_flash_attn_us": dense_us}


def time_gemv_single(torch, dev, ops, N, label, cfg_args, shape, work=None):
    from paper_2503_02236_b200.codec import Sharing, VQConfig
    from paper_2503_02236_b200.device import DeviceVQTensor

    v, bits, r, sharing = cfg_args
    cfg = VQConfig(v, bits, r, sharing)
    m, n = shape
    g = torch.Generator(device=dev)
    g.manual_seed(11)
    from paper_2503_02236_b200.codec import region_count
    nreg = region_count(shape, cfg)
    hi = work or (1 << bits)
    # 32 distinct copies so the cycle exceeds L2
    ws = []
    for _ in range(32):
        codes = torch.randint(0, hi, (r, m * n // v), generator=g, device=dev, dtype=torch.int32)
        books = (torch.randn((r * nreg, 1 << bits, v), generator=g, device=dev) * 0.1).half()
        ws.append(DeviceVQTensor.from_device_codes(codes, shape, cfg, books).relayout("gemv"))
    from paper_2503_02236_b200.stack import VQLinearStack
    sub = VQLinearStack(ws, rows=1)
    sub.x.copy_(torch.randn(sub.x.shape, generator=g, device=dev).half())
    sub.capture()
    for _ in range(3):
        sub.replay()
    kern = N.last_kernel()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        sub.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (10 * len(ws))
    x = sub.x[:m]
    alg = ws[0].algorithmic_bytes(work) + m * 2 + n * 2
    # dense fp16 cuBLAS GEMV at the same shape, also graph-replayed over > L2 of weights
    dense = [torch.randn((m, n), device=dev, dtype=torch.float16) for _ in range(max(2, (512 << 20) // (m * n * 2) + 1))]
    xd = x.reshape(1, m).contiguous()
    outs = [torch.empty((1, n), device=dev, dtype=torch.float16) for _ in dense]

    def run_dense():
        for d, o in zip(dense, outs):
            torch.matmul(xd, d, out=o)

    dense_us = graph_time(torch, run_dense, 10) / len(dense)
    del dense
    return {"config": label, "kernel": kern, "us_per_call": us, "alg_bytes": alg, "GB_s": alg / us / 1e3,
            "fp16_cublas_us": dense_us, "note": "CUDA graphs over > L2 of distinct weights (both arms)"}


def time_decode(torch, dev, batch=1, ctx=4096, reps=10, tp=False, fused=False):
    """C5: end-to-end Llama-7B-shaped decode step (VQ weights + CQ-4 KV cache), one
    CUDA graph per step at a context of `ctx` cached tokens. tp=True: this rank's
    Megatron shard (heads / ffn slice, NCCL all-reduce after o and down, captured
    in the graph; fused=True: those all-reduces fused into the GEMV over peer memory,
    tp.PeerComm)."""
    from paper_2503_02236_b200.decode import LlamaShape, VQLlamaDecoder
    dec = VQLlamaDecoder.synthetic(LlamaShape(), batch, ctx, dev, seed=3)
    if tp:
        dec = VQLlamaDecoder.tensor_parallel(dec, None, fused_collectives=fused)
        torch.cuda.empty_cache()
    world = dec.world
    dec.set_length(ctx - 1 - reps - 3)
    # (the gloo dry run of the multi-GPU path cannot capture its collectives: eager steps)
    eager = tp and os.environ.get("VQB_BENCH_SHARED_GPU") == "1"
    step = dec.run_step if eager else dec.replay
    if not eager:
        dec.capture()
    for _ in range(3):
        step()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    if dec.comm is not None:
        dec.comm.close()
    del dec
    torch.cuda.empty_cache()
    if tp:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t[0])
    return {"config": f"C5 llama7b decode quip2 weights + cq4 KV, batch {batch}, ctx {ctx}"
                      + (f", tp{world}" + (" fused peer-memory all-reduce" if fused else " NCCL all-reduce")
                         if tp else ""), "batch": batch,
            "ms_per_step": ms, "tokens_per_s": batch * 1e3 / ms, "data": "synthetic weights/KV (random init)"}


def tensor_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    return 2250.0, 2250.0, "fallback (nominal dense bf16)"


def _weights(torch, dev, cfg, shape, copies, work, seed):
    from paper_2503_02236_b200.codec import region_count
    from paper_2503_02236_b200.device import DeviceVQTensor
    m, n = shape
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    nreg = region_count(shape, cfg)
    out = []
    for _ in range(copies):
        codes = torch.randint(0, work or cfg.n_entries, (cfg.residuals, m * n // cfg.vector_size), generator=g,
                              device=dev, dtype=torch.int32)
        books = (torch.randn((cfg.residuals * nreg, cfg.n_entries, cfg.vector_size), generator=g, device=dev)
                 * 0.1).half()
        out.append(DeviceVQTensor.from_device_codes(codes, shape, cfg, books).relayout("gemv"))
    return out


def time_gemm(torch, dev, N, label, cfg, shapes, rows=1024, work=None, copies=4):
    """Prefill GEMM y = X @ dequant(W) (rows x M x N, tcgen05) per shape and in total,
    CUDA-graph replays over `copies` distinct weights, against dense fp16 cuBLAS at
    the same shape; tensor-pipe roofline = flops / time vs MEASURED_PEAKS bf16 (burst,
    the kernel is timed alone)."""
    from paper_2503_02236_b200.ops import launch_struct, workspace
    peak, _, src = tensor_peak()
    lib = N.lib()
    res, tot_flops, tot_us, tot_dense = {}, 0.0, 0.0, 0.0
    for name, m, n in shapes:
        ws = _weights(torch, dev, cfg, (m, n), copies, work, 21)
        x = torch.randn((rows, m), device=dev).half()
        ys = [torch.empty((rows, n), device=dev, dtype=torch.float16) for _ in ws]
        L = launch_struct()
        structs = [w.struct() for w in ws]
        need = max(N.check(lib.vqb_workspace_bytes(N.KERNEL_GEMM, st, rows, L)) for st in structs)
        buf = workspace(need, dev)

        def run():
            st_ = torch.cuda.current_stream(dev).cuda_stream
            for st, y in zip(structs, ys):
                N.check(lib.vqb_gemm(st, x.data_ptr(), N.F16, rows, y.data_ptr(), N.F16, L, buf.data_ptr(),
                                     buf.numel(), st_))

        us = graph_time(torch, run, 10) / len(ws)
        kern = N.last_kernel()
        # both prefill paths at this shape: fused producers vs dequantise + dense pair GEMM
        paths = {}
        for pname, flag in (("fused", N.FLAG_GEMM_FUSED), ("two_phase", N.FLAG_GEMM_TWO_PHASE)):
            L2 = launch_struct()
            L2.flags |= flag
            need2 = max(N.check(lib.vqb_workspace_bytes(N.KERNEL_GEMM, st, rows, L2)) for st in structs)
            buf2 = workspace(need2, dev)

            def run_p():
                st_ = torch.cuda.current_stream(dev).cuda_stream
                for st, y in zip(structs, ys):
                    N.check(lib.vqb_gemm(st, x.data_ptr(), N.F16, rows, y.data_ptr(), N.F16, L2, buf2.data_ptr(),
                                         buf2.numel(), st_))

            pus = graph_time(torch, run_p, 10) / len(ws)
            paths[pname] = {"kernel": N.last_kernel(), "us_per_call": round(pus, 2),
                            "TFLOP_s": round(2.0 * rows * m * n / pus / 1e6, 1)}
        dense = [torch.randn((m, n), device=dev, dtype=torch.float16) for _ in range(copies)]
        outs = [torch.empty((rows, n), device=dev, dtype=torch.float16) for _ in dense]

        def run_dense():
            for d, o in zip(dense, outs):
                torch.matmul(x, d, out=o)

        dus = graph_time(torch, run_dense, 10) / len(dense)
        flops = 2.0 * rows * m * n
        res[name] = {"shape": [rows, m, n], "kernel": kern, "us_per_call": round(us, 2),
                     "TFLOP_s": round(flops / us / 1e6, 1), "frac": round(flops / us / 1e6 / peak, 3),
                     "fp16_cublas_us": round(dus, 2), "fp16_cublas_TFLOP_s": round(flops / dus / 1e6, 1),
                     "speedup_vs_fp16": round(dus / us, 3), "paths": paths}
        tot_flops += flops
        tot_us += us
        tot_dense += dus
        del ws, dense, outs, ys
        torch.cuda.empty_cache()
    return {"config": label, "rows": rows, "per_linear": res,
            "roofline": {"bound": "tensor", "achieved": round(tot_flops / tot_us / 1e6, 1), "peak": peak,
                         "unit": "TFLOP/s", "frac": round(tot_flops / tot_us / 1e6 / peak, 3),
                         "peak_source": f"{src} bf16 burst (kernel timed alone)"},
            "fp16_cublas_TFLOP_s": round(tot_flops / tot_dense / 1e6, 1),
            "speedup_vs_fp16": round(tot_dense / tot_us, 3)}


def time_gemv_shapes(torch, dev, N, cfg, shapes, work=None, rows=1):
    """Per-call fused GEMV (batch `rows`) per shape: graph replays over > L2 of distinct
    weights, HBM roofline on the algorithmic bytes, dense fp16 cuBLAS at equal shape."""
    from paper_2503_02236_b200.stack import VQLinearStack
    hbm, _ = peaks()
    out = {}
    for name, m, n in shapes:
        code_bytes = cfg.residuals * (m * n // cfg.vector_size) * cfg.log2_entries // 8
        copies = max(2, min(48, (256 << 20) // code_bytes + 1))
        ws = _weights(torch, dev, cfg, (m, n), copies, work, 31)
        sub = VQLinearStack(ws, rows=rows)
        sub.x.copy_(torch.randn(sub.x.shape, device=dev).half())
        us = graph_time(torch, sub.launch_all, 10) / len(ws)
        kern = N.last_kernel()
        alg = ws[0].algorithmic_bytes(work) + rows * (m + n) * 2
        dense = [torch.randn((m, n), device=dev, dtype=torch.float16)
                 for _ in range(max(2, (512 << 20) // (m * n * 2) + 1))]
        xd = torch.randn((rows, m), device=dev).half()
        outs = [torch.empty((rows, n), device=dev, dtype=torch.float16) for _ in dense]

        def run_dense():
            for d, o in zip(dense, outs):
                torch.matmul(xd, d, out=o)

        dus = graph_time(torch, run_dense, 10) / len(dense)
        out[name] = {"shape": [m, n], "rows": rows, "kernel": kern, "us_per_call": round(us, 2),
                     "alg_bytes": alg, "GB_s": round(alg / us / 1e3, 1), "frac": round(alg / us / 1e3 / hbm, 3),
                     "fp16_cublas_us": round(dus, 2), "speedup_vs_fp16": round(dus / us, 2)}
        del ws, sub, dense, outs
        torch.cuda.empty_cache()
    return out


def time_zipf(torch, dev, N, m=4096, n=12288, copies=12):
    """Adaptive codebook placement on skewed codes (SURVEY §8d variant: Zipf(1.2)
    + reorder_all, V/cli.py:204-223): quip VQ<8,16,1> qkv-shaped GEMVs, batch 1,
    graph replays over > L2 of distinct weights.

    full_book:   Zipf over all 2^16 entries with the hot entries scattered (the
                 trained order), shared tier = the planned span; vs the same
                 weights after the device profile + reorder (hot entries first,
                 so the shared span catches most lookups; the rest use L2)
    working_set: Zipf over a 256-entry working set, reordered: register tier off
                 vs the planner's mu + 3 sigma register slots."""
    from paper_2503_02236_b200.codec import VQConfig
    from paper_2503_02236_b200.dataflow import ComputeOp
    from paper_2503_02236_b200.device import DeviceVQTensor
    from paper_2503_02236_b200.gpumodel import load_gpu_model
    from paper_2503_02236_b200.machine import launch_of, plan_kernel
    from paper_2503_02236_b200.ops import workspace
    from paper_2503_02236_b200.profiling import device_histograms, reorder_device

    cfg = VQConfig(8, 16, 1)
    b200 = load_gpu_model("b200")
    op = ComputeOp.gemv(m, n)
    hbm, _ = peaks()
    g = torch.Generator(device=dev)
    g.manual_seed(77)
    lib = N.lib()

    def zipf_codes(hi, count):
        p = 1.0 / torch.arange(1, hi + 1, device=dev, dtype=torch.float64) ** 1.2
        return torch.multinomial((p / p.sum()).float(), count, replacement=True, generator=g).to(torch.int32)

    def make(hi, scramble):
        ws = []
        for _ in range(copies):
            codes = zipf_codes(hi, m * n // 8)
            if scramble:
                codes = torch.randperm(1 << 16, device=dev, generator=g).to(torch.int32)[codes]
            books = (torch.randn((1, 1 << 16, 8), generator=g, device=dev) * 0.1).half()
            ws.append(DeviceVQTensor.from_device_codes(codes.view(1, -1), (m, n), cfg, books).relayout("gemv"))
        return ws

    def timed(ws, L):
        x = torch.randn((m,), device=dev).half()
        ys = [torch.empty((n,), device=dev, dtype=torch.float16) for _ in ws]
        structs = [w.struct() for w in ws]
        need = max(N.check(lib.vqb_workspace_bytes(N.KERNEL_GEMV, st, 1, L)) for st in structs)
        buf = workspace(need, dev)

        def run():
            st_ = torch.cuda.current_stream(dev).cuda_stream
            for st, y in zip(structs, ys):
                N.check(lib.vqb_gemv(st, x.data_ptr(), N.F16, 1, y.data_ptr(), N.F16, L, buf.data_ptr(),
                                     buf.numel(), st_))

        us = graph_time(torch, run, 10) / len(ws)
        info = N.last_launch()
        alg = ws[0].algorithmic_bytes(256) + (m + n) * 2
        return {"us_per_call": round(us, 2), "GB_s": round(alg / us / 1e3, 1), "frac": round(alg / us / 1e3 / hbm, 3),
                "n_shared": info["n_shared"], "n_reg": info["n_reg"]}

    out = {"config": f"quip VQ<8,16,1> {m}x{n} b1, Zipf(1.2) codes"}
    ws = make(1 << 16, scramble=True)
    plans = plan_kernel(cfg, op, b200)
    res = {"trained_order": timed(ws, launch_of(plans, op))}
    ro = [reorder_device(w) for w in ws]
    ws2 = [r[0] for r in ro]
    hist = device_histograms(ro[0][1])[0]
    ns = plans.cache_plan.n_shared
    res["reordered"] = timed(ws2, launch_of(plans, op))
    # lookups served by the shared span [0, ns) before (old index < ns) and after reordering
    sorted_counts, fwd = ro[0][1][0, 0], ro[0][2][0, 0]
    res["shared_hit_fraction_trained"] = round(float(sorted_counts[fwd[:ns]].sum()) / hist.total, 4)
    res["shared_hit_fraction_reordered"] = round(float(hist.counts[:ns].sum()) / hist.total, 4)
    out["full_book"] = res
    del ws, ws2, ro
    ws = [reorder_device(w)[0] for w in make(256, scramble=True)]
    _, counts, _ = reorder_device(ws[0])
    hist = device_histograms(counts)[0]
    hot = plan_kernel(cfg, op, b200, histogram=hist).dataflow_plan.meta["hot_register_slots"]
    planned = plan_kernel(cfg, op, b200, histogram=hist, n_reg=hot)  # the paper's mu + 3 sigma slots
    off = plan_kernel(cfg, op, b200, histogram=hist, n_reg=0)
    out["working_set"] = {"hot_register_slots": hot,
                          "register_tier_off": timed(ws, launch_of(off, op)),
                          "register_tier_planned": timed(ws, launch_of(planned, op))}
    del ws
    torch.cuda.empty_cache()
    return out


LLAMA65B = [("q", 8192, 8192), ("up", 8192, 22016), ("down", 22016, 8192)]


def time_c3(torch, dev, N):
    """C3: AQLM 2x8 (VQConfig(8, 8, 2)) at Llama-65B shapes — GEMV batch 1 at the
    per-GPU shard of tensor parallelism 1/2/4/8 (column-parallel q/up: N/tp,
    row-parallel down: M/tp), and the prefill GEMM (rows 1024) at TP1."""
    from paper_2503_02236_b200.codec import VQConfig
    cfg = VQConfig(8, 8, 2)
    gemv = {}
    for tp in (1, 2, 4, 8):
        shapes = [("q", 8192, 8192 // tp), ("up", 8192, 22016 // tp), ("down", 22016 // tp, 8192)]
        gemv[f"tp{tp}"] = time_gemv_shapes(torch, dev, N, cfg, shapes)
    gemm = time_gemm(torch, dev, N, "C3 aqlm2x8 VQ<8,8,2> llama65b prefill rows 1024", cfg, LLAMA65B, copies=2)
    return {"config": "C3 aqlm2x8 VQ<8,8,2> whole, llama65b q/up/down", "gemv_b1_per_gpu_shard": gemv,
            "gemm_rows1024_tp1": gemm}


def run_impl(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    # VQB_BENCH_SHARED_GPU=1 (dry run of the multi-GPU code path on a one-GPU box): every
    # rank on cuda:0, collectives over gloo (NCCL refuses two ranks on one device)
    shared = os.environ.get("VQB_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    if world > 1:
        dist.init_process_group("gloo" if shared else "nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import __graft_entry__
    __graft_entry__.build()
    from paper_2503_02236_b200 import _native as N
    from paper_2503_02236_b200 import ops

    stack, bytes_per = build_stack(torch, dev, rank, world, grouped=True)
    step_bytes = sum(bytes_per)
    from paper_2503_02236_b200.stack import VQLinearStack
    single = VQLinearStack(stack.weights, rows=1)  # one gemv_fast launch per linear
    single.x.copy_(stack.x)

    # per-linear kernel times: CUDA-graph replays of one linear's GEMV over 32 layers'
    # distinct weights (> L2), CUDA events on the replaying stream
    per_linear = {}
    if not args.no_extra and world == 1:
        for li, (name, m, n) in enumerate(LLAMA7B):
            ws_ = [stack.weights[layer * len(LLAMA7B) + li] for layer in range(N_LAYERS)]
            sub = VQLinearStack(ws_, rows=1)
            sub.capture()
            for _ in range(3):
                sub.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(10):
                sub.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / (10 * N_LAYERS)
            alg = algorithmic_bytes(m, n)
            per_linear[name] = {"shape": [m, n], "us_per_call": round(us, 2), "alg_bytes": alg,
                                "GB_s": round(alg / us / 1e3, 1)}
            del sub

    # tensor parallelism: the row-parallel linears' partial outputs are all-reduced,
    # one NCCL collective per row-parallel linear (64 per step), as a TP decode step does
    row_views = [stack.output_view(i) for i, nm in enumerate(stack.names) if TP_KIND[nm] == "row"]

    def collectives():
        if world > 1:
            for v in row_views:
                dist.all_reduce(v)

    def step():
        stack.replay()
        collectives()

    stack.launch_all()
    kern = N.last_kernel()  # the headline kernel (gemv_group)
    stack.capture()
    single.capture()
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    # the same step as a chain of 128 single-linear launches (the per-call kernel a
    # decode loop with dependencies between linears uses)
    for _ in range(3):
        single.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        single.replay()
        collectives()
    e1.record()
    torch.cuda.synchronize()
    ms_single = e0.elapsed_time(e1) / args.steps
    diff = float((single.y.float() - stack.y.float()).abs().max()) if world == 1 else None
    # the headline step with fp32 accumulation of every product (VQB_FLAG_EXACT_ACCUM)
    # instead of the 8-row fp16x2 windows, for comparison with the window numerics
    exact = None
    if world == 1 and not args.no_extra:
        from paper_2503_02236_b200.ops import launch_struct
        Lx = launch_struct()
        Lx.flags |= 8
        ex = VQLinearStack(stack.weights, rows=1, launches=[Lx] * len(stack.weights), grouped=True)
        ex.x.copy_(stack.x)
        ex.capture()
        for _ in range(3):
            ex.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            ex.replay()
        e1.record()
        torch.cuda.synchronize()
        ms_ex = e0.elapsed_time(e1) / args.steps
        exact = {"what": "the headline step (one grouped launch) with VQB_FLAG_EXACT_ACCUM: fp32 accumulation "
                         "of every product instead of 8-row fp16x2 windows",
                 "ms_per_step": ms_ex, "GB_s": step_bytes / (ms_ex * 1e-3) / 1e9,
                 "max_abs_diff_vs_windows": float((ex.y.float() - stack.y.float()).abs().max()),
                 "max_abs_output": float(stack.y.float().abs().max())}
        del ex
    # e2e through the public API with pinned host buffers: every step copies its inputs
    # host->device and its result device->host; StackPipeline overlaps those copies with
    # the neighbouring steps' compute (two buffer sets, separate H2D / D2H streams)
    hxs = [torch.empty(stack.x.shape, dtype=stack.x.dtype, pin_memory=True) for _ in range(2)]
    for hx in hxs:
        hx.copy_(stack.x)
    hys = [torch.empty(stack.y.shape, dtype=stack.y.dtype, pin_memory=True) for _ in range(2)]
    if world == 1:
        from paper_2503_02236_b200.stack import StackPipeline
        pipe = StackPipeline(stack)

        def e2e_steps(k):
            pipe.run([hxs[j % 2] for j in range(k)], [hys[j % 2] for j in range(k)])
    else:
        def e2e_steps(k):  # TP: the collectives sit between the copies
            for j in range(k):
                stack.run(hxs[j % 2], hys[j % 2])
                collectives()
    e2e_steps(max(args.warmup, 2))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    e2e_steps(args.steps)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = max(e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3) / args.steps
    e2e_ok = world > 1 or bool(torch.equal(torch.from_numpy(hys[(args.steps - 1) % 2].numpy()).to(dev), stack.y))
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([ms, e2e_ms, ms_single], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_ms, ms_single = float(t[0]), float(t[1]), float(t[2])

    decode_tp = None
    if world > 1 and not args.no_extra:
        decode_tp = [time_decode(torch, dev, b, tp=True) for b in (1, 16, 64)]  # C5 at N GPUs
        for b in (1, 8):  # the GEMV batches with the all-reduce fused into the epilogue (csrc/tp.cu)
            try:
                decode_tp.append(time_decode(torch, dev, b, tp=True, fused=True))
            except Exception as e:  # reported, never fatal to the scaling run
                decode_tp.append({"batch": b, "fused": True, "error": f"{type(e).__name__}: {e}"[:300]})
    if rank == 0:
        hbm, src = peaks()
        total_bytes = step_bytes * world
        value = total_bytes / (ms * 1e-3) / 1e9
        extra = {}
        if per_linear:
            extra["per_linear"] = per_linear
        if decode_tp:
            extra["decode_c5"] = decode_tp
        extra["step_per_launch"] = {
            "what": "the same step as 128 single-linear vq_gemv launches (the per-call kernels of a decode loop)",
            "ms_per_step": ms_single, "GB_s": total_bytes / (ms_single * 1e-3) / 1e9,
            "frac": total_bytes / (ms_single * 1e-3) / 1e9 / world / hbm, "launches_per_step": single.n_launches,
            "max_abs_diff_vs_grouped": diff}
        if exact:
            extra["exact_accum_step"] = exact
        want = (lambda k: True) if not args.only else (lambda k: k in args.only.split(","))
        if not args.no_extra and world == 1:
            from paper_2503_02236_b200.codec import Sharing, VQConfig
            if want("attention_c4"):
                extra["attention_c4"] = time_attention(torch, dev, ops, N)
            if want("gemv_c1"):
                extra["gemv_c1_gptvq2_q_proj"] = time_gemv_single(
                    torch, dev, ops, N, "C1 gptvq2 VQ<4,8,1> tile256 4096x4096 b1",
                    (4, 8, 1, Sharing.per_tile(256, 256)), (4096, 4096))
            if want("decode_c5"):
                extra["decode_c5"] = [time_decode(torch, dev, b) for b in (1, 2, 4, 8, 16, 32, 64)]  # BASELINE C5 sweep
            if want("gemm_c2"):
                extra["gemm_c2_prefill"] = time_gemm(
                    torch, dev, N, "C2 quip2 VQ<8,16,1> ws256 llama7b prefill rows 1024", VQConfig(8, 16, 1),
                    LLAMA7B, work=WORK)
            if want("zipf"):
                extra["zipf_adaptive_cache"] = time_zipf(torch, dev, N)
            if want("c3"):
                extra["c3_aqlm65b"] = time_c3(torch, dev, N)
            if want("gemv_c2"):
                extra["gemv_c2_quip2_q_proj"] = time_gemv_single(
                    torch, dev, ops, N, "C2 quip2 VQ<8,16,1> ws256 4096x4096 b1", (8, 16, 1, Sharing.whole_tensor()),
                    (4096, 4096), work=WORK)
        cpu = None
        if world == 1 and not args.no_cpu:
            gbs, sample, cores = cpu_sample()
            gbs1, sample1, _ = cpu_sample(seconds_budget=6.0, threads=1)
            cpu = {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "port", "sample": sample,
                   "value_1thread": gbs1, "sample_1thread": sample1, "host_cpus": os.cpu_count()}
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f16", "data": "synthetic",
            "config": {"workload": "llama7b-decode-linears quip2 VQ<8,16,1> ws256 batch1",
                       "layers": N_LAYERS, "launches_per_step": stack.n_launches,
                       "grouping": "the step's 128 independent GEMVs as one persistent stream-K launch "
                                   "(vqb_gemv_grouped); the 128-launch chain is step_per_launch",
                       "parallelism": (f"tp{world}: qkv/gate_up column-parallel, o/down row-parallel + one "
                                       f"NCCL all-reduce per row-parallel linear") if world > 1 else "single",
                       "l2": "inputs 1.6 GB/GPU > L2, no flush", "graph": True},
            "us_per_call": ms * 1e3 / stack.n_launches,
            "e2e": {"value": total_bytes / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": int(stack.x.numel() * stack.x.element_size()),
                    "d2h_bytes_per_step": int(stack.y.numel() * stack.y.element_size()),
                    "ms_per_step": e2e_ms,
                    "how": ("stack.StackPipeline: per step H2D of the inputs and D2H of the result on their own "
                            "streams, overlapping the neighbouring steps' compute" if world == 1 else
                            "VQLinearStack.run + the TP collectives, serial"),
                    "result_matches_device": e2e_ok},
            "roofline": roofline(value / world, hbm, src, kern, ms * 1e3 / stack.n_launches, per_linear),
            "kernel": kern,
            "cpu_baseline": cpu,
            "gpu_launches": stack.n_launches * args.steps,
            "clocks": clk,
        }
        line.update(extra)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--only", default="", help="comma list of extra keys to time (default: all)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_impl(args)


if __name__ == "__main__":
    main()
