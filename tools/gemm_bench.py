"""Prefill GEMM benchmark: tcgen05 VQ GEMM vs dense fp16 cuBLAS at equal shapes.

Usage: python tools/gemm_bench.py [rows] [cfg]   (cfg: quip2 | aqlm2x8)
Prints one JSON line per Llama-7B linear shape: us/call, TFLOP/s, fraction of the
measured bf16/fp16 peak (MEASURED_PEAKS.json: burst), and the cuBLAS time.
"""

import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2503_02236_b200 import _native as N  # noqa: E402
from paper_2503_02236_b200.codec import VQConfig  # noqa: E402
from paper_2503_02236_b200.device import DeviceVQTensor  # noqa: E402
from paper_2503_02236_b200.ops import vq_gemm  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    cfgname = sys.argv[2] if len(sys.argv) > 2 else "quip2"
    cfg, work = {"quip2": (VQConfig(8, 16, 1), 256), "aqlm2x8": (VQConfig(8, 8, 2), None)}[cfgname]
    peaks = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak = json.load(open(peaks))["bf16_tflops"] if os.path.exists(peaks) else 1590.0
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    shapes = [(4096, 4096), (4096, 12288), (4096, 22016), (11008, 4096)] if cfgname == "quip2" else \
        [(8192, 8192), (8192, 22016), (22016, 8192)]
    for m, n in shapes:
        s = m * n // 8
        codes = torch.randint(0, work or cfg.n_entries, (cfg.residuals, s), generator=g, device=dev,
                              dtype=torch.int32)
        books = (torch.randn((cfg.residuals, cfg.n_entries, 8), generator=g, device=dev) * 0.1).half()
        w = DeviceVQTensor.from_device_codes(codes, (m, n), cfg, books).relayout("gemv")
        x = torch.randn((rows, m), generator=g, device=dev).half()
        y = torch.empty((rows, n), device=dev, dtype=torch.float16)
        us = timed(lambda: vq_gemm(w, x, out_dtype=torch.float16))
        kern = N.last_kernel()
        dense = torch.randn((m, n), device=dev, dtype=torch.float16)
        dus = timed(lambda: torch.matmul(x, dense, out=y))
        flop = 2.0 * rows * m * n
        print(json.dumps({"cfg": cfgname, "rows": rows, "shape": [m, n], "kernel": kern, "us": round(us, 2),
                          "TFLOPs": round(flop / us / 1e6, 1), "frac_peak": round(flop / us / 1e6 / peak, 3),
                          "fp16_cublas_us": round(dus, 2), "cublas_TFLOPs": round(flop / dus / 1e6, 1)}),
              flush=True)


if __name__ == "__main__":
    main()
