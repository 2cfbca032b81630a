"""Fused-activation GEMV (vqb_gemv_xf) vs the separate RMSNorm/SiLU kernel + GEMV:
a CUDA-graph chain of 32 dependent linears (qkv-shaped and down-shaped) on distinct
weights (> L2), us per linear."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_02236_b200 import ops  # noqa: E402
from paper_2503_02236_b200.decode import WEIGHT_CFG  # noqa: E402
from paper_2503_02236_b200.device import DeviceVQTensor  # noqa: E402


def graph_us(fn, reps=10):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def main():
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(1)
    books = (torch.randn((1, 65536, 8), generator=g, device=dev) * 0.02).half()

    def weight(m, n):
        codes = torch.randint(0, 256, (1, m * n // 8), generator=g, device=dev, dtype=torch.int32)
        return DeviceVQTensor.from_device_codes(codes, (m, n), WEIGHT_CFG, books).relayout("gemv")

    L = 32
    out = {}
    for name, m, n, kind in (("qkv+norm", 4096, 4096, "norm"), ("down+silu", 11008, 4096, "silu"),
                             ("o", 4096, 4096, "plain")):
        ws = [weight(m, n) for _ in range(L)]
        nw = torch.ones(m, dtype=torch.float16, device=dev)
        res = [torch.randn((1, m), generator=g, device=dev).half() for _ in range(2)]
        x0 = torch.randn((1, 2 * m if kind == "silu" else m), generator=g, device=dev).half()

        def unfused():
            for w in ws:
                if kind == "norm":
                    ops.vq_gemv(w, ops.rmsnorm(x0, res[0], nw), out_dtype=torch.float16)
                elif kind == "silu":
                    ops.vq_gemv(w, ops.silu_mul(x0), out_dtype=torch.float16)
                else:
                    ops.vq_gemv(w, x0, out_dtype=torch.float16)

        def fused():
            cur = 0
            for w in ws:
                if kind == "norm":
                    ops.vq_gemv_rmsnorm(w, x0, res[cur], nw, 1e-5, residual_out=res[1 - cur])
                    cur ^= 1
                elif kind == "silu":
                    ops.vq_gemv_silu(w, x0)
                else:
                    ops.vq_gemv(w, x0, out_dtype=torch.float16)

        out[name] = {"unfused_us": round(graph_us(unfused) / L, 2), "fused_us": round(graph_us(fused) / L, 2)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
