"""Small driver for ncu captures of the hot kernels (one process, one GPU):

    ncu --set full --clock-control none --import-source on -k regex:gemv_group -s 1 -c 1 \
        -o gpurun_out/prof_group python tools/prof_kernels.py group

what: group  - the bench step's GEMVs (8 layers of Llama-7B quip2 linears) as one grouped launch
      single - the same linears, one gemv_fast launch each
      gemm   - prefill GEMM rows 1024 at the qkv shape (gemm_tc)
      attn   - C4 attention B16 H32 T4096 (attn_cq)
Each is run twice (warm-up + the captured launch).
"""

import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2503_02236_b200 import _native as N  # noqa: E402
from paper_2503_02236_b200 import ops  # noqa: E402


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "group"
    layers = int(os.environ.get("PROF_LAYERS", "8"))
    dev = torch.device("cuda", 0)
    if what in ("group", "single"):
        bench.N_LAYERS = layers
        stack, _ = bench.build_stack(torch, dev)
        if what == "group":
            from paper_2503_02236_b200.stack import VQLinearStack
            stack = VQLinearStack(stack.weights, rows=1, grouped=True)
        for _ in range(2):
            stack.launch_all()
    elif what == "gemm":
        from paper_2503_02236_b200.codec import VQConfig
        w = bench._weights(torch, dev, VQConfig(8, 16, 1), (4096, 12288), 1, bench.WORK, 3)[0]
        x = torch.randn((1024, 4096), device=dev).half()
        for _ in range(2):
            ops.vq_gemm(w, x, out_dtype=torch.float16)
    elif what == "attn":
        bench.time_attention(torch, dev, ops, N)
    torch.cuda.synchronize()
    print(what, N.last_kernel())


if __name__ == "__main__":
    main()
