"""Launch-list probe of the two-phase prefill GEMM (run under ncu --metrics
gpu__time_duration.sum): AQLM 2x8 8192x8192 and QuiP# 4096x4096 at rows 1024."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_02236_b200 import _native as N  # noqa: E402
from paper_2503_02236_b200 import ops  # noqa: E402
from paper_2503_02236_b200.codec import VQConfig  # noqa: E402
from paper_2503_02236_b200.device import DeviceVQTensor  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
for cfg, (m, n), work in ((VQConfig(8, 8, 2), (8192, 8192), 256), (VQConfig(8, 16, 1), (4096, 4096), 256)):
    codes = torch.randint(0, work, (cfg.residuals, m * n // 8), generator=g, device=dev, dtype=torch.int32)
    books = (torch.randn((cfg.residuals, cfg.n_entries, 8), generator=g, device=dev) * 0.05).half()
    w = DeviceVQTensor.from_device_codes(codes, (m, n), cfg, books).relayout("gemv")
    x = torch.randn((1024, m), generator=g, device=dev).half()
    for flag in (N.FLAG_GEMM_TWO_PHASE, N.FLAG_GEMM_FUSED):
        L = ops.launch_struct()
        L.flags |= flag
        for _ in range(2):
            ops.vq_gemm(w, x, out_dtype=torch.float16, launch=L)
    d = torch.randn((m, n), generator=g, device=dev).half()
    torch.matmul(x, d)
torch.cuda.synchronize()
