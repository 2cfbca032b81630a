import sys, os, torch, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2503_02236_b200 import _native as N, ops
from paper_2503_02236_b200.codec import VQConfig
from paper_2503_02236_b200.device import DeviceVQTensor
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
for cfg, (m, n) in ((VQConfig(8, 16, 1), (4096, 12288)), (VQConfig(8, 8, 2), (2048, 1024)), (VQConfig(8, 8, 1), (1024, 512))):
    codes = torch.randint(0, 256, (cfg.residuals, m * n // 8), generator=g, device=dev, dtype=torch.int32)
    books = (torch.randn((cfg.residuals, cfg.n_entries, 8), generator=g, device=dev) * 0.05).half()
    w = DeviceVQTensor.from_device_codes(codes, (m, n), cfg, books).relayout("gemv")
    dense = ops.vq_dequantize(w)
    for rows in (4, 8, 13, 16, 32, 64):
        x = torch.randn((rows, m), generator=g, device=dev).half()
        y = ops.vq_gemv(w, x, out_dtype=torch.float32)
        k = N.last_kernel()
        ref = x.float() @ dense.half().float() if cfg.residuals == 1 else x.float() @ dense
        err = ((y - ref).abs().max() / ref.abs().max()).item()
        y2 = ops.vq_gemv(w, x, out_dtype=torch.float32)
        print(cfg.residuals, cfg.log2_entries, m, n, rows, k, f"{err:.2e}", bool(torch.equal(y, y2)), flush=True)
