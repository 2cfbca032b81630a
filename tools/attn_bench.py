"""C4 decode-attention microbenchmark (one config, CUDA events, > L2 working set)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_02236_b200 import _native as N  # noqa: E402
from paper_2503_02236_b200.codec import Sharing, VQConfig  # noqa: E402
from paper_2503_02236_b200.device import DeviceVQTensor  # noqa: E402
from paper_2503_02236_b200.ops import vq_attention  # noqa: E402


def main(B=16, H=32, T=4096, C=128, v=2, reps=20):
    dev = torch.device("cuda", 0)
    cfg = VQConfig(v, 8, 1, Sharing.per_channel_group(v))
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    s = B * H * T * C // v
    kv = []
    for _ in range(2):
        codes = torch.randint(0, 256, (1, s), generator=g, device=dev, dtype=torch.int32)
        books = (torch.randn((H * C // v, 256, v), generator=g, device=dev) * 0.1).half()
        kv.append(DeviceVQTensor.from_device_codes(codes, (B, H, T, C), cfg, books).relayout("kv"))
    q = torch.randn((B, H, C), generator=g, device=dev).half()
    for _ in range(3):
        vq_attention(kv[0], kv[1], q, out_dtype=torch.float16)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        vq_attention(kv[0], kv[1], q, out_dtype=torch.float16)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    alg = 2 * s + 2 * H * (C // v) * 256 * v * 2 + B * H * C * 4
    print(json.dumps({"kernel": N.last_kernel(), "us": round(us, 2), "GB_s": round(alg / us / 1e3, 1)}))


if __name__ == "__main__":
    main(*[int(x) for x in sys.argv[1:]])
