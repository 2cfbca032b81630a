"""Per-CTA phase timeline of the CQ attention kernel (debug trace flag 32)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_02236_b200 import _native as N  # noqa: E402
from paper_2503_02236_b200.codec import Sharing, VQConfig  # noqa: E402
from paper_2503_02236_b200.device import DeviceVQTensor  # noqa: E402
from paper_2503_02236_b200 import ops  # noqa: E402


def main(B=1, H=32, T=4096, C=128, v=2):
    dev = torch.device("cuda", 0)
    cfg = VQConfig(v, 8, 1, Sharing.per_channel_group(v))
    g = torch.Generator(device=dev).manual_seed(7)
    s = B * H * T * C // v
    kv = []
    for _ in range(2):
        codes = torch.randint(0, 256, (1, s), generator=g, device=dev, dtype=torch.int32)
        books = (torch.randn((H * C // v, 256, v), generator=g, device=dev) * 0.1).half()
        kv.append(DeviceVQTensor.from_device_codes(codes, (B, H, T, C), cfg, books).relayout("kv"))
    q = torch.randn((B, H, C), generator=g, device=dev).half()
    L = ops.launch_struct()
    L.flags = 32
    for _ in range(3):
        ops.vq_attention(kv[0], kv[1], q, out_dtype=torch.float16, launch=L)
    torch.cuda.synchronize()
    ws = ops.workspace(1, dev)
    tr = ws[8192:8192 + 148 * 64].view(torch.int64).view(148, 8).cpu()
    t0 = int(tr[:, 0].min())
    rel = (tr[:, :6] - t0).double() / 1e3
    q_ = lambda c: [round(float(rel[:, c].quantile(p)), 2) for p in (0.0, 0.5, 1.0)]
    sm = lambda c: [round(float((tr[:, c].double() / 1e3).quantile(p)), 2) for p in (0.0, 0.5, 1.0)]
    print(json.dumps({"B": B, "T": T, "start": q_(0), "pdl_ok": q_(1), "end": q_(5),
                      "sum_prologue": sm(2), "sum_stream": sm(3), "sum_merge": sm(4), "spans": [int(tr[:, 6].min()), int(tr[:, 6].max())]}))


if __name__ == "__main__":
    main(*[int(x) for x in sys.argv[1:]])
