"""Per-CTA phase timeline of back-to-back batch-1 decode GEMVs (debug trace flag 32).

A chain o -> qkv -> o of quip2 GEMVs, each with its own workspace so every launch
keeps its trace; prints, per launch, the quantiles (us, relative to the first launch's
earliest CTA start) of: CTA start, prologue done (after griddepcontrol.wait), first
chunk landed, streaming done, end — and the hand-off gap to the previous launch.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_02236_b200 import ops  # noqa: E402
from paper_2503_02236_b200.codec import Sharing, VQConfig  # noqa: E402
from paper_2503_02236_b200.device import DeviceVQTensor  # noqa: E402

WS_HEAD = 16 * 1024 * 1024


def weight(dev, m, n, seed):
    cfg = VQConfig(8, 16, 1, Sharing.whole_tensor())
    g = torch.Generator(device=dev).manual_seed(seed)
    codes = torch.randint(0, 256, (1, m * n // 8), generator=g, device=dev, dtype=torch.int32)
    books = (torch.randn((1, 65536, 8), generator=g, device=dev) * 0.1).half()
    return DeviceVQTensor.from_device_codes(codes, (m, n), cfg, books).relayout("gemv")


def main():
    dev = torch.device("cuda", 0)
    shapes = [(4096, 4096), (4096, 12288), (4096, 4096), (4096, 22016), (11008, 4096)]
    ws = [weight(dev, m, n, i) for i, (m, n) in enumerate(shapes)]
    xs = [torch.randn((1, m), device=dev).half() for m, _ in shapes]
    arenas = [ops.Workspace(dev, WS_HEAD + (1 << 20)) for _ in shapes]
    L = ops.launch_struct()
    L.flags = 32
    for _ in range(3):
        for w, x, a in zip(ws, xs, arenas):
            with ops.use_workspace(a):
                ops.vq_gemv(w, x, launch=L)
    torch.cuda.synchronize()
    trs = []
    for a in arenas:
        t = a.buf[WS_HEAD:WS_HEAD + 148 * 64].view(torch.int64).view(148, 8).cpu()
        trs.append(t[t[:, 0] > 0])
    t0 = int(trs[0][:, 0].min())
    out = []
    prev_end = None
    for (m, n), t in zip(shapes, trs):
        rel = (t[:, :7].double() - t0) / 1e3
        q = lambda c: [round(float(rel[:, c].quantile(p)), 2) for p in (0.0, 0.5, 1.0)]
        end = float(rel[:, 6].max())
        out.append({"shape": f"{m}x{n}", "ctas": int(t.shape[0]), "start": q(0), "prologue": q(1),
                    "first_chunk": q(2), "stream_done": q(3), "end": q(6),
                    "handoff_us": None if prev_end is None else round(float(rel[:, 0].min()) - prev_end, 2),
                    "span_us": round(end - float(rel[:, 0].min()), 2)})
        prev_end = end
    for o in out:
        print(json.dumps(o))
    if os.environ.get("VQB_TRACE_DETAIL"):
        t = trs[int(os.environ["VQB_TRACE_DETAIL"])]
        rel = (t[:, :7].double() - int(t[:, 0].min())) / 1e3
        for i in range(t.shape[0]):
            print(i, [round(float(v), 2) for v in rel[i]], int(t[i, 7]))


if __name__ == "__main__":
    main()
