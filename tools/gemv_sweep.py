"""Per-call GEMV timing sweep (CUDA-graph replays of distinct weights, > L2).

Usage: python tools/gemv_sweep.py [--rows 1] [--cfg quip2|aqlm2x8|gptvq2]
Prints one JSON line per shape: us/call, algorithmic GB/s, fraction of the measured
HBM peak, and the dense fp16 cuBLAS time for the same shape (also graph-replayed).
"""

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2503_02236_b200 import _native as N  # noqa: E402
from paper_2503_02236_b200.codec import Sharing, VQConfig, region_count  # noqa: E402
from paper_2503_02236_b200.device import DeviceVQTensor  # noqa: E402
from paper_2503_02236_b200.ops import launch_struct, vq_gemv  # noqa: E402

CFGS = {
    "quip2": (VQConfig(8, 16, 1), 256),
    "aqlm2x8": (VQConfig(8, 8, 2), None),
    "gptvq2": (VQConfig(4, 8, 1, Sharing.per_tile(256, 256)), None),
}


def graph_time(fn, reps):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us per replay


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1)
    ap.add_argument("--cfg", default="quip2")
    ap.add_argument("--shapes", default="4096x4096,4096x12288,4096x22016,11008x4096,8192x8192,16384x16384")
    ap.add_argument("--copies", type=int, default=0, help="distinct weights cycled (0: enough for > 256 MB)")
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--n_shared", type=int, default=0)
    ap.add_argument("--split", type=int, default=0, help="M split (cluster size) override")
    ap.add_argument("--grid", type=int, default=0, help="grid limit (persistent CTAs)")
    args = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    dev = torch.device("cuda", 0)
    probe = torch.zeros(4, dtype=torch.int32, device=dev)
    N.check(N.lib().vqb_debug_smem_base(probe.data_ptr(), torch.cuda.current_stream().cuda_stream))
    print(json.dumps({"dynamic_smem_base": int(probe[0])}), flush=True)
    cfg, work = CFGS[args.cfg]
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    for shp in args.shapes.split(","):
        m, n = (int(x) for x in shp.split("x"))
        nreg = region_count((m, n), cfg)
        s = m * n // cfg.vector_size
        code_bytes = cfg.residuals * s * cfg.log2_entries // 8
        copies = args.copies or max(2, min(64, (256 << 20) // code_bytes + 1))
        ws = []
        for _ in range(copies):
            codes = torch.randint(0, work or cfg.n_entries, (cfg.residuals, s), generator=g, device=dev,
                                  dtype=torch.int32)
            books = (torch.randn((cfg.residuals * nreg, cfg.n_entries, cfg.vector_size), generator=g,
                                 device=dev) * 0.1).half()
            ws.append(DeviceVQTensor.from_device_codes(codes, (m, n), cfg, books).relayout("gemv"))
        x = torch.randn((args.rows, m), generator=g, device=dev).half()
        ys = [torch.empty((args.rows, n), device=dev, dtype=torch.float16) for _ in ws]
        L = launch_struct(n_shared=args.n_shared or None, grid_limit=args.grid)
        L.flags = args.flags
        if args.split:
            L.split_axis, L.split_factor = ord("M"), args.split
        lib = N.lib()
        structs = [w.struct() for w in ws]
        from paper_2503_02236_b200.ops import workspace
        need = max(N.check(lib.vqb_workspace_bytes(N.KERNEL_GEMV, st, args.rows, L)) for st in structs)

        bufs = []

        def run():
            buf = workspace(need, dev)
            bufs.append(buf)
            stream = torch.cuda.current_stream(dev).cuda_stream
            for st, y in zip(structs, ys):
                N.check(lib.vqb_gemv(st, x.data_ptr(), N.F16, args.rows, y.data_ptr(), N.F16, L,
                                     buf.data_ptr(), buf.numel(), stream))

        us = graph_time(run, 20) / len(ws)
        if args.flags & 32:
            torch.cuda.synchronize()
            buf = bufs[-1]
            off = 4194304
            buf[off:off + 64 * 148].zero_() if False else None
            tr = buf[off:off + 64 * 148].view(torch.int64).view(-1, 8).cpu()
            valid = tr[:, 0] > 0
            tr = tr[valid]
            t0 = int(tr[:, 0].min())
            rel = (tr[:, :7] - t0).double() / 1e3
            sms = tr[:, 7]
            import collections
            occ = collections.Counter(collections.Counter(sms.tolist()).values())
            q = lambda c: [round(float(rel[:, c].quantile(p)), 2) for p in (0.0, 0.5, 1.0)]
            print(json.dumps({"shape": [m, n], "ctas": int(valid.sum()), "ctas_per_sm_hist": dict(occ),
                              "start": q(0), "book_ready": q(1), "first_data": q(2), "compute_done": q(3),
                              "end": q(6)}), flush=True)
            pub = tr[:, 4] > 0
            fin = tr[:, 5] > 0
            print(json.dumps({"publishers": int(pub.sum()), "publish_minus_done": [round(float(x), 2) for x in ((tr[pub, 4] - tr[pub, 3]).double() / 1e3).quantile(torch.tensor([0.0, 0.5, 1.0], dtype=torch.float64))] if pub.any() else None,
                              "finishers": int(fin.sum()), "flags_seen_minus_done": [round(float(x), 2) for x in ((tr[fin, 5] - tr[fin, 3]).double() / 1e3).quantile(torch.tensor([0.0, 0.5, 1.0], dtype=torch.float64))] if fin.any() else None,
                              "end_minus_flags": [round(float(x), 2) for x in ((tr[fin, 6] - tr[fin, 5]).double() / 1e3).quantile(torch.tensor([0.0, 0.5, 1.0], dtype=torch.float64))] if fin.any() else None}), flush=True)
        kern = N.last_kernel()
        alg = ws[0].algorithmic_bytes(work) + args.rows * (m + n) * 2
        dense = [torch.randn((m, n), device=dev, dtype=torch.float16) for _ in range(max(2, min(16, (512 << 20) // (m * n * 2) + 1)))]
        outs = [torch.empty((args.rows, n), device=dev, dtype=torch.float16) for _ in dense]

        def run_dense():
            for d, o in zip(dense, outs):
                torch.matmul(x, d, out=o)

        dus = graph_time(run_dense, 20) / len(dense)
        print(json.dumps({"cfg": args.cfg, "shape": [m, n], "rows": args.rows, "kernel": kern, "split": args.split, "flags": args.flags, "copies": len(ws),
                          "us_per_call": round(us, 2), "alg_MB": round(alg / 1e6, 2),
                          "GB_s": round(alg / us / 1e3, 1), "frac_hbm": round(alg / us / 1e3 / peak, 3),
                          "fp16_cublas_us": round(dus, 2),
                          "fp16_GB_s": round(m * n * 2 / dus / 1e3, 1), "speedup_vs_fp16": round(dus / us, 2)}),
              flush=True)
        del ws, dense
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
