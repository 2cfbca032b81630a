"""End-to-end Llama-7B decode (C5): VQ weights (QuiP#-2bit, VQ<8,16,1> ws256) + CQ-4 KV
cache, one CUDA graph per step, context `ctx` tokens already cached.

Usage: python tools/decode_bench.py [batch ...] [--ctx 4096] [--layers 32]
Prints one JSON line per batch: ms/step, tokens/s."""

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2503_02236_b200.decode import LlamaShape, VQLlamaDecoder  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("batch", type=int, nargs="*", default=[1])
    ap.add_argument("--ctx", type=int, default=4096)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--gemv-max-rows", type=int, default=None)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    for b in args.batch:
        sh = LlamaShape(layers=args.layers)
        dec = VQLlamaDecoder.synthetic(sh, b, args.ctx, dev)
        if args.gemv_max_rows is not None:
            dec.gemv_max_rows = args.gemv_max_rows
        dec.set_length(args.ctx - 1 - args.reps - 3)
        dec.capture()
        for _ in range(3):
            dec.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            dec.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        print(json.dumps({"model": "llama7b-shape", "layers": args.layers, "batch": b, "ctx": args.ctx,
                          "ms_per_step": round(ms, 3), "tokens_per_s": round(b * 1e3 / ms, 1),
                          "final_len": int(dec.d_len.item())}), flush=True)
        del dec
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
