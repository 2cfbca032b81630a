"""Batch-1 fused decode step with parts replaced by no-ops (graph-timed), to split the
1.65 ms step: python tools/decode_ablate_fused.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_02236_b200 import ops  # noqa: E402
from paper_2503_02236_b200.decode import LlamaShape, VQLlamaDecoder  # noqa: E402


def timed(dec, reps=20):
    dec.set_length(4000)
    dec.capture()
    for _ in range(3):
        dec.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        dec.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    dev = torch.device("cuda", 0)
    sh = LlamaShape()
    dec = VQLlamaDecoder.synthetic(sh, 1, 4096, dev)
    out = {"full": timed(dec)}
    zero = torch.zeros((1, sh.heads, sh.head_dim), dtype=torch.float16, device=dev)
    real_attend = dec._attend
    dec._attend = lambda L, qkv: zero
    out["no_attention"] = timed(dec)
    dec._attend = real_attend
    theta = sh.rope_theta
    q_fixed = torch.zeros((1, sh.heads, sh.head_dim), dtype=torch.float16, device=dev)

    def separate(L, qkv):
        q = ops.qkv_rope_append(qkv, L.k_cache, L.v_cache, dec.d_len, theta)
        return ops.vq_attention(L.k_cache, L.v_cache, q, out_dtype=torch.float16, d_len=dec.d_len)

    def attn_only(L, qkv):
        return ops.vq_attention(L.k_cache, L.v_cache, q_fixed, out_dtype=torch.float16, d_len=dec.d_len)

    def append_only(L, qkv):
        ops.qkv_rope_append(qkv, L.k_cache, L.v_cache, dec.d_len, theta)
        return zero

    for name, fn in (("separate", separate), ("attention_only", attn_only), ("append_only", append_only)):
        dec._attend = fn
        out[name] = timed(dec)
    dec._attend = real_attend
    print(json.dumps({k: round(v, 3) for k, v in out.items()}))


if __name__ == "__main__":
    main()
