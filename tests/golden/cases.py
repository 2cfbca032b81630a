"""Golden-vector case table shared by make_golden.py (generator, needs the
reference) and the tests (consumers, run anywhere).

Each dequant case is (name, shape, vector_size, log2_entries, residuals, sharing,
tile, group_width, seed, working_entries). Shapes are small enough for the numpy
oracle to run in well under a second each.
"""

DEQUANT_CASES = [
    # BASELINE C1: GPTVQ-2, 256x256 tile-shared books (V/presets.py:55-61)
    ("gptvq2", (512, 512), 4, 8, 1, "tile", (256, 256), 0, 3, None),
    # tile sharing with partial edge tiles (V/codec.py:170-177)
    ("gptvq2_edge", (300, 520), 4, 8, 1, "tile", (256, 256), 0, 4, None),
    # BASELINE C2: QuiP#-style E8, VQ<8,16,1>, 256-entry working set
    ("quip2", (256, 512), 8, 16, 1, "whole", (0, 0), 0, 5, 256),
    # preset quip4: VQ<8,16,2> (V/presets.py:38-47)
    ("quip4", (64, 256), 8, 16, 2, "whole", (0, 0), 0, 6, 256),
    # BASELINE C3: AQLM 2x8, VQ<8,8,2>
    ("aqlm2x8", (256, 512), 8, 8, 2, "whole", (0, 0), 0, 7, None),
    # preset aqlm3: VQ<8,12,2>, misaligned 12-bit stream (V/presets.py:48-54)
    ("aqlm3", (128, 256), 8, 12, 2, "whole", (0, 0), 0, 8, None),
    # BASELINE C4: CQ-4 KV cache, 2-channel groups per head (V/presets.py:62-68)
    ("cq4", (2, 4, 64, 128), 2, 8, 1, "channel_group", (0, 0), 2, 9, None),
    # preset cq2 (V/presets.py:69-75)
    ("cq2", (2, 4, 64, 128), 4, 8, 1, "channel_group", (0, 0), 4, 10, None),
    # 2-D channel-group sharing and an odd entry count
    ("cg2d", (16, 64), 4, 4, 1, "channel_group", (0, 0), 8, 11, None),
    # v = 16, 3-bit codes, three residual levels on a 3-D tensor
    ("v16r3", (3, 8, 64), 16, 3, 3, "whole", (0, 0), 0, 12, None),
    # a residual (R=2) KV cache with per-head channel groups
    ("kv_r2", (1, 2, 32, 64), 4, 6, 2, "channel_group", (0, 0), 4, 13, None),
]

# fused-op cases: (name, dequant-case name, op, extra)
#   gemv: activation (M,) from synthetic_tensor(seed+2)
#   gemm: activation (rows, M)
#   attention: K from the case seed, V from seed+1, query from seed+2
MATMUL_CASES = [
    ("gemv_gptvq2", "gptvq2", "gemv", {}),
    ("gemv_quip2", "quip2", "gemv", {}),
    ("gemv_aqlm2x8", "aqlm2x8", "gemv", {}),
    ("gemv_aqlm3", "aqlm3", "gemv", {}),
    ("gemm_gptvq2", "gptvq2", "gemm", {"rows": 16}),
    ("gemm_quip2", "quip2", "gemm", {"rows": 8}),
]

ATTENTION_CASES = [
    ("attn_cq4", "cq4"),
    ("attn_cq2", "cq2"),
]

PRESETS_FOR_PLANS = ("quip4", "aqlm3", "gptvq2", "cq4", "cq2")

# online KV quantization (V/codec.py:367-389): (name, dequant-case name supplying the
# config and fp16-rounded books, data seed). Data = synthetic_tensor(shape, seed).
QUANTIZE_CASES = [
    ("qz_cq4", "cq4", 21),
    ("qz_cq2", "cq2", 22),
    ("qz_r2", "kv_r2", 23),
]
