python tools/attn_trace.py 1 32 4096
python tools/attn_trace.py 16 32 4096
python tools/attn_bench.py 1 32 4096
python tools/attn_bench.py 4 32 4096
