set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "attn or attention or decode" 2>&1 | tail -2
python tools/attn_trace.py 16 32 4096 128 2
python tools/attn_trace.py 1 32 4096 128 2
python tools/attn_bench.py 2>&1 | tail -1
