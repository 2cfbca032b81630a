timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
python tools/attn_trace.py 1; python tools/attn_trace.py 16
python tools/attn_bench.py
python tools/attn_bench.py 1 32 4096 128 2
timeout 900 python tools/decode_bench.py 1 16 2>&1 | tail -2
