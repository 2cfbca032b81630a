mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "${PYTEST_K:-attention or decode or fullsize or robust}" > gpurun_out/pytest_gpu.txt 2>&1; tail -5 gpurun_out/pytest_gpu.txt
python tools/attn_bench.py
python tools/decode_bench.py 1 16
VQB_DECODE_SKIP=attn python tools/decode_bench.py 1
