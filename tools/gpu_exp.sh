timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "gemm or decode" > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 900 python tools/decode_bench.py 16 64 2>&1 | tail -2
