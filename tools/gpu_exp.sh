timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "decode or rmsnorm" > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 900 python tools/decode_bench.py 1 16 2>&1 | tail -2
