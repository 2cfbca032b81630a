timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -30 gpurun_out/pytest_gpu.txt
python tools/attn_bench.py
