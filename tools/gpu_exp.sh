timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "attn or attention or smoke" > gpurun_out/pytest_gpu.txt 2>&1; tail -1 gpurun_out/pytest_gpu.txt
python tools/attn_bench.py
python tools/attn_bench.py 16 32 4096 128 4
python tools/attn_bench.py 1 32 4096 128 2
