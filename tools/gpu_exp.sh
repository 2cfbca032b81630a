timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "gemm" > gpurun_out/pytest_gpu.txt 2>&1; tail -1 gpurun_out/pytest_gpu.txt
timeout 300 python tools/gemm_bench.py 1024 quip2
timeout 300 python tools/gemm_bench.py 1024 aqlm2x8
