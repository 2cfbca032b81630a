timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "gemv or full" > gpurun_out/pytest_gpu.txt 2>&1; tail -1 gpurun_out/pytest_gpu.txt
timeout 300 python tools/gemv_sweep.py --cfg quip2 --shapes 4096x4096,4096x12288,4096x22016,11008x4096 2>&1 | tail -4
timeout 300 python tools/gemv_sweep.py --cfg aqlm2x8 --shapes 8192x8192 2>&1 | tail -1
timeout 300 python tools/gemv_sweep.py --cfg gptvq2 --shapes 4096x4096 2>&1 | tail -1
