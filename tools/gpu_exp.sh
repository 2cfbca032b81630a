timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k gemv > gpurun_out/pytest_gpu.txt 2>&1; tail -1 gpurun_out/pytest_gpu.txt
for f in 32; do timeout 120 python tools/gemv_sweep.py --cfg quip2 --shapes 4096x12288 --flags $f 2>&1 | tail -3; done
timeout 300 python tools/gemv_sweep.py --cfg quip2 --shapes 4096x4096,4096x12288,4096x22016,11008x4096 2>&1 | tail -4
for r in 2 4 8; do timeout 300 python tools/gemv_sweep.py --cfg quip2 --shapes 4096x12288 --rows $r 2>&1 | tail -1; done
