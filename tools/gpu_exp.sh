timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -20 gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-extra --no-cpu 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['clocks'])"
