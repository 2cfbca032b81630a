# quick iteration: gpu tests (subset via $1), bench, optional ncu of a kernel regex ($2)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x ${1:+-k "$1"} > gpurun_out/pytest_gpu.txt 2>&1; tail -15 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
if [ -n "$2" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s ${3:-200} -c 1 -o gpurun_out/prof_$2 python bench.py --steps 1 --warmup 1 --no-cpu ${4} > gpurun_out/ncu_$2.log 2>&1; tail -2 gpurun_out/ncu_$2.log
fi
