# Round-2 measurement: gpu tests, smoke, bench (both arms), launch list, ncu of the main kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_info.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -2 gpurun_out/bench1.err; head -c 600 gpurun_out/bench1.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; head -c 300 gpurun_out/bench_ref.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemv|attn|gemm|dequant|tp_" -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > gpurun_out/ncu_launch.log 2>&1; tail -1 gpurun_out/ncu_launch.log
cap() {  # name, kernel regex, skip, command...: full capture -> raw CSV (the .ncu-rep stays on the box)
  n=$1; k=$2; sk=$3; shift 3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $sk -c 1 -o /tmp/prof_$n "$@" > gpurun_out/ncu_$n.log 2>&1
  ncu -i /tmp/prof_$n.ncu-rep --page raw --csv > gpurun_out/raw_$n.csv 2>/dev/null
  ncu -i /tmp/prof_$n.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$n.csv 2>/dev/null
  tail -1 gpurun_out/ncu_$n.log; ls -la gpurun_out/raw_$n.csv
}
cap gemv_group gemv_group 0 python bench.py --steps 1 --warmup 3 --no-cpu --no-extra
cap attn attn_cq 2 python tools/attn_bench.py
cap gemv_tc gemv_tc 6 python tools/gemv_sweep.py --rows 16 --shapes 4096x12288 --copies 4
cap gemv_cs gemv_cs 2 python tools/gemv_sweep.py --rows 1 --shapes 4096x4096 --copies 4
cap gemm_dense gemm_dense 1 python tools/twophase_probe.py
cap gemm_pair gemm_pair 1 python tools/twophase_probe.py
timeout 300 python tools/decode_bench.py 1 2 4 8 16 32 64 > gpurun_out/decode_sweep.txt 2>&1; cat gpurun_out/decode_sweep.txt
du -sh gpurun_out
