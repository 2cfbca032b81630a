mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_fast -s 6 -c 1 -o gpurun_out/prof_gemv_b8 python tools/gemv_sweep.py --rows 8 --shapes 4096x12288 --copies 4 > gpurun_out/ncu_gemv_b8.log 2>&1; tail -2 gpurun_out/ncu_gemv_b8.log
