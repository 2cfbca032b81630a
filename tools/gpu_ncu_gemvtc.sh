mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_tc -s 6 -c 1 -o gpurun_out/prof_gemvtc python tools/gemv_sweep.py --rows 16 --shapes 4096x12288 --copies 4 > gpurun_out/ncu_gemvtc.log 2>&1; tail -1 gpurun_out/ncu_gemvtc.log
