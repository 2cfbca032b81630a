mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 4 -c 1 -o gpurun_out/prof_gemm16 python tools/gemm_bench.py 16 > gpurun_out/ncu_gemm16.log 2>&1; tail -1 gpurun_out/ncu_gemm16.log
