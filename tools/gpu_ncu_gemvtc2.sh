mkdir -p gpurun_out
timeout 300 python tools/gemv_tc_check.py > gpurun_out/tc_check.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_tc -s 6 -c 1 -o /tmp/p python tools/gemv_sweep.py --rows 16 --shapes 4096x12288 --copies 4 > /dev/null 2>&1
ncu -i /tmp/p.ncu-rep --page source --csv --print-source sass > gpurun_out/src_gemv_tc2.csv 2>/dev/null
ncu -i /tmp/p.ncu-rep --page raw --csv > gpurun_out/raw_gemv_tc2.csv 2>/dev/null
