timeout 900 python bench.py --only none > gpurun_out/r02_b5_bench.json 2> gpurun_out/r02_b5_bench.err
echo bench rc=$?
PROF_LAYERS=32 ncu --set full --clock-control none --import-source on -k regex:gemv_group -s 1 -c 1 -o /tmp/prof_group32 python tools/prof_kernels.py group > gpurun_out/r02_prof_group32.log 2>&1
ncu -i /tmp/prof_group32.ncu-rep --page raw --csv > gpurun_out/r02_prof_group32_raw.csv 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu > /dev/null 2>&1
echo ncu rc=$?
