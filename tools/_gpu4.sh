for k in group:gemv_group:1 gemm:gemm_tc:1 single:gemv_fast:40; do
  IFS=: read what pat skip <<< "$k"
  ncu --set full --clock-control none --import-source on -k regex:$pat -s $skip -c 1 -o /tmp/prof_$what python tools/prof_kernels.py $what > gpurun_out/r02_prof_$what.log 2>&1
  ncu -i /tmp/prof_$what.ncu-rep --page raw --csv > gpurun_out/r02_prof_${what}_raw.csv 2>&1
  ncu -i /tmp/prof_$what.ncu-rep --page details --csv > gpurun_out/r02_prof_${what}_details.csv 2>&1
  ncu -i /tmp/prof_$what.ncu-rep --page source --csv > gpurun_out/r02_prof_${what}_source.csv 2>&1
done
cp /tmp/prof_group.ncu-rep gpurun_out/r02_prof_group.ncu-rep
ls -la gpurun_out/
