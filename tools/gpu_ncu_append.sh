mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:qkv_rope_append -s 6 -c 1 -o /tmp/pa python tools/decode_bench.py 64 --reps 2 --layers 4 > /dev/null 2>&1
ncu -i /tmp/pa.ncu-rep --page raw --csv > gpurun_out/raw_append.csv 2>/dev/null
ncu -i /tmp/pa.ncu-rep --page source --csv --print-source sass > gpurun_out/src_append.csv 2>/dev/null
ls -la gpurun_out/raw_append.csv
