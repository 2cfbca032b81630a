mkdir -p gpurun_out
python tools/decode_bench.py 1 16 > gpurun_out/dec.txt 2>&1
VQB_DECODE_SKIP=attn python tools/decode_bench.py 1 >> gpurun_out/dec.txt 2>&1
VQB_DECODE_SKIP=norm,silu,front python tools/decode_bench.py 1 >> gpurun_out/dec.txt 2>&1
cat gpurun_out/dec.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 1200 -c 400 --csv --log-file gpurun_out/dec_launches.csv python tools/decode_bench.py 1 --reps 2 > gpurun_out/ncu_dec.log 2>&1; tail -2 gpurun_out/ncu_dec.log
