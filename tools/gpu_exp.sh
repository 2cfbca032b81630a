mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --kernel-name-base function -k regex:qkv_rope_append -s 3 -c 1 python tools/decode_bench.py 16 --layers 2 --reps 3 2>&1 | grep -E "duration|inst_exec"
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --kernel-name-base function -k regex:qkv_rope_append -s 3 -c 1 python tools/decode_bench.py 1 --layers 2 --reps 3 2>&1 | grep -E "duration|inst_exec"
python tools/decode_bench.py 1 8 16 64
