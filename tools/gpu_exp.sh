mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "decode or quant" 2>&1 | tail -2
for lib in ab/lb2.so paper_2503_02236_b200/libvqb.so; do echo $lib
VQB_LIB_PATH=$PWD/$lib timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --kernel-name-base function -k regex:qkv_rope_append -s 3 -c 1 python tools/decode_bench.py 16 --layers 2 --reps 3 2>&1 | grep -E "duration|inst_exec"
VQB_LIB_PATH=$PWD/$lib python tools/decode_bench.py 1 16
done
