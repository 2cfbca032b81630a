mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
for lib in ab/base.so paper_2503_02236_b200/libvqb.so; do echo $lib; VQB_LIB_PATH=$PWD/$lib python tools/decode_bench.py 16 64; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base function -k regex:"gemm" -s 6 -c 6 python tools/decode_bench.py 16 --layers 2 --reps 3 2>&1 | grep -E "gemm|duration"
