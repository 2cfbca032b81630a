for r in 32 64; do python tools/gemv_sweep.py --rows $r --shapes 4096x4096,4096x12288,4096x22016,11008x4096 | grep -v smem; python tools/gemm_bench.py $r 2>/dev/null | head -4; done
