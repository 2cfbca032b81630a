for rep in 1 2; do for lib in ab/base.so paper_2503_02236_b200/libvqb.so; do echo "== $lib"
for r in 1 8; do VQB_LIB_PATH=$PWD/$lib python tools/gemv_sweep.py --cfg quip2 --shapes 4096x12288,4096x4096,4096x22016,11008x4096 --rows $r 2>&1 | grep us_per | grep -o '"shape": \[[0-9, ]*\], "rows": [0-9]*\|"us_per_call": [0-9.]*' | paste - -; done; done; done
