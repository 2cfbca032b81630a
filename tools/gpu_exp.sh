timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
for rep in 1 2; do for lib in ab/base.so paper_2503_02236_b200/libvqb.so; do echo "== $lib"
for r in 1 2; do VQB_LIB_PATH=$PWD/$lib python tools/gemv_sweep.py --cfg quip2 --shapes 4096x12288,4096x4096 --rows $r 2>&1 | grep us_per | grep -o '"shape": \[[0-9, ]*\], "rows": [0-9]*\|"us_per_call": [0-9.]*' | paste - -; done
VQB_LIB_PATH=$PWD/$lib python tools/gemv_sweep.py --cfg gptvq2 --shapes 4096x4096 --rows 2 2>&1 | grep us_per | grep -o '"us_per_call": [0-9.]*'
done; done
python tools/decode_bench.py 1 2
