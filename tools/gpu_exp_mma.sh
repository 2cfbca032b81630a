for r in 4 8; do python tools/gemv_sweep.py --rows $r --shapes 4096x4096,4096x12288,4096x22016,11008x4096; done
python tools/gemv_sweep.py --rows 8 --cfg aqlm2x8 --shapes 8192x8192
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "gemv or decode" 2>&1 | tail -2
python tools/decode_bench.py 1 4 8
