timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "gemv or decode or tp or fullsize" 2>&1 | tail -3
python tools/gemv_sweep.py --rows 16 --shapes 4096x4096,4096x12288,4096x22016,11008x4096
python tools/gemm_bench.py 16 2>/dev/null | head -4
python tools/decode_bench.py 8 16
