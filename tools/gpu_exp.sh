python tools/decode_bench.py 2 4 8
python tools/decode_bench.py 2 4 8 --gemv-max-rows 1
