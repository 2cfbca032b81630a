for g in 16 74 148; do timeout 120 python tools/gemv_sweep.py --cfg quip2 --shapes 4096x12288 --flags 36 --grid $g 2>&1 | tail -3; done
for g in 16 148; do timeout 120 python tools/gemv_sweep.py --cfg quip2 --shapes 4096x12288 --flags 100 --grid $g 2>&1 | tail -3; done
