for r in 4 8 16 32 64; do python tools/gemv_sweep.py --rows $r --shapes 4096x4096,4096x12288,4096x22016,11008x4096 | grep -v smem | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print('tc', d['rows'], d['shape'], d['kernel'], d['us_per_call'], d['GB_s'], d['fp16_cublas_us'])"; done
for r in 4 8 16; do python tools/gemv_sweep.py --rows $r --flags 4096 --shapes 4096x4096,4096x12288,4096x22016,11008x4096 | grep -v smem | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print('old', d['rows'], d['shape'], d['kernel'], d['us_per_call'], d['GB_s'])"; done
