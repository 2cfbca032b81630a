timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -1 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; python -c "
import json; d=json.load(open('gpurun_out/bench1.json'))
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks']); print(d['per_linear']); print(d['attention_c4']['us_per_call'], [x['tokens_per_s'] for x in d['decode_c5']])"
for r in 2 4 8; do timeout 300 python tools/gemv_sweep.py --cfg quip2 --shapes 4096x12288 --rows $r 2>&1 | tail -1; done
timeout 900 python tools/decode_bench.py 1 8 16 64 2>&1 | tail -4
