set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
timeout 600 python bench.py --no-cpu > gpurun_out/bench1.json 2> gpurun_out/bench1.err
python -c "
import json; d=json.load(open('gpurun_out/bench1.json'))
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'])
print(d['per_linear']); print(d['attention_c4']['us_per_call'], [x['tokens_per_s'] for x in d['decode_c5']])
print(d['gemv_c1_gptvq2_q_proj']['us_per_call'], d['gemv_c2_quip2_q_proj']['us_per_call'])"
for r in 1 2; do python tools/gemv_sweep.py --cfg quip2 --shapes 4096x12288 --rows $r 2>&1 | tail -1; done
