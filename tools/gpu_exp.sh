mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
SECONDS=0; timeout 600 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench wall $SECONDS s"
python -c "
import json; d=json.load(open('gpurun_out/bench1.json'))
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'])
print(d['attention_c4']['us_per_call'], [x['tokens_per_s'] for x in d['decode_c5']])"
