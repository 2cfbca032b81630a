timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "gemm" 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --only gemm_c2,c3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ('gemm_c2_prefill',):
  print(k, d[k]['roofline'], {n: (v['kernel'], v['us_per_call'], v['paths']) for n,v in d[k]['per_linear'].items()})
g=d['c3_aqlm65b']['gemm_rows1024_tp1']; print('c3', g['roofline'], {n: (v['kernel'], v['us_per_call'], v['paths']) for n,v in g['per_linear'].items()})"
