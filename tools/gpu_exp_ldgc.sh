for e in 0 1 0 1; do VQB_GEMV_LDGC=$e python bench.py --steps 20 --warmup 5 --no-extra --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('LDGC=$e', round(d['value']), round(d['ms_per_step'],4))"; done
VQB_GEMV_LDGC=1 timeout 300 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "group" 2>&1 | tail -2
