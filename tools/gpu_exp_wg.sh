python bench.py --steps 20 --warmup 5 --no-extra --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('WG1', d['value'], d['ms_per_step'])"
VQB_GEMV_GROUP_WG=2 python bench.py --steps 20 --warmup 5 --no-extra --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('WG2', d['value'], d['ms_per_step'])"
VQB_GEMV_GROUP_WG=2 timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "group" 2>&1 | tail -2
