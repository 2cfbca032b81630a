timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_t11_gpu.log 2>&1
echo t rc=$?
timeout 900 python bench.py --only attention_c4,decode_c5,gemv_c2,gemv_c1 --no-cpu --steps 10 > gpurun_out/r02_b11.json 2> gpurun_out/r02_b11.err
echo b rc=$?
python tools/attn_trace.py 1 32 4096 > gpurun_out/r02_attn_trace11.log 2>&1
