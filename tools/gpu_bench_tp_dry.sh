# multi-GPU bench code path on one GPU: two ranks on cuda:0 over gloo (timings meaningless)
VQB_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/bench_tp_dry.json 2> gpurun_out/bench_tp_dry.err
echo rc=$?; tail -5 gpurun_out/bench_tp_dry.err; head -c 1500 gpurun_out/bench_tp_dry.json
