mkdir -p gpurun_out
# multi-rank host protocol, functional check: 2 ranks over gloo on the one GPU (no number is kept)
FLEETPLACE_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank_gloo.err; echo rc=$?; tail -5 gpurun_out/bench_2rank_gloo.err
