#!/bin/bash
mkdir -p gpurun_out
bash tools/gpu_tests.sh 2400
timeout 900 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo bench_rc=$?
