#!/bin/bash
mkdir -p gpurun_out
bash tools/gpu_tests.sh 2400
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 600 python tools/c3_trace.py > gpurun_out/c3_trace.log 2>&1; echo trace_rc=$?
