#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo bench_rc=$?
FLEETPLACE_TRACE=1 timeout 300 python tools/e2e_trace.py > gpurun_out/e2e_trace.log 2>&1; echo trace_rc=$?
