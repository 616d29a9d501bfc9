#!/bin/bash
# GPU pass: the suite, the bench, and the c5 batch call's host/device trace
mkdir -p gpurun_out
bash tools/gpu_tests.sh 2400
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
FLEETPLACE_TRACE=1 timeout 600 python tools/c5_e2e_probe.py 512 > gpurun_out/c5_trace.log 2>&1; echo trace_rc=$?
