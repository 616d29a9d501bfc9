#!/bin/bash
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; echo rc=$?
tail -c 3000 gpurun_out/bench_r1.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r1.json 2>&1; tail -c 1500 gpurun_out/bench_ref_r1.json
