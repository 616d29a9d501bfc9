#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r1c.json 2> gpurun_out/bench_r1c.err; echo rc=$?; tail -3 gpurun_out/bench_r1c.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r1c.json 2> gpurun_out/bench_ref_r1c.err; echo refrc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
