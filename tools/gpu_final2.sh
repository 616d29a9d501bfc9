#!/bin/bash
# Final GPU pass: suite, both bench arms, smoke, launch list, pass-kernel ncu
mkdir -p gpurun_out
bash tools/gpu_tests.sh 2400
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo launches_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 0 -c 1 -o gpurun_out/r2_pass_kernel_final python tools/profile_case.py --passes 3 > gpurun_out/ncu_pass.log 2>&1; echo ncu_pass_rc=$?
