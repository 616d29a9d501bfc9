mkdir -p gpurun_out
timeout 600 python tools/c3_phase_probe.py > gpurun_out/c3_phase.log 2>&1; echo rc=$?; cat gpurun_out/c3_phase.log
timeout 600 python tools/c2_pass_profile.py > gpurun_out/c2_pass_profile.log 2>&1; echo rc=$?; tail -5 gpurun_out/c2_pass_profile.log
timeout 1500 python -m pytest -m gpu -q -rf -x --timeout 300 tests > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?; tail -2 gpurun_out/bench.err
