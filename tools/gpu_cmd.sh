mkdir -p gpurun_out
timeout 1500 python -m pytest -m gpu -q -rf -x --timeout 300 tests > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
FLEETPLACE_TRACE=1 timeout 600 python tools/c5_e2e_probe.py > gpurun_out/c5_e2e_probe.log 2>&1; echo rc=$?; grep -v "^\[fleetplace trace\]" gpurun_out/c5_e2e_probe.log; grep "fleetplace trace" gpurun_out/c5_e2e_probe.log | tail -6
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?; tail -2 gpurun_out/bench.err
