mkdir -p gpurun_out
timeout 1500 python -m pytest -m gpu -q -rf --timeout 600 tests > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?; tail -2 gpurun_out/bench.err
