mkdir -p gpurun_out
timeout 600 python -m pytest -m gpu -q -rf tests/test_sharded_gpu.py tests/test_golden_runs_gpu.py > gpurun_out/pytest_part.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_part.log
# plain run of the 1024-thread helper case first (does it fault?)
FLEETPLACE_THREADS=1024 FLEETPLACE_HELPERS=-1 FLEETPLACE_ALLOW_1024_HELPERS=1 timeout 300 python tools/sanitize_case.py h40k > gpurun_out/h40k_1024.log 2>&1; echo h40k_1024_rc=$?; tail -3 gpurun_out/h40k_1024.log
FLEETPLACE_THREADS=1024 FLEETPLACE_HELPERS=-1 FLEETPLACE_ALLOW_1024_HELPERS=1 timeout 300 python tools/sanitize_case.py c2 > gpurun_out/c2_1024.log 2>&1; echo c2_1024_rc=$?; tail -3 gpurun_out/c2_1024.log
bash tools/sanitize.sh
