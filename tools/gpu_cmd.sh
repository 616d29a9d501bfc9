mkdir -p gpurun_out
timeout 600 python tools/table_probe.py > gpurun_out/table_probe.log 2>&1; echo table_rc=$?; cat gpurun_out/table_probe.log
CHAIN_CFGS=0 timeout 600 python tools/chain_probe.py > gpurun_out/chain_probe.log 2>&1; echo chain_rc=$?; cat gpurun_out/chain_probe.log
timeout 900 python -m pytest -m gpu -q -rf tests/test_kernels_gpu.py tests/test_sharded_gpu.py tests/test_golden_runs_gpu.py > gpurun_out/pytest_part.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_part.log
