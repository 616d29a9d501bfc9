mkdir -p gpurun_out
cd oracle/_ref && timeout 300 ./acceptance_b200 > ../../gpurun_out/acc_b200.log 2>&1; echo acc_rc=$?; cd ../..
tail -5 gpurun_out/acc_b200.log
timeout 900 python -m pytest -m gpu -q -rf tests/test_kernels_gpu.py tests/test_golden_runs_gpu.py tests/test_parity_gpu.py tests/test_sharded_gpu.py > gpurun_out/pytest_part.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_part.log
timeout 600 python tools/chain_probe.py > gpurun_out/chain_probe.log 2>&1; echo chain_rc=$?; cat gpurun_out/chain_probe.log
