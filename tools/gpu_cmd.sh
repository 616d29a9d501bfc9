mkdir -p gpurun_out
timeout 600 python tools/c5_e2e_probe.py > gpurun_out/c5_e2e_probe.log 2>&1; echo rc=$?; cat gpurun_out/c5_e2e_probe.log | grep -v trace
