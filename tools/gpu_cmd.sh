mkdir -p gpurun_out
timeout 600 python tools/multistep_probe.py > gpurun_out/multistep.log 2>&1; echo rc=$?; cat gpurun_out/multistep.log
