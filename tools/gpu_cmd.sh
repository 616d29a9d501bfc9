mkdir -p gpurun_out
timeout 900 python tools/c3_phase_probe.py 5000,1000000,250 1 2 > gpurun_out/c4_phase.log 2>&1; echo rc=$?; cat gpurun_out/c4_phase.log
