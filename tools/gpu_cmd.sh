mkdir -p gpurun_out
FLEETPLACE_TRACE=1 timeout 600 python tools/c5_outlier_probe.py 4 > gpurun_out/c5_outlier.log 2>&1; echo rc=$?; tail -12 gpurun_out/c5_outlier.log
