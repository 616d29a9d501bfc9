mkdir -p gpurun_out
FLEETPLACE_TRACE=1 timeout 600 python tools/c5_outlier_probe.py 14 > gpurun_out/c5_outlier.log 2>&1; echo rc=$?; grep "call " gpurun_out/c5_outlier.log
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
