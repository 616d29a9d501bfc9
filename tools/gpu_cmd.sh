mkdir -p gpurun_out
timeout 600 python tools/c4_rank_probe.py > gpurun_out/c4_rank.log 2>&1; echo rc=$?; cat gpurun_out/c4_rank.log
