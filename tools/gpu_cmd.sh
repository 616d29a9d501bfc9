mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "small_first_term" -p no:cacheprovider > gpurun_out/unclamped.log 2>&1; echo rc=$?; tail -5 gpurun_out/unclamped.log
