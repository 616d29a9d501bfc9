#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | grep -E "FAILED|passed|failed" | head -3
python tools/profile_case.py --passes 4 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 1 -c 1 -o gpurun_out/pass_full3 python tools/profile_case.py --passes 4 > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
