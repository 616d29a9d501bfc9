#!/bin/bash
# prep_words words-in-flight knob: c5 tail scenarios and the c5 share, UW=4 (shipped) vs 8 (probe build)
mkdir -p gpurun_out
for rep in 1 2; do timeout 300 python tools/c5_tail_probe.py 29,40 2>&1 | grep "threads 256"; done > gpurun_out/uw4.log
timeout 300 python tools/c5_e2e_probe.py 512 2>&1 | grep call >> gpurun_out/uw4.log
FLEETPLACE_NVCC_DEFS=FP_PREP_UW=8 timeout 900 python -m paper_2001_05291_b200._build --force > /dev/null 2>&1; echo build=$?
for rep in 1 2; do timeout 300 python tools/c5_tail_probe.py 29,40 2>&1 | grep "threads 256"; done > gpurun_out/uw8.log
timeout 300 python tools/c5_e2e_probe.py 512 2>&1 | grep call >> gpurun_out/uw8.log
