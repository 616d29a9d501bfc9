#!/bin/bash
mkdir -p gpurun_out
FLEETPLACE_NVCC_DEFS=FP_PHASE_CLOCKS timeout 900 python -m paper_2001_05291_b200._build --force > /dev/null 2>&1; echo probe_build=$?
timeout 600 python tools/c3_phase_probe.py 2000,100000,100 10 none > gpurun_out/c3_phase.log 2>&1; echo phase_rc=$?
