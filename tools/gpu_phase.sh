#!/bin/bash
# Phase-clock probe pass: rebuild with FP_PHASE_CLOCKS on the box, then c2 prefixes and the c5 tail scenario.
mkdir -p gpurun_out
FLEETPLACE_NVCC_DEFS=FP_PHASE_CLOCKS timeout 900 python -m paper_2001_05291_b200._build --force > /dev/null 2>&1; echo probe_build=$?
timeout 600 python tools/c3_phase_probe.py 500,10000,40 1 2 3 none > gpurun_out/c2_phase.log 2>&1; echo phase_rc=$?
timeout 600 python tools/c5_tail_probe.py 40 > gpurun_out/c5_tail_phase.log 2>&1; echo tail_rc=$?
