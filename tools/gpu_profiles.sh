#!/bin/bash
# Profile pass for the final round-2 build: bench launch list (no extras) and
# ncu --set full of kernel (1)'s site haversines (glibc restatement) at c4.
mkdir -p gpurun_out
timeout 600 python tools/table_probe.py 5000,1000000,250 > gpurun_out/table_probe.log 2>&1; echo probe_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo launches_rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:site_hav -c 1 -o gpurun_out/r2_site_hav python tools/table_probe.py 5000,1000000,250 > gpurun_out/ncu_site.log 2>&1; echo site_rc=$?
