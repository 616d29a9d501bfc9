mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:table_gather_packed -c 1 -o gpurun_out/r2_table_gather_packed python tools/table_probe.py 5000,1000000,250 > gpurun_out/ncu_tg.log 2>&1; echo rc=$?; tail -3 gpurun_out/ncu_tg.log
