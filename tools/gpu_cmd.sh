mkdir -p gpurun_out
python tools/chain_probe.py c3 > gpurun_out/plain_chain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:column_chain -s 1 -c 1 -o gpurun_out/r2_column_chain python tools/chain_probe.py c3 > gpurun_out/ncu_chain.log 2>&1; echo ncu_rc=$?
