mkdir -p gpurun_out
python tools/profile_case.py --passes 196 > gpurun_out/plain_pass195.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 194 -c 1 -o gpurun_out/r2_pass195 python tools/profile_case.py --passes 196 > gpurun_out/ncu_pass195.log 2>&1; echo ncu_rc=$?
