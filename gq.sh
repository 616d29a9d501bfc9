#!/bin/bash
python -m pytest tests/test_kernels_gpu.py tests/test_reference_ports_gpu.py -q -x 2>&1 | tail -2
python tools/profile_case.py --shape 5000,1000000,250 --passes 1 > gpurun_out/c4_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:column_totals --csv --log-file gpurun_out/c4_ct.csv python tools/profile_case.py --shape 5000,1000000,250 --passes 1 > /dev/null 2>&1
grep -E "duration|dram" gpurun_out/c4_ct.csv | cut -c1-250
python tools/profile_case.py --shape 500,10000,40 --passes 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:column_totals --csv python tools/profile_case.py --shape 500,10000,40 --passes 1 2>/dev/null | grep duration | cut -c1-200
