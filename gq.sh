#!/bin/bash
python -m pytest tests/test_parity_gpu.py tests/test_edge_cases_gpu.py -q -x 2>&1 | tail -2
timeout 1200 python tools/scale_probe.py --c4 --passes 1 2>&1 | tail -1
