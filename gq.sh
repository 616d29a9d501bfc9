#!/bin/bash
python -m pytest tests/test_edge_cases_gpu.py -q -x 2>&1 | tail -25
