#!/bin/bash
# GPU test pass: the whole -m gpu suite, log under gpurun_out/
mkdir -p gpurun_out
timeout ${1:-1500} python -m pytest tests -m gpu -q -rf ${2:-} > gpurun_out/pytest_gpu.log 2>&1
echo pytest_rc=$?
tail -15 gpurun_out/pytest_gpu.log
