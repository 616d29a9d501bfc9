#!/bin/bash
python -m pytest tests -m gpu -q 2>&1 | tail -1
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err; echo rc=$?; tail -3 gpurun_out/bench_r1b.err
python -c "
import json; d=json.load(open('gpurun_out/bench_r1b.json'))
print(d['value'], d['ms_per_step'], d['e2e'], d['cpu_baseline']['value'])
print(json.dumps(d['extra_workloads'], indent=1))
"
