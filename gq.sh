#!/bin/bash
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extras 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms'], d['search_stats'], d['gpu_launches'])"
timeout 600 python tools/scale_probe.py --c5 296 2>&1 | grep "c5 batch" | head -1
timeout 600 python tools/scale_probe.py --c3 --passes 1,10 2>&1 | tail -2
