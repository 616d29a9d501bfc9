#!/bin/bash
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python bench.py --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms'], d['event_counts'], d['search_stats'])"
timeout 1200 python tools/scale_probe.py --c4 --passes 1,3 2>&1 | tail -3
timeout 600 python tools/scale_probe.py --c5 296 2>&1 | tail -2
