#!/bin/bash
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for T in 512 1024; do
FLEETPLACE_THREADS=$T python bench.py --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($T, d['ms_per_step'], d['phase_ms'], d['event_counts'], d['search_stats']['evaluations'], d['search_stats']['applied_moves'])"
done
