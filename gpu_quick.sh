#!/bin/bash
python bench.py --steps 1 --warmup 1 2>&1 | tail -5
