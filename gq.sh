#!/bin/bash
python -m pytest tests/test_acceptance_gpu.py -q -x 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
