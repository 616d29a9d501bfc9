#!/bin/bash
# GPU bench pass: the driver's two arms (ours, reference), smoke, and
# optionally the reference's full c2 run on the box host (REF_FULL=1).
mkdir -p gpurun_out
if [ "${REF_FULL:-0}" = 1 ]; then
  nohup python tools/ref_full_run.py gpurun_out/r2_ref_c2_full.json > gpurun_out/ref_full.log 2>&1 &
  REFPID=$!
fi
timeout 900 python bench.py --steps ${STEPS:-5} --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
tail -3 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps ${STEPS:-5} --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
if [ -n "$REFPID" ]; then wait $REFPID; echo ref_full_rc=$?; fi
