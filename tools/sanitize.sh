#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the search kernels
# (SURVEY §5); logs under gpurun_out/sanitize/.
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool case [env...]
  local tool=$1 case=$2; shift 2
  local tag=${tool}_${case}${1:+_$(echo "$*" | tr ' =' '__')}
  env "$@" timeout 1200 $CS --tool $tool --error-exitcode 99 --print-limit 20 \
      python tools/sanitize_case.py $case > gpurun_out/sanitize/$tag.log 2>&1
  echo "$tag rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize/$tag.log | tail -1)"
}
run memcheck c1
run memcheck c2
run memcheck h40k
run memcheck c5b
run synccheck c1
run synccheck c2
run synccheck h40k
run racecheck c1
run racecheck c5b
run memcheck h40k FLEETPLACE_THREADS=1024 FLEETPLACE_HELPERS=-1 FLEETPLACE_ALLOW_1024_HELPERS=1
run synccheck h40k FLEETPLACE_THREADS=1024 FLEETPLACE_HELPERS=-1 FLEETPLACE_ALLOW_1024_HELPERS=1
