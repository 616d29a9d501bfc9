mkdir -p gpurun_out
bash tools/gpu_tests.sh 2400
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?; tail -c 300 gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
FLEETPLACE_NVCC_DEFS=FP_PHASE_CLOCKS timeout 900 python -m paper_2001_05291_b200._build --force > /dev/null 2>&1; echo probe_build=$?
timeout 600 python tools/c3_phase_probe.py 500,10000,40 3 194 198 none > gpurun_out/r2_c2_phase_clocks.log 2>&1; echo phase_rc=$?
timeout 600 python tools/c5_tail_probe.py 40 > gpurun_out/r2_c5_tail_phase.log 2>&1
