#!/bin/bash
# GPU state check: the -m gpu suite, smoke, flightline + stress bench lines
mkdir -p gpurun_out/chk
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/chk/gpu_tests.log 2>&1; echo tests_rc=$?
tail -3 gpurun_out/chk/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk/smoke.log 2>&1; echo smoke_rc=$?
for c in flightline stress; do
  timeout 900 python bench.py --config $c > gpurun_out/chk/bench_$c.log 2>&1; echo bench_${c}_rc=$?
  tail -1 gpurun_out/chk/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['workload'][:40], 'ms', round(d['ms_per_step'],3), 'frac', round(r['frac'],3), 'step', round(r['step_frac'],3), d['clocks']['sm_mhz'])"
done
