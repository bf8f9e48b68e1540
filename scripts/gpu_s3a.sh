#!/bin/bash
# session-3 re-entry check: GPU tests, smoke, bench lines for flightline and stress
mkdir -p gpurun_out/s3a
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/s3a/gpu_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/s3a/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/s3a/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/s3a/smoke.log
for c in flightline stress; do
  timeout 900 python bench.py --config $c > gpurun_out/s3a/bench_$c.log 2>&1; echo bench_${c}_rc=$?
  tail -1 gpurun_out/s3a/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['workload'][:40], 'ms', round(d['ms_per_step'],3), 'frac', round(r['frac'],3), 'step', round(r.get('step_frac',0),3), d['clocks'])"
done
