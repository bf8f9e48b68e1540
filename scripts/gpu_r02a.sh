#!/bin/bash
# round-2 check: full GPU suite, then bench lines for flightline / segment / stress
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo tests_rc=$?; grep -E "passed|failed" gpurun_out/gpu_tests.log | tail -2
for c in flightline segment stress; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; echo bench_${c}_rc=$?
  tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['workload'], 'ms', round(d['ms_per_step'],3), 'k3frac', round(r['frac'],3), 'stepfrac', round(r['step_frac'],3), {k: round(v,3) for k,v in r['kernel_ms_per_step'].items()}, d['clocks'])"
done
