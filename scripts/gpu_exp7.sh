#!/bin/bash
# compact diagonal factor: GPU tests, stress bench, microbenchmark
mkdir -p gpurun_out/e7
./scripts/micro/diag_bench
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/e7/gpu_tests.log 2>&1; echo tests_rc=$?
tail -3 gpurun_out/e7/gpu_tests.log
timeout 900 python bench.py --config stress > gpurun_out/e7/bench_stress.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/e7/bench_stress.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('stress ms', round(d['ms_per_step'],3), 'frac', round(r['frac'],3), 'step', round(r['step_frac'],3), d['clocks']['sm_mhz'], {k: round(v,3) for k,v in r['kernel_ms_per_step'].items()})"
