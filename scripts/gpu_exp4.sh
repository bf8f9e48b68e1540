#!/bin/bash
# k2w_init -> k = 0 sweep overlap (ready flags) A/B on the stress bench, then the GPU tests
mkdir -p gpurun_out/e4
for ov in 0 1; do
SMF_INIT_OVERLAP=$ov timeout 900 python bench.py --config stress > gpurun_out/e4/bench_stress_ov$ov.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/e4/bench_stress_ov$ov.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('overlap $ov', 'ms', round(d['ms_per_step'],3), 'frac', round(r['frac'],3), 'step', round(r['step_frac'],3), d['clocks']['sm_mhz'], {k: round(v,3) for k,v in r['kernel_ms_per_step'].items()})"
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/e4/gpu_tests.log 2>&1; echo tests_rc=$?
tail -3 gpurun_out/e4/gpu_tests.log
