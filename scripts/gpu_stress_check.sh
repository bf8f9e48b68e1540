#!/bin/bash
# wide-path change check: the -m gpu suite, then the stress bench line and its kernel split
mkdir -p gpurun_out/sc
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/sc/gpu_tests.log 2>&1; echo tests_rc=$?
tail -3 gpurun_out/sc/gpu_tests.log
for st in ${STAGES:-3}; do
SMF_K2W_STAGES=$st timeout 900 python bench.py --config stress > gpurun_out/sc/bench_stress_s$st.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/sc/bench_stress_s$st.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('stages $st', 'ms', round(d['ms_per_step'],3), 'frac', round(r['frac'],3), 'step', round(r['step_frac'],3), d['clocks']['sm_mhz'], {k: round(v,3) for k,v in r['kernel_ms_per_step'].items()})"
done
