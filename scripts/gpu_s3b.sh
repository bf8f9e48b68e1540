#!/bin/bash
# reading C23 (fp32 off-diagonal factor stream): GPU tests, stress bench with and without it
mkdir -p gpurun_out/s3b
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/s3b/gpu_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/s3b/gpu_tests.log
for f in 1 0; do
  SMF_WIDE_F32=$f timeout 900 python bench.py --config stress --no-cpu-baseline --e2e-steps 0 > gpurun_out/s3b/bench_stress_f$f.log 2>&1; echo bench_f${f}_rc=$?
  tail -1 gpurun_out/s3b/bench_stress_f$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('f32=$f ms', round(d['ms_per_step'],3), 'step', round(r.get('step_frac',0),3), {k: round(v,3) for k,v in r['kernel_ms_per_step'].items()}, d['clocks']['sm_mhz'])"
done
