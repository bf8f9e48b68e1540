#!/bin/bash
# stress-config (B = 425) parity + bench + ncu of the wide kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -k "wide or stress" > gpurun_out/tw.log 2>&1; echo tests_rc=$?; grep -E "passed|failed" gpurun_out/tw.log
B="python bench.py --config stress --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 900 python bench.py --config stress --steps 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bstress.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bstress.log').read().strip().splitlines()[-1]); r=d['roofline']
print(d['value']/1e9, d['ms_per_step'], r['frac'], r['step_frac'], r['kernel_time_share'], r['avg_launch_us'])"
if [ "${NCU:-0}" = 1 ]; then
  timeout 600 $B > gpurun_out/plain_s.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k1w|k2w_init|k3w" -c 3 -o gpurun_out/wide -f $B > gpurun_out/ncu_wide.log 2>&1; echo ncu_rc=$?
fi
