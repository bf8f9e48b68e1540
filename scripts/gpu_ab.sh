#!/bin/bash
# A/B: GPU parity tests, then the default bench line with an env toggle off/on, alternating.
# usage: VAR=SMF_SERPENTINE bash scripts/gpu_ab.sh
mkdir -p gpurun_out
VAR=${VAR:-SMF_SERPENTINE}
if [ "${TESTS:-1}" = 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
  echo rc=$? >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
fi
B="python bench.py --steps ${STEPS:-10} --warmup 3 --e2e-steps 0 --no-cpu-baseline ${ARGS:-}"
for r in 1 2; do
  for v in ${VALS:-0 1}; do
    env $VAR=$v timeout 600 $B > gpurun_out/ab_${v}_$r.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/ab_${v}_$r.log').read().strip().splitlines()[-1]); print('$VAR=$v', round(d['ms_per_step'],3), 'ms', d['roofline']['kernel_time_share'])"
  done
done
