#!/bin/bash
# session 4: SMF_TAIL_SPLIT 1 vs 2 on the stress bench, 8 alternations
mkdir -p gpurun_out/s4j
O=gpurun_out/s4j
B="python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --config stress"
for r in 1 2 3 4 5 6 7 8; do
  for v in 1 2; do
    env SMF_TAIL_SPLIT=$v timeout 600 $B > $O/ab_${v}_$r.log 2>&1
    python -c "import json; d=json.loads(open('$O/ab_${v}_$r.log').read().strip().splitlines()[-1]); print('SMF_TAIL_SPLIT=$v', round(d['ms_per_step'],3), 'ms', d['clocks']['sm_mhz'])"
  done
done | tee $O/tail_ab12.txt
