#!/bin/bash
# session 4: k2w_update ring shapes at the same 32 KB: 4 stages x 1 tile (variants/s4x1) vs
# 2 stages x 2 tiles (default), under ncu
mkdir -p gpurun_out/s4o
for v in s4x1 new s4x1 new; do
  if [ $v = new ]; then R=.; else R=scripts/debug/variants/$v; fi
  VARIANT_ROOT=$R timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,launch__occupancy_limit_shared_mem --clock-control none -k regex:"k2w_update" -s 35 -c 2 python scripts/debug/one_retrieve.py stress 2>&1 | grep -E 'gpu__time|inst_exec|occupancy' | tail -6 | sed "s/^/$v /"
done | tee gpurun_out/s4o/update_ncu.txt
