#!/bin/bash
# session 4: k2w_update L2 prefetch distance 0 / 2 / 4 / 8 tiles under ncu
mkdir -p gpurun_out/s4h
for v in pf0 pf2 pf4 new; do
  if [ $v = new ]; then R=.; else R=scripts/debug/variants/$v; fi
  VARIANT_ROOT=$R timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k2w_update" -s 35 -c 2 python scripts/debug/one_retrieve.py stress 2>&1 | grep -E 'gpu__time|dram__bytes|hit_rate' | tail -6 | sed "s/^/$v /"
done | tee gpurun_out/s4h/update_ncu_pf.txt
