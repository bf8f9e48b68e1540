#!/bin/bash
for v in head new; do
  if [ $v = head ]; then R=scripts/debug/variants/head; else R=.; fi
  VARIANT_ROOT=$R timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:k1w_syrk python scripts/debug/one_retrieve.py stress 2>&1 | grep -E 'gpu__time|inst_executed' | tail -2 | sed "s/^/$v /"
done
