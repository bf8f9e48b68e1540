#!/bin/bash
# k2w_init phase knock-out timings (one wave of 148 stress columns; results of the variants are garbage)
for v in base noc2 nodiag nopanel noc1 nofact; do
  echo -n "$v "; COLS=148 VARIANT_ROOT=scripts/debug/variants/x_$v timeout 300 python scripts/debug/init_waves.py 2>&1 | tail -1
done
