#!/bin/bash
# k2w_init ridge loop parallelised (+ streamed z0): per-wave times, bitwise A/B, tests
for v in head new; do
  if [ $v = head ]; then R=scripts/debug/variants/head; else R=.; fi
  echo -n "$v "; COLS=148,598 VARIANT_ROOT=$R timeout 300 python scripts/debug/init_waves.py 2>&1 | tail -2 | tr '\n' ' '; echo
done
bash scripts/gpu_exp9.sh 2>&1 | grep -v "^head {\|^new {"
