#!/bin/bash
# time K1 (+K0/K2init) for each built variant under scripts/debug/variants (debug aid)
for r in 1 2; do
for v in ${VARS:-$(ls scripts/debug/variants)}; do
  VARIANT=$v VARIANT_ROOT=$PWD/scripts/debug/variants/$v K1_KERNELS=tensor timeout 300 python scripts/debug/k1_time.py 2>&1 | tail -1
done; done
