#!/bin/bash
# k2w_update ring-depth variants (per-kernel times on the stress shape), then the wide GPU tests
mkdir -p gpurun_out/e2
for v in s2 s3; do
  VARIANT=$v VARIANT_ROOT=scripts/debug/variants/$v timeout 300 python scripts/debug/stress_time.py 2>&1 | tail -1
done
VARIANT=s4 timeout 300 python scripts/debug/stress_time.py 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/e2/gpu_tests.log 2>&1; echo tests_rc=$?
tail -3 gpurun_out/e2/gpu_tests.log
