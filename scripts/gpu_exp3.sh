#!/bin/bash
# sweep instruction-diet A/B on the stress shape (HEAD variant vs working tree), then the GPU tests
mkdir -p gpurun_out/e3
for rep in 1 2; do
VARIANT=head VARIANT_ROOT=scripts/debug/variants/head timeout 300 python scripts/debug/stress_time.py 2>&1 | tail -1
VARIANT=new timeout 300 python scripts/debug/stress_time.py 2>&1 | tail -1
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/e3/gpu_tests.log 2>&1; echo tests_rc=$?
tail -3 gpurun_out/e3/gpu_tests.log
