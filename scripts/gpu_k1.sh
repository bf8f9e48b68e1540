#!/bin/bash
# GPU parity tests + an ncu --set full capture of the statistics kernel.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo rc=$? >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
B="python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 600 $B > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_stats -s 3 -c 1 -o gpurun_out/k1 -f $B > gpurun_out/ncu_k1.log 2>&1; echo ncu_k1_rc=$?
