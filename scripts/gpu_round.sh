#!/bin/bash
# One gpurun call: GPU parity tests, the default bench line, the ncu launch list and
# one `ncu --set full` capture each of k3_sweep and k1_stats.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -s -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo rc=$? >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?
B="python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 600 $B > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
echo ncu_list_rc=$?
if [ "${FULL:-1}" = 1 ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k3_sweep -s 100 -c 1 -o gpurun_out/k3 -f $B > gpurun_out/ncu_k3.log 2>&1; echo ncu_k3_rc=$?
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_stats -s 3 -c 1 -o gpurun_out/k1 -f $B > gpurun_out/ncu_k1.log 2>&1; echo ncu_k1_rc=$?
fi
