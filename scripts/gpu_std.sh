mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench.log 2>&1; echo bench_rc=$?
python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu_rc=$?
