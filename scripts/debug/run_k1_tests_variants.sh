mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "stat or parity or tiny or segment" > gpurun_out/gpu_tests.log 2>&1; echo rc=$?; tail -1 gpurun_out/gpu_tests.log
bash scripts/debug/k1_variants.sh
