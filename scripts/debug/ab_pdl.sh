mkdir -p gpurun_out
[ "${TESTS:-1}" = 1 ] && timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$?; tail -1 gpurun_out/gpu_tests.log
B="python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
for r in 1 2; do for pdl in 0 1; do for prof in 1 0; do
 SMF_PDL=$pdl SMF_BENCH_PROF=$prof timeout 600 $B > gpurun_out/x.log 2>&1
 python -c "import json; d=json.loads(open('gpurun_out/x.log').read().strip().splitlines()[-1]); print('pdl=$pdl prof=$prof', round(d['ms_per_step'],3))" || tail -3 gpurun_out/x.log
done; done; done
