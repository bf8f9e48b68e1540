#!/bin/bash
# session 4: k2w_update with two factor tiles per ring stage (2 stages x 16 KB) vs the session's
# base build (3 stages x 8 KB): bitwise comparison, k2w_update under ncu, per-kernel times, then
# the -m gpu suite
mkdir -p gpurun_out/s4l
O=gpurun_out/s4l
COLS=598 OUT=/tmp/base.npz VARIANT_ROOT=scripts/debug/variants/base timeout 900 python scripts/debug/bitwise_ab.py 2>&1 | tail -1
COLS=598 OUT=/tmp/new.npz VARIANT_ROOT=. timeout 900 python scripts/debug/bitwise_ab.py 2>&1 | tail -1
python - <<'PY'
import numpy as np
a, b = np.load('/tmp/base.npz'), np.load('/tmp/new.npz')
for k in ('enh', 'alb', 'st'):
    x, y = a[k], b[k]
    print(k, 'bitwise identical' if x.tobytes() == y.tobytes() else 'DIFFERENT: max|d| %g' % np.nanmax(np.abs(x.astype(np.float64) - y)))
PY
for v in base new; do
  if [ $v = new ]; then R=.; else R=scripts/debug/variants/$v; fi
  VARIANT_ROOT=$R timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,launch__occupancy_limit_shared_mem --clock-control none -k regex:"k2w_update" -s 35 -c 2 python scripts/debug/one_retrieve.py stress 2>&1 | grep -E 'gpu__time|inst_exec|occupancy' | tail -6 | sed "s/^/$v /"
done | tee $O/update_ncu.txt
for r in 1 2; do
for v in base new; do
  if [ $v = new ]; then R=.; else R=scripts/debug/variants/$v; fi
  VARIANT=$v VARIANT_ROOT=$R timeout 600 python scripts/debug/stress_time.py 2>&1 | tail -1
done; done | tee $O/stress_time.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo tests_rc=$?; tail -3 $O/gpu_tests.log
