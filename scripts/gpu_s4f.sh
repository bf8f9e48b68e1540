#!/bin/bash
# session 4: k1w_syrk_i8 thin last-block items -- bitwise comparison with the session's base
# build on the stress cube, syrk time under ncu (SMF_I8_THIN=0/1), the wide statistics tests
mkdir -p gpurun_out/s4f
O=gpurun_out/s4f
COLS=598 OUT=/tmp/base.npz VARIANT_ROOT=scripts/debug/variants/base timeout 900 python scripts/debug/bitwise_ab.py 2>&1 | tail -1
COLS=598 OUT=/tmp/new.npz VARIANT_ROOT=. timeout 900 python scripts/debug/bitwise_ab.py 2>&1 | tail -1
python - <<'PY'
import numpy as np
a, b = np.load('/tmp/base.npz'), np.load('/tmp/new.npz')
for k in ('enh', 'alb', 'st'):
    x, y = a[k], b[k]
    print(k, 'bitwise identical' if x.tobytes() == y.tobytes() else 'DIFFERENT: max|d| %g' % np.nanmax(np.abs(x.astype(np.float64) - y)))
PY
for v in 0 1 0 1; do
  SMF_I8_THIN=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1w_syrk" python scripts/debug/one_retrieve.py stress 2>&1 | grep -E 'gpu__time' | tail -1 | sed "s/^/thin=$v /"
done > $O/syrk_times.txt 2>&1
cat $O/syrk_times.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "wide or stress or b626 or multi_run or grouped" > $O/gpu_tests_wide.log 2>&1; echo tests_rc=$?; tail -5 $O/gpu_tests_wide.log
