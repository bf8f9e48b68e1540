#!/bin/bash
# session 4: (1) paired-N int8 SYRK MMAs and (2) the k2w_init tail wave on a second stream --
# bitwise comparison with HEAD's build (variants/base), syrk time under ncu, stress A/B of the
# tail split, then the -m gpu suite
mkdir -p gpurun_out/s4b
O=gpurun_out/s4b
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
  if [ $v = base ]; then R=scripts/debug/variants/base; else R=.; fi
  VARIANT_ROOT=$R timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1w_syrk|k2w_init" python scripts/debug/one_retrieve.py stress 2>&1 | grep -E 'k1w_syrk|k2w_init|gpu__time' | tail -8 | sed "s/^/$v /"
done > $O/syrk_times.txt 2>&1
cat $O/syrk_times.txt
VAR=SMF_TAIL_SPLIT ARGS="--config stress" TESTS=0 STEPS=10 bash scripts/gpu_ab.sh 2>&1 | tee $O/tail_ab.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo tests_rc=$?; tail -3 $O/gpu_tests.log
