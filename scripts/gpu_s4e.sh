#!/bin/bash
# session 4: k1w_syrk_i8 with 8 epilogue warps (two per TMEM lane quadrant) vs 4 (variants/epi4):
# bitwise comparison with the session's base build, syrk time under ncu, stress bench A/B
mkdir -p gpurun_out/s4e
O=gpurun_out/s4e
COLS=598 OUT=/tmp/base.npz VARIANT_ROOT=scripts/debug/variants/base timeout 900 python scripts/debug/bitwise_ab.py 2>&1 | tail -1
COLS=598 OUT=/tmp/new.npz VARIANT_ROOT=. timeout 900 python scripts/debug/bitwise_ab.py 2>&1 | tail -1
python - <<'PY'
import numpy as np
a, b = np.load('/tmp/base.npz'), np.load('/tmp/new.npz')
for k in ('enh', 'alb', 'st'):
    x, y = a[k], b[k]
    print(k, 'bitwise identical' if x.tobytes() == y.tobytes() else 'DIFFERENT: max|d| %g' % np.nanmax(np.abs(x.astype(np.float64) - y)))
PY
for v in epi4 new epi4 new; do
  if [ $v = new ]; then R=.; else R=scripts/debug/variants/$v; fi
  VARIANT_ROOT=$R timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1w_syrk" python scripts/debug/one_retrieve.py stress 2>&1 | grep -E 'gpu__time' | tail -1 | sed "s/^/$v /"
done > $O/syrk_times.txt 2>&1
cat $O/syrk_times.txt
