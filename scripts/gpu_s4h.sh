#!/bin/bash
# session 4: k2w_update with L2 prefetch of the factor tiles (SMF_K2W_PREFETCH=8) vs none
# (variants/pf0): bitwise comparison with the session's base build, per-kernel times
# (bracketed, scripts/debug/stress_time.py) alternating, k2w_update under ncu
mkdir -p gpurun_out/s4h
O=gpurun_out/s4h
COLS=598 OUT=/tmp/base.npz VARIANT_ROOT=scripts/debug/variants/base timeout 900 python scripts/debug/bitwise_ab.py 2>&1 | tail -1
COLS=598 OUT=/tmp/new.npz VARIANT_ROOT=. timeout 900 python scripts/debug/bitwise_ab.py 2>&1 | tail -1
python - <<'PY'
import numpy as np
a, b = np.load('/tmp/base.npz'), np.load('/tmp/new.npz')
for k in ('enh', 'alb', 'st'):
    x, y = a[k], b[k]
    print(k, 'bitwise identical' if x.tobytes() == y.tobytes() else 'DIFFERENT: max|d| %g' % np.nanmax(np.abs(x.astype(np.float64) - y)))
PY
for r in 1 2 3; do
for v in pf0 new; do
  if [ $v = new ]; then R=.; else R=scripts/debug/variants/$v; fi
  VARIANT=$v VARIANT_ROOT=$R timeout 600 python scripts/debug/stress_time.py 2>&1 | tail -1
done; done | tee $O/stress_time.txt
for v in pf0 new; do
  if [ $v = new ]; then R=.; else R=scripts/debug/variants/$v; fi
  VARIANT_ROOT=$R timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k2w_update" -s 35 -c 3 python scripts/debug/one_retrieve.py stress 2>&1 | grep -E 'gpu__time|dram__bytes|hit_rate' | tail -9 | sed "s/^/$v /"
done | tee $O/update_ncu.txt
