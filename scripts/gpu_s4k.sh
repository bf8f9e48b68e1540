#!/bin/bash
# session 4: k2w_update streaming a tile-major copy of the factor (one 8 KB bulk copy per tile)
# vs TMA boxes of the row-major factor (SMF_K2W_TILED=0): bitwise comparison with the session's
# base build, per-kernel times alternating, stress bench A/B, ncu of k2w_update / k2w_init
mkdir -p gpurun_out/s4k
O=gpurun_out/s4k
COLS=598 OUT=/tmp/base.npz VARIANT_ROOT=scripts/debug/variants/base timeout 900 python scripts/debug/bitwise_ab.py 2>&1 | tail -1
COLS=598 OUT=/tmp/new.npz VARIANT_ROOT=. timeout 900 python scripts/debug/bitwise_ab.py 2>&1 | tail -1
python - <<'PY'
import numpy as np
a, b = np.load('/tmp/base.npz'), np.load('/tmp/new.npz')
for k in ('enh', 'alb', 'st'):
    x, y = a[k], b[k]
    print(k, 'bitwise identical' if x.tobytes() == y.tobytes() else 'DIFFERENT: max|d| %g' % np.nanmax(np.abs(x.astype(np.float64) - y)))
PY
for r in 1 2; do
for v in 0 1; do
  SMF_K2W_TILED=$v VARIANT=tiled$v VARIANT_ROOT=. timeout 600 python scripts/debug/stress_time.py 2>&1 | tail -1
done; done | tee $O/stress_time.txt
for v in 0 1; do
  SMF_K2W_TILED=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k2w_update|k2w_init" -s 2 -c 4 python scripts/debug/one_retrieve.py stress 2>&1 | grep -E 'k2w_|gpu__time|dram__bytes' | tail -16 | sed "s/^/tiled=$v /"
done | tee $O/update_ncu.txt
B="python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --config stress"
for r in 1 2 3 4; do
  for v in 0 1; do
    env SMF_K2W_TILED=$v timeout 600 $B > $O/ab_${v}_$r.log 2>&1
    python -c "import json; d=json.loads(open('$O/ab_${v}_$r.log').read().strip().splitlines()[-1]); print('SMF_K2W_TILED=$v', round(d['ms_per_step'],3), 'ms', d['clocks']['sm_mhz'])"
  done
done | tee $O/tiled_ab.txt
