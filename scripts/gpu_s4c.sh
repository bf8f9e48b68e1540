#!/bin/bash
# session 4: stress A/B of the k2w_init tail split (0 off, 1 init on the second stream, 2 the
# tail's statistics there too), 5 alternations; bitwise check of mode 2 and the new SYRK epilogue
mkdir -p gpurun_out/s4c
O=gpurun_out/s4c
COLS=598 OUT=/tmp/base.npz VARIANT_ROOT=scripts/debug/variants/base timeout 900 python scripts/debug/bitwise_ab.py 2>&1 | tail -1
for m in 1 2; do
SMF_TAIL_SPLIT=$m COLS=598 OUT=/tmp/new$m.npz VARIANT_ROOT=. timeout 900 python scripts/debug/bitwise_ab.py 2>&1 | tail -1
done
python - <<'PY'
import numpy as np
a = np.load('/tmp/base.npz')
for m in (1, 2):
    b = np.load('/tmp/new%d.npz' % m)
    for k in ('enh', 'alb', 'st'):
        x, y = a[k], b[k]
        print(m, k, 'bitwise identical' if x.tobytes() == y.tobytes() else 'DIFFERENT: max|d| %g' % np.nanmax(np.abs(x.astype(np.float64) - y)))
PY
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"k1w_syrk" python scripts/debug/one_retrieve.py stress 2>&1 | grep -E 'k1w_syrk|gpu__time|inst_exec' | tail -6 > $O/syrk_times.txt 2>&1
cat $O/syrk_times.txt
B="python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --config stress"
for r in 1 2 3 4 5; do
  for v in 0 1 2; do
    env SMF_TAIL_SPLIT=$v timeout 600 $B > $O/ab_${v}_$r.log 2>&1
    python -c "import json; d=json.loads(open('$O/ab_${v}_$r.log').read().strip().splitlines()[-1]); print('SMF_TAIL_SPLIT=$v', round(d['ms_per_step'],3), 'ms', d['clocks']['sm_mhz'])"
  done
done | tee $O/tail_ab.txt
