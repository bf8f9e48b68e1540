#!/bin/bash
# session-4 re-entry check of HEAD: GPU tests, smoke, bench lines for every config, launch
# lists of both paths and `--set full` captures of the wide statistics kernels changed since
# their last capture (k1w_scan, k1w_quant, k1w_syrk_i8) plus k2w_init
mkdir -p gpurun_out/s4a
O=gpurun_out/s4a
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo tests_rc=$?; tail -2 $O/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -1 $O/smoke.log
for c in flightline segment stress; do
  timeout 900 python bench.py --config $c > $O/bench_$c.log 2>&1; echo bench_${c}_rc=$?
  tail -1 $O/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['workload'][:40], 'ms', round(d['ms_per_step'],3), 'frac', round(r['frac'],3), 'step', round(r['step_frac'],3), d['clocks']['sm_mhz'], {k: round(v,3) for k,v in r['kernel_ms_per_step'].items()})"
done
timeout 900 python bench.py --config campaign > $O/bench_campaign.log 2>&1; echo campaign_rc=$?
for c in stress flightline; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_$c.csv python scripts/debug/one_retrieve.py $c > /dev/null 2>&1
done
full() {  # config regex skip tag
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" -s $3 -c 1 \
    -o /tmp/prof_$4 -f python scripts/debug/one_retrieve.py $1 > $O/$4.log 2>&1
  echo "$4 rc=$?"
  ncu -i /tmp/prof_$4.ncu-rep --page raw --csv > $O/$4.raw.csv 2>/dev/null
  ncu -i /tmp/prof_$4.ncu-rep --page details > $O/$4.details.txt 2>/dev/null
  rm -f /tmp/prof_$4.ncu-rep
}
full stress "k1w_scan" 1 st_scan
full stress "k1w_quant" 1 st_quant
full stress "k1w_syrk_i8" 1 st_syrk
full stress "k2w_init" 1 st_k2init
