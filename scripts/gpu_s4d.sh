#!/bin/bash
# session 4, after the tail split and the SYRK changes: GPU tests, smoke, bench lines for every
# config, the stress launch list and a `--set full` capture of k1w_syrk_i8
mkdir -p gpurun_out/s4d
O=gpurun_out/s4d
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo tests_rc=$?; tail -2 $O/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -1 $O/smoke.log
for c in flightline segment stress; do
  timeout 900 python bench.py --config $c > $O/bench_$c.log 2>&1; echo bench_${c}_rc=$?
  tail -1 $O/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['workload'][:40], 'ms', round(d['ms_per_step'],3), 'frac', round(r['frac'],3), 'step', round(r['step_frac'],3), d['clocks']['sm_mhz'], {k: round(v,3) for k,v in r['kernel_ms_per_step'].items()})"
done
timeout 900 python bench.py --config campaign > $O/bench_campaign.log 2>&1; echo campaign_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_stress.csv python scripts/debug/one_retrieve.py stress > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k1w_syrk_i8" -s 3 -c 1 \
    -o /tmp/prof_st_syrk -f python scripts/debug/one_retrieve.py stress > $O/st_syrk.log 2>&1
echo "st_syrk rc=$?"
ncu -i /tmp/prof_st_syrk.ncu-rep --page raw --csv > $O/st_syrk.raw.csv 2>/dev/null
ncu -i /tmp/prof_st_syrk.ncu-rep --page details > $O/st_syrk.details.txt 2>/dev/null
