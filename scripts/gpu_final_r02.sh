#!/bin/bash
# round-2 bench lines (flightline, segment, stress, campaign) and ncu refresh of the kernels
# changed since profiles/r02 was captured
mkdir -p gpurun_out/final gpurun_out/prof
for c in flightline segment stress; do
  timeout 900 python bench.py --config $c > gpurun_out/final/bench_$c.log 2>&1; echo bench_${c}_rc=$?
  tail -1 gpurun_out/final/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['workload'][:40], 'ms', round(d['ms_per_step'],3), 'frac', round(r['frac'],3), 'step', round(r['step_frac'],3), d['clocks']['sm_mhz'])"
done
timeout 900 python bench.py --config campaign > gpurun_out/final/bench_campaign.log 2>&1; echo campaign_rc=$?
full() {  # config regex skip tag
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" -s $3 -c 1 \
    -o /tmp/prof_$4 -f python scripts/debug/one_retrieve.py $1 > gpurun_out/prof/$4.log 2>&1
  echo "$4 rc=$?"
  ncu -i /tmp/prof_$4.ncu-rep --page raw --csv > gpurun_out/prof/$4.raw.csv 2>/dev/null
  ncu -i /tmp/prof_$4.ncu-rep --page details > gpurun_out/prof/$4.details.txt 2>/dev/null
  rm -f /tmp/prof_$4.ncu-rep
}
full stress "k1w_quant" 1 st_quant
full stress "k2w_update" 45 st_k2update
full stress "k2w_init" 1 st_k2init
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/prof/launches_stress.csv python scripts/debug/one_retrieve.py stress > /dev/null 2>&1
