#!/bin/bash
# round-2 refresh (v5): bench lines for every config, the stress launch list and `--set full`
# captures of the wide kernels changed since v4 (k2w_init, k1w_quant)
mkdir -p gpurun_out/r02c gpurun_out/prof3
for c in flightline segment stress; do
  timeout 900 python bench.py --config $c > gpurun_out/r02c/bench_$c.log 2>&1; echo bench_${c}_rc=$?
  tail -1 gpurun_out/r02c/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['workload'][:40], 'ms', round(d['ms_per_step'],3), 'frac', round(r['frac'],3), 'step', round(r['step_frac'],3), d['clocks']['sm_mhz'], {k: round(v,3) for k,v in r['kernel_ms_per_step'].items()})"
done
timeout 900 python bench.py --config campaign > gpurun_out/r02c/bench_campaign.log 2>&1; echo campaign_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/prof3/launches_stress.csv python scripts/debug/one_retrieve.py stress > /dev/null 2>&1
full() {  # config regex skip tag
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" -s $3 -c 1 \
    -o /tmp/prof_$4 -f python scripts/debug/one_retrieve.py $1 > gpurun_out/prof3/$4.log 2>&1
  echo "$4 rc=$?"
  ncu -i /tmp/prof_$4.ncu-rep --page raw --csv > gpurun_out/prof3/$4.raw.csv 2>/dev/null
  ncu -i /tmp/prof_$4.ncu-rep --page details > gpurun_out/prof3/$4.details.txt 2>/dev/null
  rm -f /tmp/prof_$4.ncu-rep
}
full stress "k2w_init" 1 st_k2init
full stress "k1w_quant" 1 st_quant
