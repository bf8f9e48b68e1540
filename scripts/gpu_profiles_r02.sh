#!/bin/bash
# ncu evidence for every kernel of the flightline and stress paths (round 2):
# launch lists (gpu__time_duration of every launch) and one `--set full` capture per kernel.
mkdir -p gpurun_out/prof
for c in flightline stress; do
  timeout 600 python scripts/debug/one_retrieve.py $c > gpurun_out/prof/plain_$c.log 2>&1 || exit 1
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/prof/launches_$c.csv python scripts/debug/one_retrieve.py $c > /dev/null 2>&1
done
# second retrieval's launches: skip the first retrieval's occurrences
full() {  # config regex skip tag
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" -s $3 -c 1 \
    -o /tmp/prof_$4 -f python scripts/debug/one_retrieve.py $1 > gpurun_out/prof/$4.log 2>&1
  echo "$4 rc=$?"
  # text summaries only (the reports exceed the 64 MiB gpurun_out limit)
  ncu -i /tmp/prof_$4.ncu-rep --page raw --csv > gpurun_out/prof/$4.raw.csv 2>/dev/null
  ncu -i /tmp/prof_$4.ncu-rep --page details > gpurun_out/prof/$4.details.txt 2>/dev/null
  ncu -i /tmp/prof_$4.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/prof/$4.src.csv.gz
  rm -f /tmp/prof_$4.ncu-rep
}
full flightline "k0_pilot" 1 fl_k0
full flightline "k1_stats" 1 fl_k1
full flightline "k2_init" 1 fl_k2init
full flightline "k2_update" 45 fl_k2update
full flightline "k3_sweep" 46 fl_k3
full stress "k1w_scan" 1 st_scan
full stress "k1w_quant" 1 st_quant
full stress "k1w_syrk" 1 st_syrk
full stress "k2w_init" 1 st_k2init
full stress "k2w_update" 45 st_k2update
full stress "k3w_sweep" 46 st_k3w
