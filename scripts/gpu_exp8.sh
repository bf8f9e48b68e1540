#!/bin/bash
# ncu source-level capture of k1w_quant (stress)
mkdir -p gpurun_out/e8
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k1w_quant" -s 1 -c 1 \
    -o /tmp/prof_q -f python scripts/debug/one_retrieve.py stress > gpurun_out/e8/q.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_q.ncu-rep --page source --csv --print-source sass > gpurun_out/e8/q.sass.csv 2>/dev/null
ncu -i /tmp/prof_q.ncu-rep --page details > gpurun_out/e8/q.details.txt 2>/dev/null
