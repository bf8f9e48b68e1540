#!/bin/bash
# ncu source-level capture of k2w_init (stress)
mkdir -p gpurun_out/e6
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k2w_init" -s 1 -c 1 \
    -o /tmp/prof_k2wi -f python scripts/debug/one_retrieve.py stress > gpurun_out/e6/k2wi.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_k2wi.ncu-rep --page raw --csv > gpurun_out/e6/k2wi.raw.csv 2>/dev/null
ncu -i /tmp/prof_k2wi.ncu-rep --page details > gpurun_out/e6/k2wi.details.txt 2>/dev/null
ncu -i /tmp/prof_k2wi.ncu-rep --page source --csv --print-source sass > gpurun_out/e6/k2wi.sass.csv 2>/dev/null
ncu -i /tmp/prof_k2wi.ncu-rep --page source --csv --print-source cuda > gpurun_out/e6/k2wi.cuda.csv 2>/dev/null
