#!/bin/bash
# session 4: `--set full` capture of the final k2w_update (two tiles per stage)
mkdir -p gpurun_out/s4n
O=gpurun_out/s4n
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k2w_update" -s 45 -c 1 \
    -o /tmp/prof_st_k2update -f python scripts/debug/one_retrieve.py stress > $O/st_k2update.log 2>&1
echo "st_k2update rc=$?"
ncu -i /tmp/prof_st_k2update.ncu-rep --page raw --csv > $O/st_k2update.raw.csv 2>/dev/null
ncu -i /tmp/prof_st_k2update.ncu-rep --page details > $O/st_k2update.details.txt 2>/dev/null
ncu -i /tmp/prof_st_k2update.ncu-rep --page source --csv > $O/st_k2update.source.csv 2>/dev/null
ls -la $O
