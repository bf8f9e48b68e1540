#!/bin/bash
# k3w geometry variants (per-kernel times) + one ncu --set full capture of the streamed k2w_update
mkdir -p gpurun_out/e1
for v in t16s2 t12s3p3; do
  VARIANT=$v VARIANT_ROOT=scripts/debug/variants/$v timeout 300 python scripts/debug/stress_time.py 2>&1 | tail -1
done
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k2w_update" -s 45 -c 1 \
    -o /tmp/prof_k2wu -f python scripts/debug/one_retrieve.py stress > gpurun_out/e1/k2wu.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_k2wu.ncu-rep --page raw --csv > gpurun_out/e1/k2wu.raw.csv 2>/dev/null
ncu -i /tmp/prof_k2wu.ncu-rep --page details > gpurun_out/e1/k2wu.details.txt 2>/dev/null
ncu -i /tmp/prof_k2wu.ncu-rep --page source --csv > gpurun_out/e1/k2wu.source.csv 2>/dev/null
