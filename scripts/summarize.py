"""Summarise gpurun_out/bench.log and gpurun_out/launches.csv (ncu launch list)."""
import collections
import csv
import json
import sys

d = json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
r = d['roofline']
print(f"value {d['value']/1e9:.3f} G/s  ms/step {d['ms_per_step']:.3f}  k3 frac {r['frac']:.3f}  step frac {r['step_frac']:.3f}")
print("shares", {k: round(v, 4) for k, v in r['kernel_time_share'].items()}, "clocks", d.get('clocks'))
try:
    rows = list(csv.reader(open('gpurun_out/launches.csv')))
    hdr = None
    dd = collections.defaultdict(list)
    for row in rows:
        if len(row) > 5 and row[0] == 'ID':
            hdr = row
            continue
        if hdr and len(row) == len(hdr):
            rec = dict(zip(hdr, row))
            if rec.get('Metric Name') == 'gpu__time_duration.sum':
                dd[rec['Kernel Name'][:30]].append(float(rec['Metric Value']))
    for k, v in dd.items():
        print(f"  {k:32s} n={len(v):4d} avg={sum(v)/len(v)/1e3:9.1f} us")
except FileNotFoundError:
    pass
