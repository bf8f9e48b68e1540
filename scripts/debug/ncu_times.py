import csv,collections,sys
rows=list(csv.reader(open(sys.argv[1])))
h=None;d=collections.defaultdict(list)
for r in rows:
    if 'Kernel Name' in r: h=r; continue
    if h and len(r)==len(h):
        x=dict(zip(h,r))
        if x['Metric Name']=='gpu__time_duration.sum': d[x['Kernel Name'][:40]].append(float(x['Metric Value'].replace(',','')))
for k,v in d.items(): print(k,len(v),sum(v)/len(v))
