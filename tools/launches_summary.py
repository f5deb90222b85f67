import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/launches.csv')))
hdr = None; agg = defaultdict(list)
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            agg[d['Kernel Name'].split('(')[0]].append(float(d['Metric Value']))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{sum(v)/1e6/len(v):8.3f} ms/launch  {len(v):3d}x  {sum(v)/tot*100:5.1f}%  {k}")
