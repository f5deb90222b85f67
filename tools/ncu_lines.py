"""Aggregate an `ncu --page source --print-source cuda,sass --csv` dump per CUDA source line."""
import csv, sys
from collections import defaultdict
path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = list(csv.reader(open(path)))
cur_file = None
hdr = None
agg = defaultdict(lambda: [0.0, 0.0, ''])
stall = defaultdict(lambda: defaultdict(float))
last_line = None
for r in rows:
    if not r: continue
    if r[0] == 'File Path':
        cur_file = r[1].split('/')[-1]; continue
    if r[0] == 'Line No':
        hdr = r; continue
    if hdr is None or len(r) < 8: continue
    d = dict(zip(hdr[2:], r[2:])) if len(r) == len(hdr) else None
    if r[0]:
        last_line = (cur_file, r[0], r[1])
    if d is None or not r[2].startswith('0x'):
        continue
    def f(x):
        try: return float(x)
        except: return 0.0
    key = last_line
    agg[key][0] += f(d.get('Warp Stall Sampling (All Samples)'))
    agg[key][1] += f(d.get('Instructions Executed'))
    for c in hdr:
        if c.startswith('stall_') and 'Not Issued' not in c:
            stall[key][c] += f(d.get(c))
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total samples {ts:.0f} warp-instr {ti:.3g}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    s = stall[k]; topst = sorted(s.items(), key=lambda x: -x[1])[:2]
    print(f"{v[0]/ts*100:5.1f}%s {v[1]/ti*100:5.1f}%i {k[0]}:{k[1]:>4} {k[2].strip()[:70]:70s} {[(a[6:], round(b/max(v[0],1)*100)) for a, b in topst]}")
