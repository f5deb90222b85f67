#!/bin/bash
# GPU session V: decode kernel durations (ncu launch list) for 4 config-1 images
O=gpurun_out/r2
mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum --clock-control none --csv --log-file $O/dec_launches_v.csv python tools/decode_time.py 4 > $O/dec_ncu_v.log 2>&1; echo "ncu rc=$?"; tail -2 $O/dec_ncu_v.log
python - <<'PY'
import csv
rows=list(csv.reader(l for l in open("gpurun_out/r2/dec_launches_v.csv") if not l.startswith("==")))
h=rows[0]; ki=h.index("Kernel Name"); mi=h.index("Metric Name"); vi=h.index("Metric Value"); ui=h.index("Metric Unit")
for r in rows[1:40]:
    print(r[ki][:50], r[mi], r[vi], r[ui])
PY
