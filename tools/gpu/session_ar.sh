#!/bin/bash
# GPU session AR: e2e pipeline ramp variants (timeline tool, c1, 10 repeats)
O=gpurun_out/r2
mkdir -p $O
for r in "" "0.125,0.25,0.5,0.75" "0.125,0.25,0.4,0.6,0.8" "0.1875,0.375,0.625,0.875"; do
  for rep in 1 2; do
    HDLL_PIPE_RAMP="$r" timeout 600 python tools/pipe_timeline.py 10 64 > $O/pipe_tl_r.json 2>&1
    python - "$r" <<'PY'
import json,sys
d=json.load(open('gpurun_out/r2/pipe_tl_r.json'))
ch=d['chunks']
print(repr(sys.argv[1]), d['ms_per_rep'], 'first h2d', ch[0]['h2d_end'], 'last d2h', round(ch[-1]['d2h_end']-ch[-1]['enc_end'],2), 'gaps', [round(ch[i+1]['enc_start']-ch[i]['enc_end'],2) for i in range(len(ch)-1)])
PY
  done
done
