"""Diagnostic: the e2e HostPipeline's per-chunk timeline (config 1, 64 images x repeats)."""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2309_11072_b200 as P
from paper_2309_11072_b200 import _native, container

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 64
pix = bench.generate(1, list(range(64)))
preps = [container.prepare(P.RadianceImage(p.shape[1], p.shape[0], p, [("FORMAT", "32-bit_rle_rgbe")])) for p in pix]
h_in = [torch.from_numpy(p.pixels).reshape(-1).pin_memory() for p in preps]
caps = [container.stream_capacity(p) for p in preps]
h_out = [torch.empty(min(c, 8 * p.w * p.h + (1 << 16)), dtype=torch.uint8).pin_memory() for c, p in zip(caps, preps)]
pipe = container.HostPipeline(preps, chunk=chunk, ctx=_native.context(0))
pipe.run(h_in, h_out)
pipe.run(h_in, h_out, repeats=reps)  # every buffer at its steady-state size, as in bench.py
torch.cuda.synchronize()
pipe.timeline = []
t0 = time.perf_counter()
pipe.run(h_in, h_out, repeats=reps)
wall = time.perf_counter() - t0
torch.cuda.synchronize()
tl = pipe.timeline
e0 = tl[0][2]
rows = [(w, ci, round(e0.elapsed_time(ev), 3)) for w, ci, ev in tl]
by = {}
for w, ci, t in rows:
    by.setdefault(ci, {})[w] = t
print(json.dumps({"wall_ms": round(wall * 1e3, 2), "ms_per_rep": round(wall * 1e3 / reps, 2),
                  "chunks": [dict(ci=k, **v) for k, v in sorted(by.items())]}, indent=0))
