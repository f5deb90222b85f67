"""Diagnostic: per-step device times and per-stage breakdown of the batched encode."""
import sys, time, json
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2309_11072_b200 as P
from paper_2309_11072_b200 import _native, container

nimg = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 1
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 8
import os
cache = f"/tmp/hdll_gen_{cfg}_{nimg}.npy"  # speed-up for repeated A/B runs only
if os.path.exists(cache):
    pix = list(np.load(cache))
else:
    pix = bench.generate(cfg, list(range(nimg)))
    if len({p.shape for p in pix}) == 1:
        np.save(cache, np.stack(pix))
preps = [container.prepare(P.RadianceImage(p.shape[1], p.shape[0], p, [("FORMAT", "32-bit_rle_rgbe")])) for p in pix]
dev = torch.device("cuda", 0)
d_in = [torch.from_numpy(p.pixels).to(dev) for p in preps]
caps = [container.stream_capacity(p) for p in preps]
d_out = [torch.empty(c, dtype=torch.uint8, device=dev) for c in caps]
d_len = torch.zeros(nimg, dtype=torch.int64, device=dev)
st = torch.cuda.current_stream(dev)
ctx = _native.context(0)
for s in range(steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    container.encode_device(preps, [t.data_ptr() for t in d_in], [t.data_ptr() for t in d_out], caps, d_len.data_ptr(), st.cuda_stream, 0)
    e1.record(st)
    rc = _native.lib().hdll_b200_sync(ctx.handle)
    torch.cuda.synchronize()
    print(json.dumps({"step": s, "rc": rc, "ms": round(e0.elapsed_time(e1), 3), "wall_ms": round((time.perf_counter() - t0) * 1e3, 3),
                      "stages": {k: round(v, 3) for k, v in container._stage_times(ctx).items()}}), flush=True)
