"""Decode throughput: GPU decode_hdr of a batch of config-1 streams (device-timed)."""
import sys, time, json
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2309_11072_b200 as P
from paper_2309_11072_b200 import decode as D

nimg = int(sys.argv[1]) if len(sys.argv) > 1 else 64
pix = bench.generate(1, list(range(nimg)))
h, w = pix[0].shape[:2]
imgs = [P.RadianceImage(w, h, p, [("FORMAT", "32-bit_rle_rgbe")]) for p in pix]
streams = [P.deserialize(b) if isinstance(b, (bytes, bytearray)) else b for b in P.encode_batch(imgs)]
dev = torch.device("cuda", 0)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = D.decode_hdr_batch(streams)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    ok = all(np.array_equal(o.pixels, p) for o, p in zip(out, pix))
    print(json.dumps({"images": nimg, "ms": round(ms, 2), "mpix_s": round(nimg * w * h / ms / 1e3, 1), "lossless": ok}))
