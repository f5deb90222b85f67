"""Throughput of the .hdr scanline coder: write_hdr / parse_hdr of config-1 images."""
import sys, time, json
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2309_11072_b200 as P
from paper_2309_11072_b200 import hdr_io

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
pix = bench.generate(1, list(range(n)))
h, w = pix[0].shape[:2]
imgs = [P.RadianceImage(w, h, p, [("FORMAT", "32-bit_rle_rgbe")]) for p in pix]
files = [hdr_io.write_hdr(im) for im in imgs]
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    files = [hdr_io.write_hdr(im) for im in imgs]
    torch.cuda.synchronize(); tw = time.perf_counter() - t0
    t0 = time.perf_counter()
    back = [hdr_io.parse_hdr(f, keep_on_device=True) for f in files]
    torch.cuda.synchronize(); tr = time.perf_counter() - t0
    ok = all(np.array_equal(b.pixels.cpu().numpy(), p) for b, p in zip(back, pix))
    print(json.dumps({"images": n, "MB": round(sum(map(len, files)) / 1e6, 1), "write_mpix_s": round(n * w * h / tw / 1e6, 1),
                      "parse_mpix_s": round(n * w * h / tr / 1e6, 1), "roundtrip": ok}))
