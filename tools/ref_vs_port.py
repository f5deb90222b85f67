"""The CPU baseline's calibration (run in the build container; needs /root/reference).

Times the real reference encoder (hdll.container.encode + serialize, from a
scratch copy of /root/reference/pkg, numba warmed up) and the oracle port
(oracle/, what bench.py's cpu_baseline and --impl reference time on the GPU
box) on the same config-1 image, one process, OpenBLAS 1 thread, and checks
their streams are equal.  Result: profiles/r02/ref_vs_port.json.

    cp -r /root/reference/pkg /tmp/refcopy/ && python tools/ref_vs_port.py
"""
import os, sys, time
os.environ["OPENBLAS_NUM_THREADS"] = "1"
sys.path.insert(0, "/tmp/refcopy/pkg/src"); sys.path.insert(0, "/root/repo")
import numpy as np
from hdll import RadianceImage, container
from oracle import hdll_oracle as O
from paper_2309_11072_b200 import synth
px = synth.make_config(1, 0)
img = RadianceImage(1920, 1080, px, [("FORMAT", "32-bit_rle_rgbe")])
container.encode(img)  # numba warm-up
O.encode(px, header_vars=[("FORMAT", "32-bit_rle_rgbe")])
import json
rows = []
for _ in range(3):
    t = time.perf_counter(); a = container.serialize(container.encode(img)); tr = time.perf_counter() - t
    t = time.perf_counter(); b = O.encode(px, header_vars=[("FORMAT", "32-bit_rle_rgbe")]); to = time.perf_counter() - t
    rows.append({"reference_s": round(tr, 3), "port_s": round(to, 3), "equal": a == b})
    print(rows[-1])
ref = min(r["reference_s"] for r in rows); port = min(r["port_s"] for r in rows)
out = {"image": "config-1 image 0 (1920x1080)", "processes": 1, "openblas_threads": 1,
       "reference_mpix_s": round(2.0736 / ref, 3), "port_mpix_s": round(2.0736 / port, 3),
       "port_over_reference": round(ref / port, 2), "streams_equal": all(r["equal"] for r in rows), "runs": rows}
json.dump(out, open("profiles/r02/ref_vs_port.json", "w"), indent=1)
print(out)
