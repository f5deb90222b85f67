"""Decode timing (host stream in, host pixels out): decode_hdr and decode_sdr of
one config-1 image and decode_hdr_batch of NIMG; python tools/decode_time.py [NIMG]"""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np
import bench
import paper_2309_11072_b200 as P

nimg = int(sys.argv[1]) if len(sys.argv) > 1 else 64
pix = bench.generate(1, list(range(nimg)))
h, w = pix[0].shape[:2]
imgs = [P.RadianceImage(w, h, p, [("FORMAT", "32-bit_rle_rgbe")]) for p in pix]
streams = [P.deserialize(b) if isinstance(b, (bytes, bytearray)) else b for b in P.encode_batch(imgs)]


def timed(fn, reps=3):
    fn()
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3, r


t1, one = timed(lambda: P.decode_hdr(streams[0]))
ts, _ = timed(lambda: P.decode_sdr(streams[0]))
tb, outs = timed(lambda: P.decode_hdr_batch(streams), reps=2)
ok = np.array_equal(one.pixels, pix[0]) and all(np.array_equal(o.pixels, p) for o, p in zip(outs, pix))
print(json.dumps({"decode_hdr_one_ms": round(t1, 2), "decode_sdr_one_ms": round(ts, 2), "batch_images": nimg,
                  "batch_ms": round(tb, 2), "batch_mpix_s": round(nimg * w * h / tb / 1e3, 1), "lossless": ok}))
