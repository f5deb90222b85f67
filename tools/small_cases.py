"""Small invocations of every kernel family in one process (tools/gpu/session_sanitize.sh).  Written to run
under compute-sanitizer; the tool is closed on this GPU pool, so the session runs it plainly.

Encodes a few small images (ragged sizes, sigma 0 / 1 / 2.5, global regression, slrme off, a mixed
batch), decodes them on the GPU, runs the two coder plugins, the Radiance .hdr scanline kernels and
the tile-sharded path at 2 and 3 emulated bands, and checks every result against the oracle
(oracle/ is the checker here, as in the tests).
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2309_11072_b200 as P  # noqa: E402
from oracle import hdll_oracle as O  # noqa: E402
from paper_2309_11072_b200 import synth, tiled  # noqa: E402

HV = [("FORMAT", "32-bit_rle_rgbe")]
fails = 0


def check(name, ok):
    global fails
    print(("ok   " if ok else "FAIL ") + name, flush=True)
    fails += 0 if ok else 1


def image(px):
    return P.RadianceImage(px.shape[1], px.shape[0], px, HV)


def crop(px, h, w):
    return np.ascontiguousarray(px[:h, :w])


base = synth.make_config(0, 0, scale=0.25)  # 128 x 192
cases = [("c0 128x192 sigma 1", base, dict()),
         ("ragged 45x67 sigma 1", crop(base, 45, 67), dict()),
         ("ragged 9x250 sigma 2.5", crop(synth.make_config(0, 1, scale=0.5), 9, 250), dict(sigma=2.5)),
         ("sigma 0", crop(base, 64, 96), dict(sigma=0.0)),
         ("quality 20", crop(base, 40, 56), dict(quality=20)),
         ("slrme off", crop(base, 33, 47), dict(slrme=False)),
         ("1x1", crop(base, 1, 1), dict())]
streams = []
for name, px, kw in cases:
    got = P.serialize(P.encode(image(px), **kw))
    want = O.encode(px, header_vars=HV, **kw)
    check("encode " + name, got == want)
    streams.append((name, px, got))

# a mixed batch through encode_batch (default parameters for every image), then the batched and single decoders
imgs = [image(px) for _, px, _ in streams[:4]]
outs = P.encode_batch(imgs)
check("encode_batch", all(bytes(o) == O.encode(px, header_vars=HV) for o, (_, px, _) in zip(outs, streams[:4])))
dec = P.decode_hdr_batch([P.deserialize(s) for _, _, s in streams])
check("decode_hdr_batch", all(np.array_equal(d.pixels, px) for d, (_, px, _) in zip(dec, streams)))
for name, px, s in streams[:3]:
    st = P.deserialize(s)
    check("decode_hdr " + name, np.array_equal(P.decode_hdr(st).pixels, px))
    tr = {}
    O.encode(px, header_vars=HV, trace=tr, **dict(cases[[c[0] for c in cases].index(name)][2]))
    check("decode_sdr " + name, np.array_equal(P.decode_sdr(st).as_array(), np.asarray(tr["s"]).reshape(px.shape[0], px.shape[1], 3)))

# coder plugins through the registry (frames + CRC on the device)
rng = np.random.default_rng(7)
plane = (rng.integers(0, 4, (37, 53)) * 60).astype(np.uint8)
pay = P.lossless_encode(plane)
check("plane coder encode", pay == O.lossless_payload(plane))
check("plane coder decode", np.array_equal(P.lossless_decode(pay), plane))
sdr = rng.integers(0, 256, (21, 30, 3), dtype=np.uint8)
lpay = P.lossy_encode(P.SdrImage.from_array(sdr))
wpay, wdec, _ = O.lossy_encode(sdr, 85)
check("lossy coder encode", lpay == wpay)
check("lossy coder decode", np.array_equal(P.lossy_decode(lpay).as_array(), wdec))

# Radiance .hdr scanlines
for rle in (True, False):
    blob = P.write_hdr(image(base), rle=rle)
    check(f"hdr io rle={rle}", np.array_equal(P.parse_hdr(blob).pixels, base))

# tile-sharded, emulated bands on one GPU
for world, sig in ((2, 1.0), (3, 0.0)):
    got = tiled.encode_tiled(image(base), world, sigma=sig, return_bytes=True)
    check(f"tiled world {world} sigma {sig}", bytes(got) == O.encode(base, header_vars=HV, sigma=sig))

print("failures:", fails)
sys.exit(1 if fails else 0)
