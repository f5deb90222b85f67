"""Diagnostic: does co-scheduling two half batches on two streams beat one batch?"""
import sys, time, json
sys.path.insert(0, ".")
import torch
import bench
import paper_2309_11072_b200 as P
from paper_2309_11072_b200 import _native, container

nimg = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 2
pix = bench.generate(1, list(range(nimg)))
h, w = pix[0].shape[:2]
preps = [container.prepare(P.RadianceImage(w, h, p, [("FORMAT", "32-bit_rle_rgbe")])) for p in pix]
dev = torch.device("cuda", 0)
d_in = [torch.from_numpy(p.pixels).to(dev) for p in preps]
caps = [container.stream_capacity(p) for p in preps]
d_out = [torch.empty(c, dtype=torch.uint8, device=dev) for c in caps]
d_len = torch.zeros(nimg, dtype=torch.int64, device=dev)
ctxs = [_native.Context(0) for _ in range(ns)]
streams = [torch.cuda.Stream(dev) for _ in range(ns)]
per = nimg // ns

def run_split():
    for k in range(ns):
        sl = slice(k * per, (k + 1) * per)
        container.encode_device(preps[sl], [t.data_ptr() for t in d_in[sl]], [t.data_ptr() for t in d_out[sl]], caps[sl],
                                d_len.data_ptr() + 8 * k * per, streams[k].cuda_stream, 0, ctx=ctxs[k])

def run_one():
    container.encode_device(preps, [t.data_ptr() for t in d_in], [t.data_ptr() for t in d_out], caps,
                            d_len.data_ptr(), streams[0].cuda_stream, 0, ctx=ctxs[0])

for name, fn in (("one", run_one), ("split", run_split), ("one", run_one), ("split", run_split)):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    print(json.dumps({"mode": name, "streams": ns if name == "split" else 1, "ms": round((time.perf_counter() - t0) / 3 * 1e3, 3)}))
