"""Where decode_hdr_batch's time goes (host sections around the C call): python tools/decode_prof.py [NIMG]"""
import ctypes, json, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2309_11072_b200 as P
from paper_2309_11072_b200 import _native, decode as D

nimg = int(sys.argv[1]) if len(sys.argv) > 1 else 64
pix = bench.generate(1, list(range(nimg)))
h, w = pix[0].shape[:2]
streams = [P.deserialize(b) if isinstance(b, (bytes, bytearray)) else b
           for b in P.encode_batch([P.RadianceImage(w, h, p, []) for p in pix])]
dev = torch.device("cuda", 0)
for rep in range(2):
    t0 = time.perf_counter()
    jobs = [D._Job(st, False) for st in streams]
    t1 = time.perf_counter()
    outs = [torch.empty(j.h * j.w * 4, dtype=torch.uint8, device=dev) for j in jobs]
    arr = (_native.DecodeImage * len(jobs))(*[j.struct() for j in jobs])
    ptrs = (ctypes.c_void_p * len(jobs))(*[o.data_ptr() for o in outs])
    status = np.zeros(len(jobs), np.uint32)
    ctx = _native.context(0)
    t2 = time.perf_counter()
    _native.check(_native.lib().hdll_b200_decode_batch(ctx.handle, arr, len(jobs), ptrs,
                                                       status.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                                       torch.cuda.current_stream(dev).cuda_stream), "decode")
    t3 = time.perf_counter()
    res = [o.cpu().numpy() for o in outs]
    t4 = time.perf_counter()
    print(json.dumps({"jobs_ms": round((t1 - t0) * 1e3, 1), "structs_ms": round((t2 - t1) * 1e3, 1),
                      "c_call_ms": round((t3 - t2) * 1e3, 1), "d2h_ms": round((t4 - t3) * 1e3, 1)}), flush=True)
