import sys, time
sys.path.insert(0, ".")
import torch
import bench
import paper_2309_11072_b200 as P
from paper_2309_11072_b200 import container, _native
n = 32
pix = bench.generate(1, list(range(n)))
h, w = pix[0].shape[:2]
preps = [container.prepare(P.RadianceImage(w, h, p)) for p in pix]
dev = torch.device("cuda", 0)
d_in = [torch.from_numpy(p.pixels).to(dev) for p in preps]
caps = [container.stream_capacity(p) for p in preps]
d_out = [torch.empty(c, dtype=torch.uint8, device=dev) for c in caps]
d_len = torch.zeros(n, dtype=torch.int64, device=dev)
s = torch.cuda.Stream(dev); s2 = torch.cuda.Stream(dev)
big_h = torch.empty(300 << 20, dtype=torch.uint8).pin_memory()
big_d = torch.empty(300 << 20, dtype=torch.uint8, device=dev)
ctx = _native.context(0)
def enc():
    container.encode_device(preps, [t.data_ptr() for t in d_in], [t.data_ptr() for t in d_out], caps, d_len.data_ptr(), s.cuda_stream, 0)
for mode in ["alone", "h2d", "d2h", "alone"]:
    for rep in range(3):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        if mode == "h2d":
            with torch.cuda.stream(s2): big_d.copy_(big_h, non_blocking=True)
        if mode == "d2h":
            with torch.cuda.stream(s2): big_h.copy_(big_d, non_blocking=True)
        e0.record(s); enc(); e1.record(s)
        torch.cuda.synchronize()
    print(mode, round(e0.elapsed_time(e1), 2))
