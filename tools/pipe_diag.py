"""Timeline of container.HostPipeline: per chunk H2D / compute / D2H intervals (ms)."""
import sys, time
sys.path.insert(0, ".")
import torch
import bench
import paper_2309_11072_b200 as P
from paper_2309_11072_b200 import container

nimg = int(sys.argv[1]) if len(sys.argv) > 1 else 64
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 8
pix = bench.generate(1, list(range(nimg)))
h, w = pix[0].shape[:2]
preps = [container.prepare(P.RadianceImage(w, h, p)) for p in pix]
h_in = [torch.from_numpy(p.pixels).pin_memory().view(-1) for p in preps]
h_out = [torch.empty(container.stream_capacity(p), dtype=torch.uint8).pin_memory() for p in preps]
pipe = container.HostPipeline(preps, chunk=chunk)
pipe.run(h_in, h_out)
torch.cuda.synchronize()
# instrument: wrap streams' work with events
evs = []
orig_encode = container.encode_device
def enc(*a, **k):
    s = torch.cuda.ExternalStream(a[5])
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s); r = orig_encode(*a, **k); e1.record(s); evs.append(("comp", e0, e1)); return r
container.encode_device = enc
t0 = time.perf_counter()
base = torch.cuda.Event(enable_timing=True); base.record()
pipe.run(h_in, h_out)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3
print(f"wall {wall:.1f} ms")
for name, e0, e1 in evs:
    print(name, f"{base.elapsed_time(e0):7.2f} -> {base.elapsed_time(e1):7.2f}")
