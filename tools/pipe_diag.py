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
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
pipe.run(h_in, h_out, repeats=reps)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3
print(f"wall {wall:.1f} ms for {reps} x {nimg} images ({nimg * reps * w * h / wall / 1e3:.0f} Mpix/s)")
prev = None
busy = 0.0
for name, e0, e1 in evs:
    a, b = base.elapsed_time(e0), base.elapsed_time(e1)
    busy += b - a
    gap = "" if prev is None else f"  gap {a - prev:6.2f}"
    print(name, f"{a:7.2f} -> {b:7.2f} ({b - a:6.2f}){gap}")
    prev = b
print(f"compute busy {busy:.1f} ms of {wall:.1f}")
