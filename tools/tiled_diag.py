"""Diagnostic: host gap / pending device work between one-rank tiled encodes (c3)."""
import gc, os, sys, time
sys.path.insert(0, ".")
import numpy as np, torch, torch.distributed as dist
import paper_2309_11072_b200 as P
from paper_2309_11072_b200 import _native, container, tiled, synth

os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29611")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
use_nccl = "--gloo" not in sys.argv
dist.init_process_group("nccl" if use_nccl else "gloo", device_id=dev if use_nccl else None)
pix = synth.make_config(3, 0)
h, w = pix.shape[:2]
image = P.RadianceImage(w, h, pix, [("FORMAT", "32-bit_rle_rgbe")])
prep = container.prepare(image, blas_kernel="skylakex", blas_threads=1)
specs = tiled.band_plan(w, h, 1, prep.params.radius)
ex = tiled.TorchExchange(); ex.specs = specs
s = specs[0]
rows = torch.from_numpy(np.ascontiguousarray(prep.pixels[s.crow0:s.crow1])).to(dev)
ctx = _native.context(0)
stream = torch.cuda.current_stream(dev)
cap = container.stream_capacity(prep)
out = (torch.empty(cap, dtype=torch.uint8, device=dev), torch.zeros(1, dtype=torch.int64, device=dev))
if "--nogc" in sys.argv:
    gc.disable()
for i in range(6):
    t0 = time.perf_counter()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    n = tiled.encode_band(ex, prep, rows.data_ptr(), s, ctx, stream.cuda_stream, dev, out=out)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"step {i}: pre-sync {1e3*(t1-t0):.3f} ms, encode_band {1e3*(t2-t1):.3f} ms, post-sync {1e3*(t3-t2):.3f} ms, "
          f"phases {tiled.last_phase_ms}", flush=True)
dist.destroy_process_group()
