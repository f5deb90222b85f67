#!/usr/bin/env python3
"""Full-size BASELINE-config digests from the REAL reference encoder.

Run in the build container only (the reference does not exist on the GPU box):

    python tests/golden/make_config_golden.py [--workers 7] [--only c1,c2,...] [--threads T]

Encodes every image of BASELINE configs 1, 2, 2b, 3 and 4 at their stated
sizes with `hdll.container.encode` (reference defaults: Q=85, sigma=1.0,
SLRME on, coders 1/1; plus sigma=0 variants) from a scratch copy of
/root/reference/pkg, one image per worker process with OpenBLAS pinned to one
thread (the thread count is a parity parameter; --threads
T pins it to T instead, for the sigma > 0 cases, into config_golden_tT.json:
a sigma = 0 fit sums integers, so its stream does not depend on T), and
records the SHA-256 and length of each serialized stream and of its regression
table.  The inputs are regenerated from `paper_2309_11072_b200.synth` (seeded
numpy), so only the digests are committed:

  tests/golden/config_golden.json

tests/test_gpu_configs.py encodes the same images on the B200 and compares.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import shutil
import sys
import tempfile
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent

# (config, index, sigma): every job of the digest file
def jobs(only=None, threads=1):
    out = []
    out += [("c1", 1, i, 1.0) for i in range(64)]
    out += [("c1.s0", 1, i, 0.0) for i in range(8)]
    out += [("c2", 2, 0, 1.0), ("c2.s0", 2, 0, 0.0), ("c2b", 21, 0, 1.0), ("c2b.s0", 21, 0, 0.0)]
    out += [("c3", 3, 0, 1.0), ("c3.s0", 3, 0, 0.0)]
    out += [("c4", 4, i, 1.0) for i in range(1024)]
    if threads > 1:
        out = [j for j in out if j[3] != 0.0]
    if only:
        out = [j for j in out if j[0] in only]
    return out


_SCRATCH = None
_THREADS = 1


def _init(scratch, threads=1):
    global _SCRATCH, _THREADS
    _SCRATCH = scratch
    _THREADS = threads
    os.environ["OPENBLAS_NUM_THREADS"] = str(threads)
    sys.path.insert(0, str(Path(scratch) / "pkg" / "src"))
    sys.path.insert(0, str(REPO))


def _run(job):
    import hashlib

    from threadpoolctl import threadpool_info, threadpool_limits

    from hdll import RadianceImage, container
    from paper_2309_11072_b200 import synth

    name, cfg, idx, sigma = job
    px = synth.make_config(cfg, idx)
    h, w = px.shape[:2]
    img = RadianceImage(w, h, px, [("FORMAT", "32-bit_rle_rgbe")])
    t = time.perf_counter()
    with threadpool_limits(limits=_THREADS, user_api="blas"):
        stream = container.encode(img, sigma=sigma)
    dt = time.perf_counter() - t
    blob = container.serialize(stream)
    tab = b"".join(f"{e.channel},{e.exponent},{e.a!r},{e.b!r},{e.count};".encode()
                   for e in stream.regression_table.entries)
    blas = [i.get("architecture") for i in threadpool_info() if i["user_api"] == "blas"]
    return {"name": name, "config": cfg, "index": idx, "sigma": sigma, "h": h, "w": w,
            "stream_sha256": hashlib.sha256(blob).hexdigest(), "stream_len": len(blob),
            "table_sha256": hashlib.sha256(tab).hexdigest(), "entries": len(stream.regression_table.entries),
            "ref_encode_s": round(dt, 3), "blas": blas[0] if blas else None}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=max(1, (os.cpu_count() or 2) - 1))
    ap.add_argument("--only", default=None, help="comma-separated job names (c1, c1.s0, c2, ...)")
    ap.add_argument("--threads", type=int, default=1, help="OpenBLAS threads of the reference (the ddot split)")
    args = ap.parse_args()
    only = set(args.only.split(",")) if args.only else None
    out_path = HERE / ("config_golden.json" if args.threads == 1 else f"config_golden_t{args.threads}.json")
    old = json.loads(out_path.read_text()) if out_path.exists() else {"cases": []}
    done = {(c["name"], c["index"]) for c in old["cases"]} if only else set()
    todo = [j for j in jobs(only, args.threads) if (j[0], j[2]) not in done]
    scratch = tempfile.mkdtemp(prefix="hdll_ref_")
    shutil.copytree("/root/reference/pkg", Path(scratch) / "pkg")
    # big images first so the pool's tail is short
    todo.sort(key=lambda j: -(1 if j[1] in (3,) else 0))
    results = list(old["cases"]) if only else []
    t0 = time.time()
    with ProcessPoolExecutor(args.workers, initializer=_init, initargs=(scratch, args.threads)) as ex:
        for k, r in enumerate(ex.map(_run, todo, chunksize=1)):
            results.append(r)
            if k % 32 == 0 or r["h"] * r["w"] > 8e6:
                print(f"[{time.time() - t0:7.1f}s] {k + 1}/{len(todo)} {r['name']}#{r['index']} "
                      f"{r['w']}x{r['h']} ref {r['ref_encode_s']}s", flush=True)
    shutil.rmtree(scratch, ignore_errors=True)
    order = {n: i for i, n in enumerate(dict.fromkeys(j[0] for j in jobs()))}
    results.sort(key=lambda r: (order.get(r["name"], 99), r["index"]))
    import numpy as np
    meta = {"generator": "tests/golden/make_config_golden.py",
            "reference": "/root/reference/pkg (hdll 0.1.0), container.encode + serialize",
            "params": "quality 85, slrme on, global_regression off, lossy 1, lossless 1, TmoParams()",
            "blas_threads": args.threads, "numpy": np.__version__,
            "inputs": "paper_2309_11072_b200.synth.make_config(config, index) (seed 1000*config + index)",
            "cases": results}
    out_path.write_text(json.dumps(meta, indent=0) + "\n")
    print(f"wrote {len(results)} digests to {out_path} in {time.time() - t0:.0f}s")
    return 0


if __name__ == "__main__":
    sys.exit(main())
