#!/usr/bin/env python3
"""Benchmark: HDR encode Mpix/s with a bit-exact HDLL v1 stream (BASELINE.json).

Workload (default): BASELINE config 1 -- ONE batch of 64 synthetic 1920x1080
RGBE images (config-1 generator, seeds 1000 + i), reference defaults (Q=85,
sigma=1.0, SLRME on, coders 1/1), sharded over the N GPUs ("strong" scaling:
the batch is fixed, rank r encodes its LPT share of it with no data-path
collective).  One step = the encode of every local image, RGBE resident in HBM
-> serialized streams resident in HBM; the timed region is bracketed by a
barrier and a CUDA synchronize on both sides, and the max over ranks is
reported.

    python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference]
                    [--config 0|1|2|3|4|21] [--weak] [--sigma S]

--gpus N > 1 without a torchrun environment re-launches itself through
`torch.distributed.run` with N ranks (one per GPU, NCCL).  --weak gives every
rank its own --images images instead.  --config 4 is the whole 1024-image
mixed-size stream (LPT over the ranks, encoded in batches of <= --chunk-mpx
Mpx); --config 3 runs the tile-sharded single-image path when N > 1.

--impl reference times the reference algorithm's CPU implementation (the
oracle port, oracle/: C loops + numpy, bit-identical to the reference) on the
host cores, one image per worker process, on the same config.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import subprocess
import sys
import threading
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "HDR encode Mpix/s, bit-exact bitstream, % of HBM roofline"
UNIT = "Mpix/s"
GOLDEN = ROOT / "tests" / "golden" / "config_golden.json"
DEFAULT_IMAGES = {0: 64, 1: 64, 2: 1, 21: 1, 3: 1, 4: 1024}


def _gen(args):
    cfg, idx, scale = args
    from paper_2309_11072_b200 import synth
    return synth.make_config(cfg, idx, scale=scale)


def generate(cfg: int, indices, scale: float = 1.0, workers: int | None = None):
    workers = workers or min(len(indices), os.cpu_count() or 4, 32)
    if workers <= 1 or len(indices) == 1:
        return [_gen((cfg, i, scale)) for i in indices]
    with ProcessPoolExecutor(workers) as ex:
        return list(ex.map(_gen, [(cfg, i, scale) for i in indices], chunksize=4))


def _oracle_encode(args):
    px, sigma, kernel, threads = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import hdll_oracle as O
    t = time.perf_counter()
    blob = O.encode(px, sigma=sigma, header_vars=[("FORMAT", "32-bit_rle_rgbe")], blas_kernel=kernel,
                    blas_threads=threads)
    return blob, time.perf_counter() - t


def blas_params(args, hb):
    """The parity model of the reference's np.dot on this host (SURVEY.md App.
    A.5): the detected OpenBLAS kernel (SKYLAKEX when the core type is not
    modelled) and thread count, which fixes the level-1 split of large bins;
    --blas-threads overrides the count."""
    kernel = hb["kernel"] if hb["kernel"] is not None else 0
    threads = args.blas_threads if args.blas_threads else (hb["threads"] or 1)
    return kernel, max(1, min(int(threads), 64))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn(args) -> int:
    """--gpus N > 1 outside torchrun: re-launch this script with N ranks (the
    driver's own launch line), NCCL's init log left on so the ranks show."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


STAGE_KERNEL = {"tonemap": "hdll::k_tm_nodes", "base": "hdll::k_base_layer", "prefilter": "hdll::k_prefilter_cols",
                "fit": "hdll::k_sort_scatter", "estimate": "hdll::k_estimate", "crc": "hdll::k_crc_chunks",
                "entropy_dct": "hdll::k_entropy_dct", "entropy_plane": "hdll::k_entropy_plane",
                "assemble": "hdll::k_assemble"}


def pipe_util(stage):
    """The stage's main kernel's busiest execution pipe, % of that pipe's peak
    (profiles/pipe_util.json, from the committed ncu --set full capture -- not
    measured by this run)."""
    f = ROOT / "profiles" / "pipe_util.json"
    if not f.exists():
        return None
    k = STAGE_KERNEL.get(stage)
    e = json.loads(f.read_text()).get(k)
    if not e:
        return None
    return {"kernel": k, "pipe": e["pipe"], "pct_of_pipe_peak": e["pct"], "issue_active_pct": e["issue_pct"],
            "source": "profiles/pipe_util.json (ncu --set full)"}


def compute_ceilings(stage_ms: dict):
    """Each stage's time against its own measured compute ceiling
    (profiles/ceilings.json: per-launch executed-instruction counts from ncu x
    the B200 pipe rates measured by tools/peaks_fp64_alu.cu)."""
    f = ROOT / "profiles" / "ceilings.json"
    if not f.exists():
        return None
    d = json.loads(f.read_text())
    out = {}
    for stage, e in d.get("stages", {}).items():
        if stage in stage_ms and stage_ms[stage] > 0 and e.get("min_ms"):
            out[stage] = {"bound": e["bound"], "ceiling_ms_per_step": e["min_ms"], "measured_ms": round(stage_ms[stage], 4),
                          "frac": round(e["min_ms"] / stage_ms[stage], 4)}
    return {"stages": out, "source": "profiles/ceilings.json", "peaks": d.get("peaks")}


def golden_digests(config: int, sigma: float, threads: int = 1):
    """{index: (sha256, len)} of the reference's own streams with OpenBLAS at
    `threads` threads (tests/golden/config_golden.json, config_golden_tT.json;
    a sigma = 0 stream does not depend on the thread count)."""
    path = GOLDEN if threads == 1 or sigma == 0.0 else GOLDEN.with_name(f"config_golden_t{threads}.json")
    if not path.exists():
        return {}
    name = {1: "c1", 2: "c2", 21: "c2b", 3: "c3", 4: "c4"}.get(config)
    if name is None:
        return {}
    if sigma == 0.0:
        name += ".s0"
    elif sigma != 1.0:
        return {}
    return {c["index"]: (c["stream_sha256"], c["stream_len"]) for c in json.loads(path.read_text())["cases"]
            if c["name"] == name}


def shard(args, rank, world):
    """(local image indices, pixel count of every image of the job)"""
    from paper_2309_11072_b200 import dist as D, synth

    if args.weak:
        n_total = args.images * world
        indices = [rank * args.images + i for i in range(args.images)]
    else:
        n_total = args.images
        indices = None
    def scaled(h, w):
        return max(1, int(round(h * args.scale))) * max(1, int(round(w * args.scale)))
    if args.config == 4:
        sizes = [scaled(h, w) for h, w in synth.config4_sizes()[:n_total]]
    else:
        base = {0: (512, 768), 1: (1080, 1920), 2: (2160, 4096), 21: (2160, 4096), 3: (4320, 7680)}[args.config]
        sizes = [scaled(*base)] * n_total
    if indices is None:
        indices = D.local_indices(sizes, rank, world)
    return indices, sizes


def chunks_by_pixels(npx, budget, order=None):
    """consecutive image ranges (of `order`, default the job's order) of at most
    `budget` pixels (at least one image each)"""
    out, cur, acc = [], [], 0
    for i in (range(len(npx)) if order is None else order):
        n = npx[i]
        if cur and acc + n > budget:
            out.append(cur)
            cur, acc = [], 0
        cur.append(i)
        acc += n
    if cur:
        out.append(cur)
    return out


def run_b200(args):
    rank, world, local = dist_env()
    indices, all_sizes = shard(args, rank, world)
    pix = generate(args.config, indices, args.scale)  # before any CUDA work (forked workers)
    if args.dry_run:
        return run_dry(args, indices, pix)

    import torch

    import paper_2309_11072_b200 as P
    from paper_2309_11072_b200 import _native, container

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1 or os.environ.get("HDLL_BENCH_FORCE_DIST"):  # (the env: the N > 1 plumbing exercised on one GPU)
        import torch.distributed as dist
        if "MASTER_ADDR" not in os.environ:
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0", WORLD_SIZE="1")
        dist.init_process_group("nccl", device_id=dev)

    hb = container.host_blas()
    kernel, threads = blas_params(args, hb)
    nimg = len(indices)
    images = [P.RadianceImage(p.shape[1], p.shape[0], p, [("FORMAT", "32-bit_rle_rgbe")]) for p in pix]
    preps = [container.prepare(im, quality=args.quality, sigma=args.sigma, blas_kernel=kernel, blas_threads=threads)
             for im in images]
    npx_l = [p.w * p.h for p in preps]
    npx = sum(npx_l)
    order = None
    if args.batch_order == "size":  # batches of like-sized images (outputs stay in job order)
        order = sorted(range(len(npx_l)), key=lambda i: -npx_l[i])
    groups = chunks_by_pixels(npx_l, args.chunk_mpx * 1e6, order)

    # inputs resident in HBM; one output set reused by every batch of the step
    d_in = [torch.from_numpy(p.pixels).to(dev) for p in preps]
    caps = [container.stream_capacity(p) for p in preps]
    out_sz = max(sum(-(-caps[i] // 256) * 256 for i in g) for g in groups) if groups else 0
    d_out = torch.empty(max(out_sz, 256), dtype=torch.uint8, device=dev)
    pos0 = [sum(len(x) for x in groups[:k]) for k in range(len(groups))]  # the groups' slots in d_len
    g_off = []
    for g in groups:
        o, offs = 0, []
        for i in g:
            offs.append(o)
            o += -(-caps[i] // 256) * 256
        g_off.append(offs)
    d_len = torch.zeros(max(nimg, 1), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    lib = _native.lib()
    ctx = _native.context(local)
    base_ptr = d_out.data_ptr()

    def run_group(k):
        g = groups[k]
        container.encode_device([preps[i] for i in g], [d_in[i].data_ptr() for i in g],
                                [base_ptr + o for o in g_off[k]], [caps[i] for i in g],
                                d_len.data_ptr() + 8 * pos0[k], stream.cuda_stream, local, ctx)

    def step():
        for k in range(len(groups)):
            run_group(k)

    # verification pass (also the first warm-up): every local stream, hashed
    digests, lens = {}, [0] * nimg
    stage_acc: dict = {}
    launches = 0
    keep = max(args.cpu_sample, 64)  # streams kept on the host: oracle check, section sizes
    for k, g in enumerate(groups):
        run_group(k)
        _native.check(lib.hdll_b200_sync(ctx.handle), "verify")
        launches += lib.hdll_b200_last_launch_count(ctx.handle)
        for st, v in container._stage_times(ctx).items():
            stage_acc[st] = stage_acc.get(st, 0.0) + v
        nl = d_len.cpu().numpy()
        for j, i in enumerate(g):
            blob = bytes(d_out[g_off[k][j]: g_off[k][j] + int(nl[pos0[k] + j])].cpu().numpy())
            digests[indices[i]] = (hashlib.sha256(blob).hexdigest(), len(blob))
            lens[i] = len(blob)
            if i < keep:
                preps[i].blob = blob
    for _ in range(args.warmup - 1):
        step()
    _native.check(lib.hdll_b200_sync(ctx.handle), "warmup")
    stage_ms = stage_acc if len(groups) > 1 else container._stage_times(ctx)

    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    _native.check(lib.hdll_b200_sync(ctx.handle), "timed steps")
    ms = ev0.elapsed_time(ev1) / args.steps
    out_bytes = int(sum(lens))

    # ---- end to end through host buffers: pinned H2D + encode + D2H of every stream,
    #      chunks pipelined so transfers overlap compute (container.HostPipeline) ----
    h_in = [torch.from_numpy(p.pixels).reshape(-1).pin_memory() for p in preps]
    h_out = [torch.empty(min(c, 8 * n + (1 << 16)), dtype=torch.uint8).pin_memory() for c, n in zip(caps, npx_l)]
    chunk = args.chunk if args.config != 4 else min(args.chunk, 32)
    pipe = container.HostPipeline(preps, device=local, chunk=chunk, ctx=ctx,  # the device leg's arena
                                  by_size=args.batch_order == "size")
    pipe.run(h_in, h_out)  # warm-up (allocations)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    e2e_lens = pipe.run(h_in, h_out, repeats=args.steps)  # the steps stream back to back
    e2e_ms = (time.perf_counter() - t0) * 1000.0 / args.steps
    h2d_bytes = sum(p.pixels.nbytes for p in preps)
    e2e_ok = all(hashlib.sha256(bytes(h_out[i][: e2e_lens[i]].numpy())).hexdigest() == digests[indices[i]][0]
                 for i in range(nimg))

    # ---- max over ranks, totals, every rank's digests ----
    vals = torch.tensor([ms, e2e_ms], dtype=torch.float64, device=dev)
    all_digests = digests
    e2e_all = e2e_ok
    if dist:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
        tot = torch.tensor([float(npx), float(out_bytes), float(h2d_bytes), float(launches)], dtype=torch.float64,
                           device=dev)
        dist.all_reduce(tot)
        total_px, total_out, total_h2d = float(tot[0]), float(tot[1]), float(tot[2])
        parts = [None] * world
        dist.all_gather_object(parts, (digests, e2e_ok))
        all_digests = {}
        for d, _ in parts:
            all_digests.update(d)
        e2e_all = all(ok for _, ok in parts)
    else:
        total_px, total_out, total_h2d = float(npx), float(out_bytes), float(h2d_bytes)
    ms, e2e_ms = float(vals[0]), float(vals[1])

    # ---- parity: reference digests (SKYLAKEX, this thread count) and the oracle on this host ----
    ref = golden_digests(args.config, args.sigma, threads) if args.scale == 1.0 else {}
    par_ref = None
    if ref and kernel != 0:
        par_ref = {"checked": 0, "note": "the reference digests were made with OpenBLAS SKYLAKEX; this host's "
                                         "kernel differs, parity is checked against the oracle's model of it"}
    if ref and kernel == 0:
        common = [i for i in all_digests if i in ref]
        par_ref = {"checked": len(common), "equal": sum(all_digests[i] == ref[i] for i in common),
                   "of_job": len(all_digests),
                   "source": "tests/golden/config_golden.json (the reference's own streams, "
                             "tests/golden/make_config_golden.py)"}
    cpu = None
    par_oracle = None
    if rank == 0 and not args.no_cpu:
        sample = min(args.cpu_sample, nimg)
        cores = min(sample, os.cpu_count() or 1)
        t0 = time.perf_counter()
        with ProcessPoolExecutor(cores) as ex:
            res = list(ex.map(_oracle_encode, [(p.pixels, args.sigma, kernel, threads) for p in preps[:sample]]))
        wall = time.perf_counter() - t0
        cpu = {"value": sum(npx_l[:sample]) / wall / 1e6, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{sample} of the job's config-{args.config} images, one per process (oracle/ C+numpy "
                         f"port, bit-identical to the reference), wall {wall:.1f}s on {cores} worker processes"}
        par_oracle = {"checked": sample, "equal": sum(preps[i].blob == res[i][0] for i in range(sample)),
                      "blas_kernel": kernel, "blas_threads": threads}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    dec = None if args.no_decode else decode_timing(args, P, preps, npx_l)
    value = total_px / (ms / 1000.0) / 1e6
    e2e_value = total_px / (e2e_ms / 1000.0) / 1e6
    peak, peak_src = peaks()
    alg_bytes = 4.0 * total_px + total_out  # 4 B/px RGBE read + stream bytes written
    achieved = alg_bytes / world / (ms / 1000.0) / 1e9
    dom = max(stage_ms, key=stage_ms.get)
    secs = {"base": 0, "e": 0, "res": 0}
    kept = [i for i in range(nimg) if getattr(preps[i], "blob", None) is not None]
    for i in kept:  # section sizes of the kept local streams, scaled to the rank's images
        sz = P.section_sizes(P.deserialize(preps[i].blob))
        secs["base"] += sz["base"]
        secs["e"] += sz["exponent"]
        secs["res"] += sz["residual_r"] + sz["residual_g"] + sz["residual_b"]
    sampled_px = sum(npx_l[i] for i in kept)
    scale_sec = npx / sampled_px if sampled_px else 0.0
    stage_alg = {  # compulsory bytes of the stage's function over the rank's images
        "tonemap": 12.0 * npx, "base": 13.0 * npx, "prefilter": 27.0 * npx, "fit": 28.0 * npx,
        "estimate": 32.0 * npx, "crc": 7.0 * npx, "entropy_dct": 6.0 * npx + secs["base"] * scale_sec,
        "entropy_plane": 4.0 * npx + (secs["e"] + secs["res"]) * scale_sec, "assemble": 2.0 * out_bytes,
    }
    dom_achieved = stage_alg[dom] / (stage_ms[dom] / 1000.0) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "traffic_per_px.json"
    if tfile.exists():
        t = json.loads(tfile.read_text()).get(dom)
        traffic = round(t * npx) if t else None
    sizes_desc = (f"{len(all_sizes)} x {preps[0].w}x{preps[0].h}" if len(set(all_sizes)) == 1
                  else f"{len(all_sizes)} mixed-size images ({sum(all_sizes) / 1e6:.1f} Mpx)")
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: BASELINE config-{args.config} generator (paper datasets unavailable), "
                f"seeds 1000*config+i",
        "config": {"workload": (f"c{args.config}: {sizes_desc} RGBE, "
                                + (f"{args.images} images per GPU" if args.weak else f"one job sharded over {world} GPU(s)")),
                   "images_total": len(all_sizes), "images_rank0": nimg, "quality": args.quality,
                   "sigma": args.sigma, "slrme": True,
                   "sharding": "LPT on pixel count (dist.lpt_assign), no data-path collective"
                   if not args.weak else "contiguous image ranges per rank",
                   "batches_per_step_rank0": len(groups),
                   "batch_order": "like-sized images per batch (outputs in job order)"
                   if args.batch_order == "size" else "job order",
                   "l2": "inputs (%.0f MB/GPU) exceed the 126 MB L2" % (h2d_bytes / 1e6),
                   "host_blas": hb, "blas_model": {"kernel": ["skylakex", "haswell"][kernel], "threads": threads}},
        "roofline": {"bound": "hbm", "achieved": round(dom_achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(dom_achieved / peak, 5), "traffic": traffic, "peak_source": peak_src,
                     "kernel": f"stage {dom} (k_entropy_plane + fix-up)" if dom == "entropy_plane" else f"stage {dom}",
                     "alg_bytes_per_launch": round(stage_alg[dom] / len(groups)),
                     "launch_ms": round(stage_ms[dom] / len(groups), 4),
                     "note": "integer/latency bound, not HBM bound (DESIGN.md section 4)",
                     "busiest_pipe": pipe_util(dom)},
        "pipeline_roofline": {"achieved": round(achieved, 2), "unit": "GB/s", "frac": round(achieved / peak, 5),
                              "scope": "whole encode step (SURVEY 8d: 4 B/px RGBE + stream bytes)",
                              "bytes_per_px": round(alg_bytes / total_px, 3)},
        "compute_ceilings": compute_ceilings({k: v for k, v in stage_ms.items()}),
        "stage_ms": {k: round(v, 4) for k, v in stage_ms.items()},
        "dominant_stage": dom,
        "e2e": {"value": round(e2e_value, 3), "unit": UNIT, "h2d_bytes_per_step": int(total_h2d),
                "d2h_bytes_per_step": int(total_out) + 8 * len(all_sizes), "chunk_images": chunk,
                "path": "container.HostPipeline: pinned H2D, encode, D2H of each stream; chunks (and consecutive "
                        "steps) overlapped",
                "streams_equal_device_run": e2e_all},
        "gpu_launches": int(launches) * args.steps,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "parity_vs_reference": par_ref,
        "parity_vs_oracle": par_oracle,
        "decode": dec,
    }
    if args.digests:
        line["stream_sha256"] = [all_digests[i][0] for i in sorted(all_digests)]
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def decode_timing(args, P, preps, npx_l):
    """GPU decode_hdr / decode_sdr through the public
    API (host stream in, host pixels out), one image and a batch of the kept
    streams, checked lossless; beside it the oracle's decoder on one image on
    a host core.  The adaptive-Rice streams decode one GPU thread per stream
    (DESIGN.md section 6), so batches are where the GPU decoder is fast."""
    kept = [i for i in range(len(preps)) if getattr(preps[i], "blob", None) is not None][:64]
    if not kept:
        return None
    streams = [P.deserialize(preps[i].blob) for i in kept]
    px = sum(npx_l[i] for i in kept)

    def timed(fn, reps=2):
        fn()
        best = 1e30
        for _ in range(reps):
            t0 = time.perf_counter()
            r = fn()
            best = min(best, time.perf_counter() - t0)
        return best, r

    t1, img = timed(lambda: P.decode_hdr(streams[0]))
    tb, imgs = timed(lambda: P.decode_hdr_batch(streams), reps=1)
    ts1, _ = timed(lambda: P.decode_sdr(streams[0]))
    ok = np.array_equal(img.pixels, preps[kept[0]].pixels) and all(
        np.array_equal(o.pixels, preps[i].pixels) for o, i in zip(imgs, kept))
    out = {"unit": UNIT, "lossless_roundtrip": ok,
           "decode_hdr_one_image": {"ms": round(t1 * 1e3, 2), "value": round(npx_l[kept[0]] / t1 / 1e6, 3)},
           "decode_hdr_batch": {"images": len(kept), "ms": round(tb * 1e3, 2), "value": round(px / tb / 1e6, 3)},
           "decode_sdr_one_image": {"ms": round(ts1 * 1e3, 2), "value": round(npx_l[kept[0]] / ts1 / 1e6, 3)},
           "path": "paper_2309_11072_b200.decode_hdr / decode_hdr_batch / decode_sdr (host stream -> host pixels)"}
    if not args.no_cpu:
        from oracle import hdll_oracle as O
        t0 = time.perf_counter()
        O.decode_hdr(preps[kept[0]].blob)
        tc = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": round(npx_l[kept[0]] / tc / 1e6, 3), "unit": UNIT, "cores": 1, "kind": "port",
                               "sample": "one image, oracle decode_hdr (oracle/ port of container.py:238-280)",
                               "ms": round(tc * 1e3, 1)}
    return out


def run_dry(args, indices, pix):
    """Plumbing check without a GPU (tests/test_bench_spawn.py): the ranks
    shard the job exactly as a GPU run does, 'encode' each image as the SHA-256
    of its RGBE bytes, and rank 0 gathers the per-image digests over gloo.  It
    times nothing and prints value null."""
    import torch.distributed as dist

    rank, world, _ = dist_env()
    local = {i: hashlib.sha256(np.ascontiguousarray(p).tobytes()).hexdigest() for i, p in zip(indices, pix)}
    merged = local
    if world > 1:
        dist.init_process_group("gloo")
        parts = [None] * world
        dist.all_gather_object(parts, local)
        merged = {}
        for p in parts:
            assert not set(p) & set(merged), "an image was assigned to two ranks"
            merged.update(p)
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "value": None, "n_gpus": world,
                          "scaling": "weak" if args.weak else "strong", "images_total": len(merged),
                          "per_rank": None, "stream_sha256": [merged[i] for i in sorted(merged)]}), flush=True)


def run_tiled(args):
    """Config 3: one 7680x4320 image, tile-sharded over the ranks.

    Each rank codes a band of rows (paper_2309_11072_b200.tiled, NCCL exchanges
    between the phases); rank 0 assembles the stream.  "strong" scaling: the
    total work is one image whatever N.  Timed: CUDA events on each rank's
    stream around the whole band encode (its phases synchronize with the host
    exchanges), max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2309_11072_b200 as P
    from paper_2309_11072_b200 import _native, container, tiled

    rank, world, local = dist_env()
    pix = generate(3, [0], args.scale)[0]
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or not dist.is_initialized():
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(_free_port()))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)
    h, w = pix.shape[:2]
    image = P.RadianceImage(w, h, pix, [("FORMAT", "32-bit_rle_rgbe")])
    kernel, threads = blas_params(args, container.host_blas())
    prep = container.prepare(image, quality=args.quality, sigma=args.sigma, blas_kernel=kernel, blas_threads=threads)
    radius = prep.params.radius if prep.sigma_milli else 0
    specs = tiled.band_plan(w, h, world, radius)
    ex = tiled.TorchExchange()
    ex.specs = specs
    s = specs[rank]
    rows_h = torch.from_numpy(np.ascontiguousarray(prep.pixels[s.crow0: s.crow1])).pin_memory()
    rows = rows_h.to(dev)
    ctx = _native.context(local)
    stream = torch.cuda.current_stream(dev)
    cap = container.stream_capacity(prep)
    out = (torch.empty(cap, dtype=torch.uint8, device=dev), torch.zeros(1, dtype=torch.int64, device=dev))

    def step():
        return tiled.encode_band(ex, prep, rows.data_ptr(), s, ctx, stream.cuda_stream, dev, out=out)

    for _ in range(args.warmup):
        n_out = step()
    launches = _native.lib().hdll_b200_last_launch_count(ctx.handle)
    dist.barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            n_out = step()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    # end to end: pinned H2D of the band's rows, encode, D2H of the stream on rank 0
    h_out = torch.empty(cap, dtype=torch.uint8).pin_memory()
    dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        rows.copy_(rows_h, non_blocking=True)
        n_e = step()
        if rank == 0:
            h_out[:n_e].copy_(out[0][:n_e])
    torch.cuda.synchronize(dev)
    e2e_ms = (time.perf_counter() - t0) * 1000.0 / args.steps
    vals = torch.tensor([ms, e2e_ms], dtype=torch.float64, device=dev)
    dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms, e2e_ms = float(vals[0]), float(vals[1])
    if rank != 0:
        dist.destroy_process_group()
        return
    npx = w * h
    blob = bytes(out[0][:n_out].cpu().numpy())
    ref = golden_digests(3, args.sigma, threads) if args.scale == 1.0 and kernel == 0 else {}
    par_ref = None
    if ref:
        par_ref = {"checked": 1, "equal": int((hashlib.sha256(blob).hexdigest(), len(blob)) == ref[0]),
                   "source": "tests/golden/config_golden.json"}
    cpu = None if args.no_cpu else tiled_cpu_sample(args)
    peak, peak_src = peaks()
    alg = 4.0 * npx + n_out
    achieved = alg / world / (ms / 1000.0) / 1e9
    line = {
        "metric": METRIC, "value": round(npx / (ms / 1000.0) / 1e6, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: BASELINE config-3 generator (config-0 scene at 7680x4320), seed 3000",
        "config": {"workload": f"c3: 1 x {w}x{h} RGBE image, tile-sharded over {world} ranks (row bands)",
                   "width": w, "height": h, "quality": args.quality, "sigma": args.sigma,
                   "bands": [[b.row0, b.row1] for b in specs],
                   "l2": "input %.0f MB exceeds the 126 MB L2" % (4 * npx / 1e6)},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 5), "traffic": None, "peak_source": peak_src,
                     "kernel": "whole tiled encode (SURVEY 8d: 4 B/px RGBE + stream bytes)"},
        "e2e": {"value": round(npx / (e2e_ms / 1000.0) / 1e6, 3), "unit": UNIT,
                "h2d_bytes_per_step": int(4 * npx), "d2h_bytes_per_step": int(n_out),
                "path": "each rank: pinned H2D of its band rows; rank 0: D2H of the stream"},
        "gpu_launches": launches * args.steps,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "parity_vs_reference": par_ref,
        "phase_ms_rank0": dict(tiled.last_phase_ms),
    }
    print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def tiled_cpu_sample(args):
    """Oracle port on a 1920x1080 render of the config-3 scene (bounded sample)."""
    px = generate(3, [0], 0.25)[0]
    t0 = time.perf_counter()
    _oracle_encode((px, args.sigma, 0, 1))
    wall = time.perf_counter() - t0
    return {"value": px.shape[0] * px.shape[1] / wall / 1e6, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"config-3 scene at scale 0.25 ({px.shape[1]}x{px.shape[0]}), one process, wall {wall:.1f}s"}


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    sample = max(1, min(cores, args.images))
    pix = generate(args.config, list(range(sample)), args.scale)
    from paper_2309_11072_b200.container import host_blas
    hb = host_blas()
    kernel, threads = blas_params(args, hb)
    shapes = {p.shape[:2] for p in pix}
    with ProcessPoolExecutor(sample) as ex:
        list(ex.map(_oracle_encode, [(pix[0], args.sigma, kernel, threads)]))  # warm the workers
        for _ in range(args.warmup):
            list(ex.map(_oracle_encode, [(p, args.sigma, kernel, threads) for p in pix]))
        t0 = time.perf_counter()
        for _ in range(args.steps):
            list(ex.map(_oracle_encode, [(p, args.sigma, kernel, threads) for p in pix]))
        wall = (time.perf_counter() - t0) / args.steps
    value = sum(p.shape[0] * p.shape[1] for p in pix) / wall / 1e6
    desc = (f"{sample} x {pix[0].shape[1]}x{pix[0].shape[0]}" if len(shapes) == 1
            else f"{sample} mixed-size images")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(wall * 1000, 2), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: BASELINE config-{args.config} generator, seeds 1000*config+i",
        "config": {"workload": f"c{args.config}: {desc} RGBE images per step, one per host core "
                               "(bounded sample of the job)",
                   "images_per_step": sample, "quality": args.quality, "sigma": args.sigma, "host_blas": hb},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": sample, "kind": "port",
                         "sample": f"{sample} images per step, one per process (oracle/ port of the reference)"},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--images", type=int, default=None,
                    help="images in the job (default 64 for c0/c1, 1024 for c4, 1 for c2/c3); per rank with --weak")
    ap.add_argument("--weak", action="store_true", help="every rank encodes its own --images images")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--quality", type=int, default=85)
    ap.add_argument("--sigma", type=float, default=1.0)
    ap.add_argument("--cpu-sample", type=int, default=16)
    ap.add_argument("--chunk", type=int, default=64, help="images per HostPipeline chunk (e2e leg)")
    ap.add_argument("--blas-threads", type=int, default=None,
                    help="OpenBLAS thread count of the parity model (default: this host's, as threadpoolctl reports)")
    ap.add_argument("--chunk-mpx", type=float, default=160.0, help="Mpx per batched device encode")
    ap.add_argument("--batch-order", choices=("stream", "size"), default=None,
                    help="cut the job into batches in stream order or of like-sized images "
                         "(default: size for the mixed-size config 4, stream otherwise)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-decode", action="store_true", help="skip the decode_hdr / decode_sdr timing")
    ap.add_argument("--tiled", action="store_true", help="config 3: tile-sharded path even on one rank")
    ap.add_argument("--digests", action="store_true", help="add every stream's SHA-256 to the JSON line")
    ap.add_argument("--dry-run", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.images is None:
        args.images = DEFAULT_IMAGES.get(args.config, 1)
    if args.batch_order is None:
        args.batch_order = "size" if args.config == 4 else "stream"
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    if args.impl == "reference":
        run_reference(args)
    elif args.config == 3 and (dist_env()[1] > 1 or args.tiled):
        run_tiled(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
