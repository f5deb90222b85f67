#!/usr/bin/env python3
"""Generate the golden parity vectors from the REAL reference encoder.

Run in the build container only (the reference does not exist on the GPU box):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to a scratch directory (numba writes caches next
to the sources, and /root/reference is read-only), imports `hdll` from there,
and records for every case the SHA-256 of the serialized stream and of each
per-stage trace array (container.py:224-229), plus the regression table.

Outputs (committed):
  tests/golden/inputs.npz   - RGBE inputs of the small cases (uint8)
  tests/golden/golden.json  - digests + metadata of every case

Cases that are large are regenerated from `paper_2309_11072_b200.synth`
(deterministic numpy) instead of being stored.  BLAS parity parameters are
pinned per case with threadpoolctl.
"""

from __future__ import annotations

import hashlib
import json
import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))


def sha(b) -> str:
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


def main() -> int:
    scratch = Path(tempfile.mkdtemp(prefix="hdll_ref_"))
    shutil.copytree("/root/reference/pkg", scratch / "pkg")
    sys.path.insert(0, str(scratch / "pkg" / "src"))
    from threadpoolctl import threadpool_info, threadpool_limits

    from hdll import RadianceImage, TmoParams, container, corpus
    from hdll.radiance_io import read_hdr_file

    from paper_2309_11072_b200 import synth

    blas = [(i.get("architecture"), i.get("num_threads")) for i in threadpool_info() if i["user_api"] == "blas"]
    arch = blas[0][0] if blas else "unknown"
    kernel = {"SkylakeX": 0, "Haswell": 1}.get(arch, -1)

    inputs: dict[str, np.ndarray] = {}
    cases = []

    def run(name, px, header_vars, orientation="-Y +X", blas_threads=1, store=True, source=None, **kw):
        h, w = px.shape[:2]
        img = RadianceImage(w, h, px, list(header_vars), orientation)
        trace: dict = {}
        rkw = dict(kw)
        if "tmo" in rkw:  # stored as a plain dict (JSON); the reference takes TmoParams
            rkw["tmo"] = TmoParams(**rkw["tmo"])
        with threadpool_limits(limits=blas_threads, user_api="blas"):
            try:
                stream = container.encode(img, trace=trace, **rkw)
                blob = container.serialize(stream)
                err = None
            except Exception as ex:  # error parity cases
                blob, err = None, type(ex).__name__
        rec = {"name": name, "h": h, "w": w, "kwargs": kw, "header_vars": list(map(list, header_vars)),
               "orientation": orientation, "blas_kernel": kernel, "blas_threads": blas_threads,
               "error": err}
        if source is not None:
            rec["source"] = source
        if store:
            inputs[name] = px
        if blob is not None:
            rec.update(stream_sha256=sha(blob), stream_len=len(blob),
                       sdr_sha256=sha(trace["sdr"].as_array()), s_sha256=sha(trace["s"].as_array()),
                       m_star_sha256=sha(b"".join(np.ascontiguousarray(p).tobytes() for p in trace["m_star"])),
                       residuals_sha256=sha(b"".join(np.ascontiguousarray(p).tobytes() for p in trace["residuals"])),
                       table=[[e.channel, e.exponent, e.a, e.b, e.count] for e in trace["table"].entries])
            dec = container.decode_hdr(stream)
            assert dec == img, name
        cases.append(rec)

    # 1. the reference's own golden corpus (pkg/tests/make_fixtures.py: seed 123, size 96)
    cdir = scratch / "corpus96"
    corpus.make_corpus(cdir, seed=123, size=96)
    for nm in ("gradient_00", "steps_00", "affine_00"):
        img = read_hdr_file(cdir / f"{nm}.hdr")
        for mode, kw in (("slrme", dict(slrme=True)), ("noslrme", dict(slrme=False))):
            run(f"fixture_{nm}.{mode}", img.pixels, img.header_vars, img.resolution_orientation, **kw)
    # the remaining corpus scenes at 48x48 (tests/conftest.py mini_corpus, seed 11)
    mdir = scratch / "corpus48"
    corpus.make_corpus(mdir, seed=11, size=48)
    for p in sorted(mdir.glob("*.hdr")):
        img = read_hdr_file(p)
        run(f"mini_{p.stem}", img.pixels, img.header_vars, img.resolution_orientation)
        run(f"mini_{p.stem}.q30s0", img.pixels, img.header_vars, img.resolution_orientation, quality=30, sigma=0.0)

    # 2. degenerate and ragged sizes (test_container.py:289-295 style) and modes
    rng = np.random.default_rng(20260101)
    sizes = [(1, 1), (1, 2), (2, 1), (3, 5), (7, 7), (8, 8), (9, 17), (17, 9), (1, 33), (33, 1), (5, 64), (13, 19)]
    for i, (h, w) in enumerate(sizes):
        px = rng.integers(0, 256, (h, w, 4), dtype=np.uint8)
        if i % 2:
            px[..., 3] = rng.integers(124, 134, (h, w))
        run(f"ragged_{h}x{w}", px, [("FORMAT", "32-bit_rle_rgbe")])
        run(f"ragged_{h}x{w}.s0", px, [], sigma=0.0)
    modes = [dict(), dict(slrme=False), dict(global_regression=True), dict(sigma=0.0), dict(sigma=0.333),
             dict(sigma=2.5), dict(quality=1), dict(quality=30), dict(quality=49), dict(quality=50),
             dict(quality=100), dict(sigma=0.0, global_regression=True), dict(sigma=65.535)]
    for i, kw in enumerate(modes):
        px = synth.make_config(0, 100 + i, scale=0.09)  # 46x69 config-0 generator
        run(f"mode_{i}", px, [("FORMAT", "32-bit_rle_rgbe"), ("", "# note"), ("EXPOSURE", "2.0")],
            "+X -Y" if i == 3 else "-Y +X", **kw)
    # zeros / flat / all-black / constant / non-canonical
    black = np.zeros((24, 40, 4), np.uint8)
    run("all_black", black, [])
    flat = np.zeros((40, 24, 4), np.uint8)
    flat[...] = (200, 100, 50, 130)
    run("flat", flat, [])
    run("flat.s0", flat, [], sigma=0.0)
    nz = np.zeros((20, 30, 4), np.uint8)
    nz[..., 3] = 130  # (0,0,0,130) decodes to non-zero radiance
    run("zero_mant_quads", nz, [])
    runs = np.zeros((16, 600, 4), np.uint8)  # long rows: runs of exactly 255 / 510 / mismatching ends
    runs[...] = (10, 20, 30, 120)
    runs[3, 255:] = (11, 21, 31, 121)
    runs[5, 510:] = (12, 20, 30, 120)
    runs[7, ::2] = (200, 200, 200, 140)
    run("long_runs", runs, [])
    # tone-map parameters (tonemap.py:22-37): gamma on both sides of the GPU's
    # MUFU cut-over (1 / gamma = 4), explicit white point, key, epsilon
    for i, tmo in enumerate([dict(gamma=1.0), dict(gamma=0.2, key=0.36), dict(white_point=2.5, gamma=2.4),
                             dict(gamma=0.05, epsilon=1e-4), dict(key=0.05, white_point=0.5)]):
        run(f"tmo_{i}", synth.make_config(0, 200 + i, scale=0.09), [("FORMAT", "32-bit_rle_rgbe")], tmo=tmo)
    # extreme 1 / gamma (the GPU's fp32 gamma pass stops at 1 / gamma = 32) and
    # dark quads with E in {0, 1}: their radiance is subnormal in fp32, so the
    # fp32 pass must hand them to the fp64 pow (m^g is far from 0 for small g)
    for i, tmo in enumerate([dict(gamma=0.002), dict(gamma=0.005), dict(gamma=0.03)]):
        run(f"tmo_x{i}", synth.make_config(0, 210 + i, scale=0.09), [("FORMAT", "32-bit_rle_rgbe")], tmo=tmo)
    dark = synth.make_config(0, 220, scale=0.09)
    drng = np.random.default_rng(220)
    sel = drng.random(dark.shape[:2]) < 0.15
    dark[sel, :3] = drng.integers(1, 256, (int(sel.sum()), 3), dtype=np.uint8)
    dark[sel, 3] = drng.integers(0, 2, int(sel.sum()), dtype=np.uint8)
    for i, tmo in enumerate([dict(gamma=20.0), dict(), dict(gamma=0.005), dict(gamma=100.0, key=0.5)]):
        run(f"dark_{i}", dark, [("FORMAT", "32-bit_rle_rgbe")], tmo=tmo)
    # error parity
    run("err_sigma", rng.integers(0, 256, (4, 4, 4), dtype=np.uint8), [], sigma=70.0)
    run("err_quality", rng.integers(0, 256, (4, 4, 4), dtype=np.uint8), [], quality=0)

    # 3. regions > 10,000 px: OpenBLAS thread split is a parity parameter
    for T in (1, 2, 8):
        px = synth.make_config(0, 0, scale=0.5)  # 256x384, regions up to ~20k px
        run(f"c0half_T{T}", px, [("FORMAT", "32-bit_rle_rgbe")], blas_threads=T, store=(T == 1),
            source="synth.make_config(0, 0, scale=0.5)")
    px = synth.make_config(21, 0, scale=0.125)  # 270x512 wide range, ~250 bins
    run("c2b_eighth", px, [], source="synth.make_config(21, 0, scale=0.125)")

    # 4. full-size config 0 (the PR1 oracle config), regenerated from synth
    px = synth.make_config(0, 0)
    run("c0_full", px, [("FORMAT", "32-bit_rle_rgbe")], store=False, source="synth.make_config(0, 0)")
    run("c0_full.s0", px, [("FORMAT", "32-bit_rle_rgbe")], store=False, source="synth.make_config(0, 0)",
        sigma=0.0)

    np.savez_compressed(HERE / "inputs.npz", **inputs)
    from hdll.rgbe import float_to_rgbe
    f2r = sha(float_to_rgbe(synth.config1_scene(1000, 135, 240)))  # pins synth.float_to_rgbe
    out = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/pkg (hdll 0.1.0)",
           "numpy": np.__version__, "blas": blas, "cases": cases, "float_to_rgbe_sha256": f2r}
    (HERE / "golden.json").write_text(json.dumps(out, indent=1) + "\n")
    shutil.rmtree(scratch, ignore_errors=True)
    print(f"wrote {len(cases)} cases, {len(inputs)} stored inputs")
    return 0


if __name__ == "__main__":
    sys.exit(main())
