"""BASELINE configs at their stated sizes: the B200 stream equals the REAL
reference's, byte for byte (SHA-256 of the serialized stream).

The digests in tests/golden/config_golden.json were produced by the reference
itself (`hdll.container.encode` + `serialize`, tests/golden/make_config_golden.py,
OpenBLAS SKYLAKEX with 1 thread) from the same seeded synthetic inputs
(`synth.make_config`), so nothing here needs /root/reference or the oracle:

  * c1: all 64 1920x1080 images of the batch (sigma 1) and 8 at sigma 0, one
    batched device pass;
  * c2 (4096x2160, ~61 exponent bins) and c2b (254 bins), sigma 1 and 0;
  * c3 (7680x4320) plain, and tile-sharded into 2 and 4 row bands (the N-rank
    path of tiled.py, ranks as threads on this GPU);
  * c4: the whole 1024-image mixed-size stream, in batches of 64.

The reference's regression sums depend on the OpenBLAS kernel and thread count
for exponent bins above 10,000 samples, so the B200 runs
with the parameters the digests were made with (SKYLAKEX, 1 thread).
"""

from __future__ import annotations

import hashlib
import json
import os
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden" / "config_golden.json"
HV = [("FORMAT", "32-bit_rle_rgbe")]


def _cases():
    if not GOLDEN.exists():
        return {}
    out: dict = {}
    for c in json.loads(GOLDEN.read_text())["cases"]:
        out.setdefault(c["name"], []).append(c)
    return out


CASES = _cases()


def _gen(args):
    cfg, idx = args
    from paper_2309_11072_b200 import synth
    return synth.make_config(cfg, idx)


def _generate(jobs):
    workers = max(1, min(len(jobs), (os.cpu_count() or 2), 32))
    if workers == 1:
        return [_gen(j) for j in jobs]
    with ProcessPoolExecutor(workers) as ex:
        return list(ex.map(_gen, jobs))


def _sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


@pytest.fixture(scope="module")
def P():
    import paper_2309_11072_b200 as P
    from paper_2309_11072_b200 import _native
    _native.context(0)
    return P


def _check_batch(P, cases, sigma):
    """encode the cases' images in one batched device pass, compare digests"""
    pix = _generate([(c["config"], c["index"]) for c in cases])
    imgs = [P.RadianceImage(p.shape[1], p.shape[0], p, HV) for p in pix]
    blobs = P.encode_batch(imgs, sigma=sigma, blas_kernel="skylakex", blas_threads=1)
    bad = [(c["name"], c["index"]) for c, b in zip(cases, blobs)
           if len(b) != c["stream_len"] or _sha(b) != c["stream_sha256"]]
    assert not bad, f"{len(bad)} of {len(cases)} streams differ from the reference: {bad[:8]}"


@pytest.mark.skipif("c1" not in CASES, reason="config_golden.json missing")
@pytest.mark.parametrize("name,sigma", [("c1", 1.0), ("c1.s0", 0.0)])
def test_config1_batch_matches_reference(name, sigma, P):
    cases = CASES[name]
    for k in range(0, len(cases), 32):
        _check_batch(P, cases[k:k + 32], sigma)


@pytest.mark.skipif("c2" not in CASES, reason="config_golden.json missing")
@pytest.mark.parametrize("name,sigma", [("c2", 1.0), ("c2.s0", 0.0), ("c2b", 1.0), ("c2b.s0", 0.0)])
def test_config2_matches_reference(name, sigma, P):
    (case,) = CASES[name]
    pix = _gen((case["config"], case["index"]))
    img = P.RadianceImage(pix.shape[1], pix.shape[0], pix, HV)
    blob = P.serialize(P.encode(img, sigma=sigma, blas_kernel="skylakex", blas_threads=1))
    assert len(blob) == case["stream_len"]
    assert _sha(blob) == case["stream_sha256"]


@pytest.fixture(scope="module")
def c3_image(P):
    pix = _gen((3, 0))
    return P.RadianceImage(pix.shape[1], pix.shape[0], pix, HV)


@pytest.mark.skipif("c3" not in CASES, reason="config_golden.json missing")
@pytest.mark.parametrize("name,sigma", [("c3", 1.0), ("c3.s0", 0.0)])
def test_config3_matches_reference(name, sigma, P, c3_image):
    (case,) = CASES[name]
    blob = P.serialize(P.encode(c3_image, sigma=sigma, blas_kernel="skylakex", blas_threads=1))
    assert _sha(blob) == case["stream_sha256"]


@pytest.mark.skipif("c3" not in CASES, reason="config_golden.json missing")
@pytest.mark.parametrize("world,sigma,name", [(2, 1.0, "c3"), (4, 1.0, "c3"), (4, 0.0, "c3.s0")])
def test_config3_tiled_matches_reference(world, sigma, name, P, c3_image):
    from paper_2309_11072_b200 import tiled
    (case,) = CASES[name]
    blob = tiled.encode_tiled(c3_image, world, sigma=sigma, blas_kernel="skylakex", blas_threads=1,
                              return_bytes=True)
    assert _sha(blob) == case["stream_sha256"]


@pytest.mark.skipif("c4" not in CASES, reason="config_golden.json missing")
def test_config4_stream_matches_reference(P):
    cases = CASES["c4"]
    assert len(cases) == 1024
    for k in range(0, len(cases), 64):
        _check_batch(P, cases[k:k + 64], 1.0)


# The same configs against the reference run with OpenBLAS at 16 threads
# (config_golden_t16.json: the level-1 split of every bin above 10,000
# samples into 16 chunks, as numpy on a 16-thread host computes np.dot) --
# the parity model bench.py uses on the GPU box, whose host reports 16.
GOLDEN16 = GOLDEN.with_name("config_golden_t16.json")


def _cases16():
    if not GOLDEN16.exists():
        return {}
    out: dict = {}
    for c in json.loads(GOLDEN16.read_text())["cases"]:
        out.setdefault(c["name"], []).append(c)
    return out


CASES16 = _cases16()


@pytest.mark.skipif("c1" not in CASES16, reason="config_golden_t16.json missing")
def test_config1_matches_reference_16_threads(P):
    cases = CASES16["c1"]
    for k in range(0, len(cases), 32):
        chunk = cases[k:k + 32]
        pix = _generate([(c["config"], c["index"]) for c in chunk])
        imgs = [P.RadianceImage(p.shape[1], p.shape[0], p, HV) for p in pix]
        blobs = P.encode_batch(imgs, sigma=1.0, blas_kernel="skylakex", blas_threads=16)
        bad = [c["index"] for c, b in zip(chunk, blobs) if _sha(b) != c["stream_sha256"]]
        assert not bad, f"c1 images {bad[:8]} differ from the 16-thread reference"


@pytest.mark.skipif("c3" not in CASES16, reason="config_golden_t16.json missing")
@pytest.mark.parametrize("name", ["c2", "c2b", "c3"])
def test_single_images_match_reference_16_threads(name, P):
    (case,) = CASES16[name]
    pix = _gen((case["config"], case["index"]))
    img = P.RadianceImage(pix.shape[1], pix.shape[0], pix, HV)
    blob = P.serialize(P.encode(img, sigma=1.0, blas_kernel="skylakex", blas_threads=16))
    assert _sha(blob) == case["stream_sha256"]


@pytest.mark.skipif("c3" not in CASES16, reason="config_golden_t16.json missing")
def test_config3_tiled_matches_reference_16_threads(P, c3_image):
    from paper_2309_11072_b200 import tiled
    (case,) = CASES16["c3"]
    blob = tiled.encode_tiled(c3_image, 4, sigma=1.0, blas_kernel="skylakex", blas_threads=16, return_bytes=True)
    assert _sha(blob) == case["stream_sha256"]


@pytest.mark.skipif("c4" not in CASES16, reason="config_golden_t16.json missing")
def test_config4_matches_reference_16_threads(P):
    cases = CASES16["c4"]
    for k in range(0, len(cases), 64):
        chunk = cases[k:k + 64]
        pix = _generate([(c["config"], c["index"]) for c in chunk])
        imgs = [P.RadianceImage(p.shape[1], p.shape[0], p, HV) for p in pix]
        blobs = P.encode_batch(imgs, sigma=1.0, blas_kernel="skylakex", blas_threads=16)
        bad = [c["index"] for c, b in zip(chunk, blobs) if _sha(b) != c["stream_sha256"]]
        assert not bad, f"c4 images {bad[:8]} differ from the 16-thread reference"
