"""CPU tests of the host side: data model, serialization, argument errors,
the C-ABI library load/exports and the synthetic input generators.  No GPU."""

from __future__ import annotations

import ctypes
import hashlib
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2309_11072_b200 as P
from conftest import golden_pixels
from oracle import hdll_oracle as O
from paper_2309_11072_b200 import _native, container, synth

REPO = Path(__file__).resolve().parent.parent


def test_library_exports_every_header_symbol():
    """The C ABI library loads without a GPU and exports include/hdll_b200.h."""
    header = (REPO / "include" / "hdll_b200.h").read_text()
    declared = set(re.findall(r"\b(hdll_b200_[a-z_]+)\s*\(", header))
    assert declared == set(_native.EXPORTS)
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    for name in declared:
        assert hasattr(lib, name), name
    assert _native.lib().hdll_b200_status_string(0) == b"ok"


def test_stream_capacity_bounds_worst_case():
    cap = _native.lib().hdll_b200_stream_capacity(9, 17, 100, 50)
    # 64 bits per sample per plane and <= 544 bytes per 8x8 block per component
    assert cap >= 100 + 50 + 2 + 14 * 768 + 5 * 17 + 4 * 9 * 17 * 8 + 3 * 2 * 3 * 544


def test_deserialize_serialize_roundtrip_on_reference_streams(golden):
    data, inputs = golden
    for case in data["cases"][:20]:
        if case["error"]:
            continue
        px = golden_pixels(case, inputs)
        blob = O.encode(px, header_vars=[tuple(h) for h in case["header_vars"]], orientation=case["orientation"],
                        **case["kwargs"])
        s = P.deserialize(blob)
        assert P.serialize(s) == blob
        assert s.slrme == bool(case["kwargs"].get("slrme", True))
        assert len(s.regression_table) == len(case["table"])
        sizes = P.section_sizes(s)
        assert sum(sizes.values()) == len(blob)
        assert abs(P.bitrate_bpp(s) - len(blob) * 8 / (case["w"] * case["h"])) < 1e-12


def test_header_bytes_match_oracle():
    px = synth.make_config(0, 1, scale=0.05)
    img = P.RadianceImage(px.shape[1], px.shape[0], px, [("FORMAT", "32-bit_rle_rgbe"), ("", "# c")], "+X -Y")
    prep = container.prepare(img, quality=30, sigma=0.333)
    blob = O.encode(px, quality=30, sigma=0.333, header_vars=img.header_vars, orientation="+X -Y")
    assert blob.startswith(prep.pre)
    s = P.deserialize(blob)
    assert s.sigma_milli == 333 and s.lossy_spec.quality == 30
    assert prep.post in blob


def test_gaussian_taps_match_reference_formula():
    for sigma in (0.333, 1.0, 2.5, 65.535):
        assert np.array_equal(container.gaussian_kernel(sigma), O.gaussian_taps(sigma))
    t = container.gaussian_kernel(1.0)
    # SURVEY.md App. A.3 taps for sigma = 1
    assert t[3] == 0.3990502796524549 and t[0] == 0.004433048175243745


@pytest.mark.parametrize("kw,exc", [
    (dict(sigma=66.0), ValueError), (dict(sigma=-0.1), ValueError), (dict(quality=0), ValueError),
    (dict(quality=101), ValueError), (dict(lossless_coder=7), P.UnknownCoderError),
    (dict(lossy_coder=9), P.UnknownCoderError)])
def test_argument_errors_match_reference(kw, exc):
    img = P.RadianceImage(4, 4, np.zeros((4, 4, 4), np.uint8))
    with pytest.raises(exc):
        container._prepare(img, kw.get("quality", 85), kw.get("sigma", 1.0), True, False,
                           kw.get("lossy_coder", 1), kw.get("lossless_coder", 1), None, None, None, False)


def test_empty_image_is_stream_error():
    with pytest.raises(P.StreamError):
        container.prepare(P.RadianceImage(0, 0, np.zeros((0, 0, 4), np.uint8)))


def test_tmo_params_validation():
    with pytest.raises(ValueError):
        P.TmoParams(key=0)
    with pytest.raises(ValueError):
        P.TmoParams(epsilon=1e-2)
    with pytest.raises(ValueError):
        P.TmoParams(white_point=-1.0)


def test_regression_table_validation():
    with pytest.raises(ValueError):
        P.RegressionTable([P.RegressionEntry(0, 1, float("inf"), 0.0, 3)])
    with pytest.raises(ValueError):
        P.RegressionTable([P.RegressionEntry(0, 1, 1.0, 0.0, 3), P.RegressionEntry(0, 1, 1.0, 0.0, 3)])
    t = P.RegressionTable([P.RegressionEntry(2, 1, 1.0, 0.0, 3), P.RegressionEntry(0, 9, 1.0, 0.0, 3)])
    assert [(e.channel, e.exponent) for e in t.entries] == [(0, 9), (2, 1)]


def test_dual_layer_stream_consistency_checks():
    tab = P.RegressionTable()
    with pytest.raises(P.StreamError):
        P.DualLayerStream(1, 1, True, P.LossyCoderSpec(), P.LosslessCoderSpec(), 0, b"", tab, [], "-Y +X", b"")


def test_deserialize_rejects_corruption(golden):
    data, inputs = golden
    case = data["cases"][0]
    blob = O.encode(golden_pixels(case, inputs), header_vars=[tuple(h) for h in case["header_vars"]],
                    orientation=case["orientation"], **case["kwargs"])
    with pytest.raises(P.StreamError):
        P.deserialize(b"XXXX" + blob[4:])
    with pytest.raises(P.StreamError):
        P.deserialize(blob + b"\0")
    sdr_only = P.deserialize(blob[: len(blob) - sum(len(p) for p in P.deserialize(blob).residual_payloads)
                                  - len(P.deserialize(blob).e_payload)])
    assert sdr_only.sdr_only


def test_float_to_rgbe_matches_reference_digest():
    """synth.float_to_rgbe restates rgbe.py:16-67; the digest was produced by the
    reference's own float_to_rgbe on the same scene (tests/golden/make_golden.py)."""
    import json
    g = json.loads((REPO / "tests" / "golden" / "golden.json").read_text())
    want = g["float_to_rgbe_sha256"]
    got = hashlib.sha256(synth.float_to_rgbe(synth.config1_scene(1000, 135, 240)).tobytes()).hexdigest()
    assert got == want


def test_native_fails_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        _native.Context(0)


@pytest.mark.parametrize("nimg,chunk,repeats", [(64, 64, 10), (64, 64, 1), (64, 64, 3), (5, 2, 4), (9, 8, 7), (3, 8, 2),
                                                (1, 1, 5), (17, 4, 3)])
def test_host_pipeline_chunks_cover_the_stream_in_order(nimg, chunk, repeats):
    """HostPipeline._chunks: every image of the repeated batch exactly once, in
    order, no chunk above `chunk`, ramped (smaller) ends when the stream is long."""
    h = container.HostPipeline.__new__(container.HostPipeline)
    h.preps, h.chunk, h.order = [None] * nimg, chunk, list(range(nimg))
    chunks = h._chunks(repeats)
    flat = [i for c in chunks for i in c]
    assert flat == list(range(nimg)) * repeats
    h.order = list(reversed(range(nimg)))  # by_size: the given order, repeated
    assert [i for c in h._chunks(repeats) for i in c] == h.order * repeats
    c = min(chunk, nimg)
    assert all(1 <= len(k) <= c for k in chunks)
    if nimg * repeats >= 3 * c and c >= 4:
        assert len(chunks[0]) <= c // 4 and len(chunks[-1]) <= c // 2


def test_bench_parity_model_follows_the_host_blas():
    """bench.py encodes with this host's OpenBLAS kernel and thread count (the
    streams `hdll.encode` computes here) unless --blas-threads overrides it,
    and compares with the reference digests made at that thread count."""
    import argparse

    import bench

    hb = {"kernel": 0, "threads": 16}
    assert bench.blas_params(argparse.Namespace(blas_threads=None), hb) == (0, 16)
    assert bench.blas_params(argparse.Namespace(blas_threads=1), hb) == (0, 1)
    assert bench.blas_params(argparse.Namespace(blas_threads=None), {"kernel": None, "threads": None}) == (0, 1)
    assert bench.blas_params(argparse.Namespace(blas_threads=None), {"kernel": 1, "threads": 200}) == (1, 64)
    one = bench.golden_digests(1, 1.0, 1)
    assert len(one) == 64
    assert bench.golden_digests(1, 0.0, 16) == bench.golden_digests(1, 0.0, 1)  # sigma 0: thread-independent
    t16 = bench.golden_digests(1, 1.0, 16)
    if t16:  # tests/golden/config_golden_t16.json present
        assert len(t16) == 64
        # the 16-way split moves float32 a / b only where an fp64 sum sits near a
        # rounding boundary: config 2's streams differ, config 1's do not
        assert bench.golden_digests(2, 1.0, 16) != bench.golden_digests(2, 1.0, 1)
    assert bench.golden_digests(1, 1.0, 7) == {}  # no digests at that thread count: the oracle checks
