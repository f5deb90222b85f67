"""GPU parity: the B200 path (through the C ABI) against the pinned oracle.

Bar: bit-exact bytes.  Per-stage traces (container.py:224-229) are compared
first so a failure names the stage.  Sizes here are ones the CPU oracle
finishes in seconds; full BASELINE sizes are covered by size-independent
properties (round trip, batch == single) in test_gpu_configs.py and test_gpu_decode.py.
"""

from __future__ import annotations

import hashlib
import zlib

import numpy as np
import pytest

from conftest import golden_pixels, load_golden
from oracle import hdll_oracle as O

pytestmark = pytest.mark.gpu


def sha(b) -> str:
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


@pytest.fixture(scope="module")
def gpu():
    import paper_2309_11072_b200 as P
    from paper_2309_11072_b200 import _native
    _native.context(0)  # fails loudly without a device / library
    return P


def _image(P, px, header_vars=(), orientation="-Y +X"):
    h, w = px.shape[:2]
    return P.RadianceImage(w, h, np.ascontiguousarray(px, np.uint8), [tuple(hv) for hv in header_vars], orientation)


def _payloads(blob: bytes):
    s = __import__("paper_2309_11072_b200").deserialize(blob)
    return s


# ---------------------------------------------------------------------------
# plugin seams
# ---------------------------------------------------------------------------
def _planes(rng):
    grad = (np.add.outer(np.arange(24), np.arange(33)) % 256).astype(np.uint8)
    runs = np.full((6, 700), 9, np.uint8)
    runs[1, 255:] = 10
    runs[2, 510:] = 11
    runs[3, ::3] = 200
    runs[4, 300:301] = 1
    return {
        "random": rng.integers(0, 256, (24, 33), dtype=np.uint8),
        "constant": np.full((24, 33), 77, np.uint8),
        "gradient": grad,
        "adversarial": np.tile(np.array([[0, 255]], np.uint8), (24, 17))[:, :33],
        "tiny": np.array([[9]], np.uint8),
        "row": rng.integers(0, 4, (1, 97), dtype=np.uint8),
        "col": rng.integers(0, 4, (97, 1), dtype=np.uint8),
        "runs": runs,
        "wide": rng.integers(0, 3, (5, 2000), dtype=np.uint8),
        "smooth": (rng.integers(0, 8, (64, 65), dtype=np.uint8) * 16 + 64).astype(np.uint8),
        "c0_e": __import__("paper_2309_11072_b200.synth", fromlist=["x"]).make_config(0, 3, scale=0.3)[..., 3],
    }


def test_lossless_plane_coder_plugin(gpu):
    from paper_2309_11072_b200.codec import MedRicePlaneCoderB200
    rng = np.random.default_rng(7)
    coder = MedRicePlaneCoderB200()
    for name, plane in _planes(rng).items():
        body, crc = coder.encode_with_crc(plane)
        h, w = plane.shape
        ref = np.frombuffer(b"", np.uint8)
        want = bytes(np.array([w, h], "<u4").tobytes()) + O.plane_bits(plane)
        assert crc == zlib.crc32(np.ascontiguousarray(plane).tobytes()), name
        assert body == want, name


def test_lossless_plane_random_shapes(gpu):
    from paper_2309_11072_b200.codec import MedRicePlaneCoderB200
    rng = np.random.default_rng(11)
    coder = MedRicePlaneCoderB200()
    for t in range(40):
        h, w = int(rng.integers(1, 70)), int(rng.integers(1, 300))
        kind = t % 4
        if kind == 0:
            plane = rng.integers(0, 256, (h, w), dtype=np.uint8)
        elif kind == 1:
            plane = (rng.integers(0, 8, (h, w)) * 16 + 64).astype(np.uint8)
        elif kind == 2:
            plane = (rng.integers(0, 2, (h, w)) * 255).astype(np.uint8)
        else:
            plane = np.repeat(rng.integers(0, 3, (h, 1 + w // 40)), 40, axis=1)[:, :w].astype(np.uint8)
        body, _ = coder.encode_with_crc(plane)
        assert body[8:] == O.plane_bits(plane), (t, h, w, kind)


def test_lossy_coder_plugin(gpu):
    from paper_2309_11072_b200.codec import BlockDctCoderB200
    rng = np.random.default_rng(5)
    coder = BlockDctCoderB200()
    for (h, w), q in [((8, 8), 85), ((1, 1), 85), ((9, 17), 30), ((24, 40), 100), ((13, 70), 1),
                      ((64, 64), 50), ((37, 300), 85)]:
        rgb = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        if q == 50:
            rgb = np.repeat(np.repeat(rgb[::8, ::8], 8, 0), 8, 1)[:h, :w]
        sdr = gpu.SdrImage.from_array(rgb)
        body, dec, crc = coder.encode_with_crc(sdr, q)
        payload, ref_dec, _ = O.lossy_encode(rgb, q)
        assert np.array_equal(dec, ref_dec), (h, w, q)
        assert crc == zlib.crc32(ref_dec.tobytes()), (h, w, q)
        assert body == payload[9:], (h, w, q)


# ---------------------------------------------------------------------------
# golden vectors of the real reference
# ---------------------------------------------------------------------------
def _golden_cases():
    data, _ = load_golden()
    return data["cases"]


@pytest.mark.parametrize("case", _golden_cases(), ids=lambda c: c["name"])
def test_encode_matches_reference_golden(case, gpu):
    _, inputs = load_golden()
    px = golden_pixels(case, inputs)
    img = _image(gpu, px, case["header_vars"], case["orientation"])
    kw = dict(case["kwargs"])
    if "tmo" in kw:
        kw["tmo"] = gpu.TmoParams(**kw["tmo"])
    if case["error"]:
        with pytest.raises(ValueError):
            gpu.encode(img, blas_kernel=max(case["blas_kernel"], 0), blas_threads=case["blas_threads"], **kw)
        return
    tr: dict = {}
    stream = gpu.encode(img, trace=tr, blas_kernel=max(case["blas_kernel"], 0),
                        blas_threads=case["blas_threads"], **kw)
    assert sha(tr["sdr"].as_array()) == case["sdr_sha256"], "tone-map SDR"
    assert sha(tr["s"].as_array()) == case["s_sha256"], "decoded SDR S"
    got_table = [[e.channel, e.exponent, e.a, e.b, e.count] for e in stream.regression_table.entries]
    assert got_table == case["table"], "regression table"
    assert sha(b"".join(np.ascontiguousarray(p).tobytes() for p in tr["m_star"])) == case["m_star_sha256"], "M*"
    assert sha(b"".join(np.ascontiguousarray(p).tobytes() for p in tr["residuals"])) == case["residuals_sha256"]
    blob = gpu.serialize(stream)
    assert len(blob) == case["stream_len"]
    assert sha(blob) == case["stream_sha256"]


# ---------------------------------------------------------------------------
# oracle parity on config generators at oracle-friendly sizes
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("cfg,scale,sigma", [(0, 1.0, 1.0), (0, 1.0, 0.0), (1, 0.5, 1.0), (21, 0.25, 1.0),
                                             (2, 0.25, 1.0), (4, 0.5, 1.0)])
def test_config_images_match_oracle(cfg, scale, sigma, gpu):
    from paper_2309_11072_b200 import synth
    px = synth.make_config(cfg, 0, scale=scale)
    img = _image(gpu, px, [("FORMAT", "32-bit_rle_rgbe")])
    tr: dict = {}
    got = gpu.serialize(gpu.encode(img, sigma=sigma, trace=tr))
    otr: dict = {}
    want = O.encode(px, sigma=sigma, header_vars=[("FORMAT", "32-bit_rle_rgbe")], trace=otr)
    assert np.array_equal(tr["sdr"].as_array(), otr["sdr"])
    assert np.array_equal(tr["s"].as_array(), otr["s"])
    for c in range(3):
        assert np.array_equal(tr["m_star"][c], otr["m_star"][c]), c
    assert got == want


def test_blas_threads_parameter(gpu):
    """Regions > 10,000 px: the modelled OpenBLAS thread split changes bits."""
    from paper_2309_11072_b200 import synth
    px = synth.make_config(21, 1, scale=0.25)
    img = _image(gpu, px)
    for kern in (0, 1):
        for T in (1, 3, 8):
            got = gpu.serialize(gpu.encode(img, blas_kernel=kern, blas_threads=T))
            want = O.encode(px, blas_kernel=kern, blas_threads=T)
            assert got == want, (kern, T)


def test_batch_equals_single(gpu):
    from paper_2309_11072_b200 import synth
    imgs = [_image(gpu, synth.make_config(4, i, scale=0.1)) for i in range(5)]
    imgs.append(_image(gpu, synth.make_config(0, 9, scale=0.05)))
    batch = gpu.encode_batch(imgs)
    for img, blob in zip(imgs, batch):
        assert blob == gpu.serialize(gpu.encode(img))


def test_errors(gpu):
    px = np.zeros((4, 4, 4), np.uint8)
    with pytest.raises(gpu.StreamError):
        gpu.encode(gpu.RadianceImage(0, 0, np.zeros((0, 0, 4), np.uint8)))
    with pytest.raises(ValueError):
        gpu.encode(_image(gpu, px), sigma=66.0)
    with pytest.raises(ValueError):
        gpu.encode(_image(gpu, px), quality=101)
    with pytest.raises(gpu.UnknownCoderError):
        gpu.encode(_image(gpu, px), lossless_coder=99)


# ---------------------------------------------------------------------------
# wide rows: the plane coder cuts rows wider than 2048 samples into segments
# whose automaton entry state comes from a scan (runs carried across them)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("w,h,kind", [(4100, 24, "scene"), (9000, 12, "flat"), (6000, 10, "stripes"),
                                      (2049, 16, "scene"), (65536 + 8, 2, "flat"), (9000, 6, "const")])
def test_wide_rows_match_oracle(w, h, kind, gpu):
    from paper_2309_11072_b200 import synth
    rng = np.random.default_rng(w + h)
    if kind == "scene":
        px = np.tile(synth.make_config(0, 1), (1, -(-w // 768), 1))[:h, :w].copy()
    elif kind == "const":  # every segment inside one run: only the row end emits its chunks
        px = np.zeros((h, w, 4), np.uint8)
        px[...] = (140, 130, 120, 128)
        px[h // 2:] = (7, 7, 7, 100)
    elif kind == "flat":  # long constant runs crossing every segment boundary, a few breaks
        px = np.zeros((h, w, 4), np.uint8)
        px[...] = (140, 130, 120, 128)
        for y in range(h):
            for x in rng.integers(0, w, 5):
                px[y, x] = rng.integers(0, 256, 4)
    else:  # runs of random lengths around the 255-chunk and segment sizes
        px = np.zeros((h, w, 4), np.uint8)
        for y in range(h):
            x = 0
            while x < w:
                ln = int(rng.choice([1, 3, 254, 255, 256, 510, 2047, 2048, 2049, 3000]))
                px[y, x:x + ln] = rng.integers(0, 256, 4)
                x += ln
    img = _image(gpu, px, [("FORMAT", "32-bit_rle_rgbe")])
    got = gpu.serialize(gpu.encode(img))
    want = O.encode(px, header_vars=[("FORMAT", "32-bit_rle_rgbe")])
    assert got == want


# ---------------------------------------------------------------------------
# tone-map parameters: the fp32 gamma pass uses MUFU approximations up to
# 1 / gamma = 4 and the accurate fp32 functions beyond; both defer undecided
# bytes to the fp64 pow (tonemap.py:80-118)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("tmo", [dict(gamma=1.0), dict(gamma=0.2, key=0.36), dict(white_point=2.5, gamma=2.4),
                                 dict(gamma=0.05, epsilon=1e-4)])
def test_tmo_params_match_oracle(tmo, gpu):
    from paper_2309_11072_b200 import synth
    px = synth.make_config(0, 3, scale=0.25)
    img = _image(gpu, px, [("FORMAT", "32-bit_rle_rgbe")])
    got = gpu.serialize(gpu.encode(img, tmo=gpu.TmoParams(**tmo)))
    want = O.encode(px, tmo=tmo, header_vars=[("FORMAT", "32-bit_rle_rgbe")])
    assert got == want
