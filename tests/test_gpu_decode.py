"""GPU decoder: decode_hdr / decode_sdr against the oracle's
decoder (a restatement of container.py:233-280 pinned to the reference) on
the golden streams produced by the real reference, on GPU-encoded config
images, and on corrupted streams (the reference's exceptions, in its order)."""

import hashlib

import numpy as np
import pytest

from conftest import golden_pixels, load_golden
from oracle import hdll_oracle as O

pytestmark = pytest.mark.gpu

DATA, INPUTS = load_golden()
CASES = [c for c in DATA["cases"] if not c.get("error") and c["h"] * c["w"] <= 200_000]


@pytest.fixture(scope="module")
def P():
    import paper_2309_11072_b200 as P
    return P


def _golden_stream(case):
    """The case's stream as the reference writes it (the oracle is pinned to the
    case's stream_sha256 in tests/test_oracle.py)."""
    px = golden_pixels(case, INPUTS)
    kw = dict(case["kwargs"])
    blob = O.encode(px, header_vars=[tuple(hv) for hv in case["header_vars"]], orientation=case["orientation"],
                    blas_kernel=max(case["blas_kernel"], 0), blas_threads=case["blas_threads"], **kw)
    return px, blob


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_decode_golden_streams(P, case):
    px, blob = _golden_stream(case)
    st = P.deserialize(blob)
    sdr = P.decode_sdr(st)
    assert sdr.as_array().shape == (st.height, st.width, 3)
    # the base layer decodes to the encoder's decoded SDRI S, as the reference's does
    assert hashlib.sha256(np.ascontiguousarray(sdr.as_array()).tobytes()).hexdigest() == case["s_sha256"]
    if st.sdr_only:
        with pytest.raises(P.StreamError):
            P.decode_hdr(st)
        return
    img = P.decode_hdr(st)
    assert np.array_equal(img.pixels, px)                  # lossless
    assert np.array_equal(img.pixels, O.decode_hdr(blob))  # == the reference decoder


@pytest.mark.parametrize("cfg,scale,sigma", [(0, 1.0, 1.0), (0, 1.0, 0.0), (1, 0.5, 1.0), (21, 0.25, 1.0)])
def test_roundtrip_config_images(P, cfg, scale, sigma):
    from paper_2309_11072_b200 import synth

    px = synth.make_config(cfg, 0, scale=scale)
    h, w = px.shape[:2]
    img = P.RadianceImage(w, h, px, [("FORMAT", "32-bit_rle_rgbe")])
    st = P.encode(img, sigma=sigma)
    out = P.decode_hdr(st)
    assert np.array_equal(out.pixels, px)
    assert out.header_vars == img.header_vars


def test_batch_decode(P):
    from paper_2309_11072_b200 import synth

    imgs = []
    for i, (h, w) in enumerate([(64, 96), (33, 17), (128, 200)]):
        px = synth.make_config(0, i, scale=1.0)[:h, :w].copy()
        imgs.append(P.RadianceImage(w, h, px, []))
    streams = [P.deserialize(b) if isinstance(b, (bytes, bytearray)) else b for b in P.encode_batch(imgs)]
    outs = P.decode_hdr_batch(streams)
    for im, out in zip(imgs, outs):
        assert np.array_equal(out.pixels, im.pixels)


def _stream(P):
    from paper_2309_11072_b200 import synth

    px = synth.make_config(0, 3, scale=1.0)[:48, :64].copy()
    return P.encode(P.RadianceImage(64, 48, px, []))


def test_corrupt_bits_raise(P):
    import dataclasses

    st = _stream(P)
    # flip a byte in the middle of the R residual bitstream: bits or CRC fail
    r = bytearray(st.residual_payloads[0])
    r[len(r) // 2] ^= 0x5A
    bad = dataclasses.replace(st, residual_payloads=(bytes(r),) + tuple(st.residual_payloads[1:]))
    with pytest.raises((P.ChecksumError, P.CorruptPayloadError)):
        P.decode_hdr(bad)
    # truncated base body
    b = st.base_payload
    cut = b[:9 + 8 + 10]
    cut = (len(cut) - 4).to_bytes(4, "little") + cut[4:]
    with pytest.raises((P.CorruptPayloadError, P.ChecksumError)):
        P.decode_sdr(dataclasses.replace(st, base_payload=cut))
    # frame length mismatch
    with pytest.raises(P.CorruptPayloadError):
        P.decode_hdr(dataclasses.replace(st, e_payload=st.e_payload[:-1]))


def test_crc_mismatch_raises_checksum(P):
    import dataclasses

    st = _stream(P)
    e = bytearray(st.e_payload)
    e[5] ^= 1  # CRC field
    with pytest.raises(P.ChecksumError):
        P.decode_hdr(dataclasses.replace(st, e_payload=bytes(e)))


def test_missing_table_entry_raises(P):
    import dataclasses

    st = _stream(P)
    entries = [e for e in st.regression_table.entries if e.channel != 1]
    bad = dataclasses.replace(st, regression_table=P.RegressionTable(entries))
    with pytest.raises(P.StreamError):
        P.decode_hdr(bad)


def test_sdr_only_stream(P):
    st = P.DualLayerStream(**{**_stream(P).__dict__, "e_payload": None, "residual_payloads": None,
                              "slrme": False, "regression_table": P.RegressionTable([])})
    with pytest.raises(P.StreamError):
        P.decode_hdr(st)
    assert P.decode_sdr(st).as_array().shape == (48, 64, 3)


def _outcome(fn):
    try:
        return ("ok", fn())
    except Exception as e:  # the failure itself is what is compared
        return ("fail", type(e).__name__)


@pytest.mark.parametrize("seed", [0, 1])
def test_coder_bodies_truncated_or_flipped(P, seed):
    """The coders' decode of damaged bodies fails exactly when the reference's
    does (oracle decode_plane / lossy_decode_bits restate _kernels.py:219-262,
    :327-378), and decodes to the same plane / SDRI when it does not: every
    truncation of the last 24 bytes, 24 random cuts and 48 single-byte flips of
    the base body and of the E and R bodies."""
    from paper_2309_11072_b200 import codec, synth

    rng = np.random.default_rng(seed)
    px = synth.make_config(0, 5 + seed, scale=1.0)[:40, :56].copy()
    st = P.encode(P.RadianceImage(56, 40, px, []))
    h, w = 40, 56
    pc, dc = codec.MedRicePlaneCoderB200(), codec.BlockDctCoderB200()
    bodies = [("base", st.base_payload[9:]), ("e", st.e_payload[9:]), ("r", st.residual_payloads[0][9:])]
    for kind, body in bodies:
        bits = body[8:]
        variants = [bits[:n] for n in range(max(0, len(bits) - 24), len(bits))]
        variants += [bits[: int(n)] for n in rng.integers(0, len(bits), 24)]
        for _ in range(48):
            b = bytearray(bits)
            b[int(rng.integers(0, len(b)))] ^= int(rng.integers(1, 256))
            variants.append(bytes(b))
        for v in variants:
            if kind == "base":
                got = _outcome(lambda: dc.decode(body[:8] + v, 85).as_array())
                want = _outcome(lambda: O.lossy_decode_bits(v, h, w, 85))
            else:
                got = _outcome(lambda: pc.decode(body[:8] + v))
                want = _outcome(lambda: O.decode_plane(v, h, w))
            assert got[0] == want[0], (kind, len(v), got[1] if got[0] == "fail" else "", want)
            if got[0] == "ok":
                assert np.array_equal(np.asarray(got[1]), want[1]), (kind, len(v))
