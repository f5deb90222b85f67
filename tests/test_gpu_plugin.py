"""The drop-in seams on the B200, written like the reference's
own tests (pkg/tests/test_codec_core.py TestPlaneCoder / TestLossyCoder,
pkg/tests/test_container.py):

  * the coder registry and framed payloads (codec_core.py:225-331, :505-548):
    B200 coders as id 1, custom coders, CRC and corruption errors;
  * the coders' GPU decode against the oracle;
  * `encode(timings=)` carries the reference's stage keys
    (test_container.py:115-120), `decode_hdr(trace=)` rebuilds the encoder's
    M* and S (test_container.py:105-113);
  * decode_sdr == the reference's decoded S on every golden case;
  * host pipeline bytes == the device-resident batch;
  * concurrent encode() calls from several threads == serial calls.
"""

from __future__ import annotations

import hashlib
import struct
import threading
import zlib

import numpy as np
import pytest

from conftest import golden_pixels, load_golden
from oracle import hdll_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2309_11072_b200 as P
    from paper_2309_11072_b200 import _native
    _native.context(0)
    return P


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def _planes(rng):
    grad = np.add.outer(np.arange(24), np.arange(33)) % 256
    return {
        "random": rng.integers(0, 256, (24, 33), dtype=np.uint8),
        "constant": np.full((24, 33), 77, np.uint8),
        "gradient": grad.astype(np.uint8),
        "adversarial": np.tile(np.array([[0, 255]], np.uint8), (24, 17))[:, :33],
        "tiny": np.array([[9]], np.uint8),
        "runs": np.repeat(rng.integers(0, 3, (7, 12)), 60, axis=1).astype(np.uint8),
    }


# --------------------------------------------------------------------------
# lossless coder id 1 (TestPlaneCoder)
# --------------------------------------------------------------------------
def test_plane_roundtrip_all_shapes(P, rng):
    for name, plane in _planes(rng).items():
        payload = P.lossless_encode(plane)
        assert payload[9 + 8:] == O.plane_bits(plane), name  # body == the reference coder's
        out = P.lossless_decode(payload)
        assert out.dtype == np.uint8 and out.shape == plane.shape
        assert (out == plane).all(), name


def test_plane_decoder_reads_oracle_stream(P, rng):
    from paper_2309_11072_b200.codec import MedRicePlaneCoderB200
    plane = rng.integers(0, 200, (13, 19), dtype=np.uint8)
    body = struct.pack("<II", 19, 13) + O.plane_bits(plane)
    assert (MedRicePlaneCoderB200().decode(body) == plane).all()


def test_constant_plane_below_point1_bpp(P):
    plane = np.full((256, 256), 200, np.uint8)
    assert len(P.lossless_encode(plane)) * 8.0 / plane.size < 0.1


def test_plane_unknown_coder(P):
    with pytest.raises(P.UnknownCoderError):
        P.lossless_encode(np.zeros((2, 2), np.uint8), P.LosslessCoderSpec(coder_id=99))


def test_register_custom_coder(P, rng):
    class Doubler:  # stores every byte twice (test_codec_core.py:219-237)
        def encode(self, plane):
            return struct.pack("<II", plane.shape[1], plane.shape[0]) + bytes(
                b for v in plane.tobytes() for b in (v, v))

        def decode(self, body):
            w, h = struct.unpack_from("<II", body, 0)
            return np.frombuffer(body[8:], np.uint8)[::2].reshape(h, w).copy()

    P.register_lossless_coder(201, Doubler(), replace=True)
    with pytest.raises(ValueError):
        P.register_lossless_coder(201, Doubler())
    plane = rng.integers(0, 256, (4, 5), dtype=np.uint8)
    spec = P.LosslessCoderSpec(coder_id=201)
    assert (P.lossless_decode(P.lossless_encode(plane, spec), spec) == plane).all()
    assert P.payload_coder_id(P.lossless_encode(plane, spec)) == 201


def test_checksum_fault_injection(P, rng):
    plane = rng.integers(0, 256, (16, 16), dtype=np.uint8)
    payload = bytearray(P.lossless_encode(plane))
    for pos in (9, len(payload) // 2, len(payload) - 1):
        corrupt = bytearray(payload)
        corrupt[pos] ^= 0x40
        with pytest.raises((P.ChecksumError, P.CorruptPayloadError)):
            P.lossless_decode(bytes(corrupt))


def test_crc_mismatch_specifically(P, rng):
    plane = rng.integers(0, 256, (8, 8), dtype=np.uint8)
    payload = bytearray(P.lossless_encode(plane))
    payload[5] ^= 0xFF  # a CRC byte
    with pytest.raises(P.ChecksumError):
        P.lossless_decode(bytes(payload))


def test_plane_body_errors(P):
    from paper_2309_11072_b200.codec import MedRicePlaneCoderB200
    c = MedRicePlaneCoderB200()
    with pytest.raises(P.CorruptPayloadError, match="shorter than its dimensions"):
        c.decode(b"\x01\x00")
    with pytest.raises(P.CorruptPayloadError, match="zero plane dimension"):
        c.decode(struct.pack("<II", 0, 4))
    with pytest.raises(P.CorruptPayloadError, match="corrupt plane bitstream"):
        c.decode(struct.pack("<II", 64, 64) + b"\xff")  # ends long before 4096 samples


# --------------------------------------------------------------------------
# lossy coder id 1 (TestLossyCoder)
# --------------------------------------------------------------------------
def _const(P, color, size=(16, 16)):
    arr = np.zeros(size + (3,), np.uint8)
    arr[...] = color
    return P.SdrImage.from_array(arr)


def test_q100_gray_constants_exact(P):
    spec = P.LossyCoderSpec(quality=100)
    for v in range(0, 256, 17):
        img = _const(P, (v, v, v), (8, 8))
        assert P.lossy_decode(P.lossy_encode(img, spec), spec) == img


@pytest.mark.parametrize("h,w,q", [(24, 24, 85), (13, 21, 85), (1, 1, 50), (40, 72, 30), (9, 100, 1)])
def test_lossy_decode_equals_encoders_reconstruction(P, rng, h, w, q):
    rgb = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    spec = P.LossyCoderSpec(quality=q)
    payload = P.lossy_encode(P.SdrImage.from_array(rgb), spec)
    ref_payload, ref_dec, _ = O.lossy_encode(rgb, q)
    assert payload == ref_payload
    out = P.lossy_decode(payload, spec)
    assert (out.width, out.height) == (w, h)
    assert np.array_equal(out.as_array(), ref_dec)
    assert P.lossy_decode(payload, spec) == out  # deterministic


def test_lossy_corrupt_payload_detected(P, rng):
    img = P.SdrImage.from_array(rng.integers(0, 256, (16, 16, 3), dtype=np.uint8))
    payload = bytearray(P.lossy_encode(img))
    payload[len(payload) // 2] ^= 0x10
    with pytest.raises((P.ChecksumError, P.CorruptPayloadError)):
        P.lossy_decode(bytes(payload))
    payload = bytearray(P.lossy_encode(img))
    payload[6] ^= 0x01  # a CRC byte
    with pytest.raises(P.ChecksumError):
        P.lossy_decode(bytes(payload))


def test_lossy_unknown_coder(P):
    with pytest.raises(P.UnknownCoderError):
        P.lossy_encode(_const(P, (1, 2, 3)), P.LossyCoderSpec(coder_id=42))


def test_lossy_decode_returns_given_sdr_type(P, rng):
    from paper_2309_11072_b200.codec import BlockDctCoderB200

    class MySdr(P.SdrImage):
        pass

    rgb = rng.integers(0, 256, (8, 16, 3), dtype=np.uint8)
    c = BlockDctCoderB200(sdr_type=MySdr)
    body, raw = c.encode(P.SdrImage.from_array(rgb), 85)
    out = c.decode(body, 85)
    assert isinstance(out, MySdr) and out.as_array().tobytes() == raw


# --------------------------------------------------------------------------
# encode / decode hooks (test_container.py)
# --------------------------------------------------------------------------
def _gradient_image(P, size=24):
    from paper_2309_11072_b200 import synth
    px = synth.make_config(0, 7, scale=size / 512.0)
    return P.RadianceImage(px.shape[1], px.shape[0], px, [("FORMAT", "32-bit_rle_rgbe")])


def test_timings_collected(P):
    timings: dict = {}
    P.encode(_gradient_image(P), timings=timings)
    for stage in ("tonemap", "base_encode", "base_decode", "prefilter", "fit", "estimate", "residual",
                  "enhancement_encode"):
        assert stage in timings
    first = dict(timings)
    P.encode(_gradient_image(P), timings=timings)  # accumulates like container._tick
    assert timings["fit"] >= first["fit"] and timings["h2d_encode_d2h"] > first["h2d_encode_d2h"]


def test_decoder_rebuilds_encoder_m_star(P):
    img = _gradient_image(P, 48)
    enc_trace: dict = {}
    stream = P.encode(img, trace=enc_trace)
    dec_trace: dict = {}
    assert P.decode_hdr(stream, trace=dec_trace) == img
    for a, b in zip(enc_trace["m_star"], dec_trace["m_star"]):
        assert (a == b).all()
    assert dec_trace["s"] == enc_trace["s"]


_DATA, _INPUTS = load_golden()
_SDR_CASES = [c for c in _DATA["cases"] if not c.get("error") and c["h"] * c["w"] <= 400_000]


@pytest.mark.parametrize("case", _SDR_CASES, ids=[c["name"] for c in _SDR_CASES])
def test_decode_sdr_matches_reference_s(P, case):
    """decode_sdr of the reference's stream == the reference's decoded S (its trace["s"])."""
    px = golden_pixels(case, _INPUTS)
    img = P.RadianceImage(px.shape[1], px.shape[0], px, [tuple(hv) for hv in case["header_vars"]],
                          case["orientation"])
    kw = dict(case["kwargs"])
    if "tmo" in kw:
        kw["tmo"] = P.TmoParams(**kw["tmo"])
    stream = P.encode(img, blas_kernel=max(case["blas_kernel"], 0), blas_threads=case["blas_threads"], **kw)
    assert hashlib.sha256(P.serialize(stream)).hexdigest() == case["stream_sha256"]
    s = P.decode_sdr(stream)
    assert hashlib.sha256(np.ascontiguousarray(s.as_array()).tobytes()).hexdigest() == case["s_sha256"]


# --------------------------------------------------------------------------
# host pipeline and re-entrancy
# --------------------------------------------------------------------------
def test_host_pipeline_bytes_equal_device_batch(P):
    import torch

    from paper_2309_11072_b200 import container, synth
    imgs = [synth.make_config(4, i, scale=0.15) for i in range(11)]
    preps = [container.prepare(P.RadianceImage(p.shape[1], p.shape[0], p, [])) for p in imgs]
    want = P.encode_batch([pr.image for pr in preps])
    h_in = [torch.from_numpy(pr.pixels).reshape(-1).pin_memory() for pr in preps]
    h_out = [torch.empty(container.stream_capacity(pr), dtype=torch.uint8).pin_memory() for pr in preps]
    for chunk, by_size in ((1, False), (3, False), (4, False), (16, False), (3, True), (4, True)):
        pipe = container.HostPipeline(preps, chunk=chunk, by_size=by_size)
        for repeats in (1, 3):
            lens = pipe.run(h_in, h_out, repeats=repeats)
            got = [bytes(h_out[i][: lens[i]].numpy()) for i in range(len(preps))]
            assert got == want, (chunk, by_size, repeats)


def test_concurrent_encode_calls_equal_serial(P):
    from paper_2309_11072_b200 import synth
    imgs = [P.RadianceImage(p.shape[1], p.shape[0], p, []) for p in
            (synth.make_config(4, 20 + i, scale=0.12) for i in range(8))]
    want = [P.serialize(P.encode(im)) for im in imgs]
    got = [None] * len(imgs)
    errs = []

    def work(k):
        try:
            for _ in range(3):
                tr: dict = {}
                st = P.encode(imgs[k], trace=tr)
                got[k] = P.serialize(st)
                assert tr["s"].width == imgs[k].width
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ths = [threading.Thread(target=work, args=(k,)) for k in range(len(imgs))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errs, errs
    assert got == want


def test_batch_on_two_streams_shares_context_safely(P):
    """Back-to-back async batches on different non-blocking streams of one context."""
    import torch

    from paper_2309_11072_b200 import _native, container, synth
    dev = torch.device("cuda", 0)
    preps = [container.prepare(P.RadianceImage(p.shape[1], p.shape[0], p, []))
             for p in (synth.make_config(1, i, scale=0.25) for i in range(6))]
    want = P.encode_batch([pr.image for pr in preps])
    ins = [torch.from_numpy(pr.pixels).to(dev) for pr in preps]
    caps = [container.stream_capacity(pr) for pr in preps]
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    outs1 = [torch.empty(c, dtype=torch.uint8, device=dev) for c in caps]
    outs2 = [torch.empty(c, dtype=torch.uint8, device=dev) for c in caps]
    l1 = torch.zeros(6, dtype=torch.int64, device=dev)
    l2 = torch.zeros(6, dtype=torch.int64, device=dev)
    ctx = _native.context(0)
    for outs, lens, s in ((outs1, l1, s1), (outs2, l2, s2)):
        container.encode_device(preps, [t.data_ptr() for t in ins], [t.data_ptr() for t in outs], caps,
                                lens.data_ptr(), s.cuda_stream, 0, ctx)
    _native.check(_native.lib().hdll_b200_sync(ctx.handle))
    torch.cuda.synchronize()
    for outs, lens in ((outs1, l1), (outs2, l2)):
        n = lens.cpu().numpy()
        assert [bytes(outs[i][: n[i]].cpu().numpy()) for i in range(6)] == want
