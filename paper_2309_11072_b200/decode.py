"""GPU decoder: decode_hdr / decode_sdr (container.py:233-280).

Host side mirrors the reference's parsing and error behaviour
(codec_core.py:234-244 `_unframe`, :260-331 / :455-476 coder `decode`,
container.py:233-280); the C ABI `hdll_b200_decode_batch` (csrc/decode.cu)
decodes the coder bodies and rebuilds S, S*, M* and the RGBE quads on the
device.  Errors are raised in the reference's order: base layer (body, bits,
CRC), exponent plane, regression-table lookup, then the R, G, B residuals.
"""

from __future__ import annotations

import ctypes
import struct

import numpy as np

from . import _native
from .container import (ChecksumError, CorruptPayloadError, DualLayerStream, RadianceImage, SdrImage, StreamError,
                        UnknownCoderError, gaussian_kernel)

__all__ = ["decode_hdr", "decode_sdr", "decode_hdr_batch"]

_NAMES = ("image", "plane", "plane", "plane", "plane")


def _unframe(payload: bytes, spec_id: int, what: str):
    """codec_core.py:234-244 plus the coder lookup of lossy/lossless_decode."""
    if len(payload) < 9:
        raise CorruptPayloadError("payload shorter than its framing")
    (length,) = struct.unpack_from("<I", payload, 0)
    if 4 + length != len(payload):
        raise CorruptPayloadError(f"payload length field {length} does not match {len(payload) - 4} bytes")
    coder_id = payload[4]
    (crc,) = struct.unpack_from("<I", payload, 5)
    if coder_id != spec_id:
        raise UnknownCoderError(f"payload coded with id {coder_id}, spec says {spec_id}")
    if coder_id != 1:
        raise UnknownCoderError(f"{what} coder id {coder_id} is not available on the B200 path")
    kind = "image" if what == "lossy" else "plane"
    if len(payload) - 9 < 8:
        raise CorruptPayloadError(f"{kind} body shorter than its dimensions")
    w, h = struct.unpack_from("<II", payload, 9)
    if w == 0 or h == 0:
        raise CorruptPayloadError(f"zero {kind} dimension")
    return crc, w, h, 17  # the coder bits start 17 bytes in: referenced in place, not copied


class _Job:
    """One stream's decode inputs, and the deferred host errors in reference order."""

    def __init__(self, stream: DualLayerStream, sdr_only: bool):
        self.stream, self.sdr_only = stream, sdr_only
        self.errors = [None] * 5
        self.bodies = [b""] * 5  # (payload, offset of its coder bits)
        self.offs = [0] * 5
        self.crcs = [0] * 5
        w = h = None
        pays = [stream.base_payload] if sdr_only else [stream.base_payload, stream.e_payload, *stream.residual_payloads]
        for k, pay in enumerate(pays):
            try:
                crc, pw, ph, off = _unframe(pay, stream.lossy_spec.coder_id if k == 0 else stream.lossless_spec.coder_id,
                                            "lossy" if k == 0 else "lossless")
                if k == 0:
                    w, h = pw, ph
                    if not sdr_only and (pw, ph) != (stream.width, stream.height):
                        raise StreamError("base layer does not match the stream dimensions")
                elif (pw, ph) != (stream.width, stream.height):
                    raise StreamError(("exponent" if k == 1 else "residual") + " plane does not match the stream dimensions")
                self.crcs[k], self.bodies[k], self.offs[k] = crc, bytes(pay), off
            except (CorruptPayloadError, UnknownCoderError, StreamError) as e:
                self.errors[k] = e
        self.w = w if w is not None else stream.width
        self.h = h if h is not None else stream.height
        self.ok_to_run = self.errors[0] is None
        a = np.full(768, np.nan, np.float32)
        b = np.full(768, np.nan, np.float32)
        for e in stream.regression_table.entries:
            a[e.channel * 256 + e.exponent] = e.a
            b[e.channel * 256 + e.exponent] = e.b
        self.a32, self.b32 = a, b
        self.taps = None
        self.radius = 0
        if stream.slrme and stream.sigma_milli and not sdr_only:
            self.taps = np.ascontiguousarray(gaussian_kernel(stream.sigma_milli / 1000.0))
            self.radius = (self.taps.size - 1) // 2

    def struct(self) -> _native.DecodeImage:
        s = self.stream
        im = _native.DecodeImage()
        im.width, im.height = self.w, self.h
        im.quality = s.lossy_spec.quality
        im.slrme = int(bool(s.slrme))
        im.sigma_milli = s.sigma_milli
        im.radius = self.radius
        im.sdr_only = int(self.sdr_only)
        im.taps = self.taps.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if self.taps is not None else None
        im.a32 = self.a32.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        im.b32 = self.b32.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        for k in range(5):
            pay, off = self.bodies[k], self.offs[k]
            n = max(len(pay) - off, 0)
            im.body[k] = (ctypes.cast(ctypes.c_char_p(pay), ctypes.c_void_p).value + off) if n else None
            im.body_len[k] = n
            im.crc[k] = self.crcs[k]
        return im

    def raise_first(self, status: int):
        """The reference's first failure: per payload framing/body, bits, CRC;
        the table lookup between the exponent plane and the residuals."""
        order = [0] if self.sdr_only else [0, 1, "table", 2, 3, 4]
        for k in order:
            if k == "table":
                if status & _native.DEC_NO_ENTRY:
                    raise StreamError("regression table incomplete: an exponent has no entry")
                continue
            if self.errors[k] is not None:
                raise self.errors[k]
            if status & (_native.DEC_BAD << k):
                raise CorruptPayloadError("corrupt DCT bitstream" if k == 0 else "corrupt plane bitstream")
            if status & (_native.DEC_CRC << k):
                raise ChecksumError(f"{_NAMES[k]} payload failed its CRC-32 check")


def _decode_trace(ctx, index: int, j: "_Job", px: np.ndarray, trace: dict):
    """decode_hdr's trace hook (container.py:269-271): the decoded S and M*
    (M* = (M - r) & 255, r the decoded residual planes)."""
    n3 = 3 * j.w * j.h
    buf = np.empty(n3, np.uint8)
    _native.check(_native.lib().hdll_b200_trace(ctx.handle, index, 16 | 1, buf.ctypes.data, n3), "decode trace")
    trace["s"] = SdrImage.from_array(buf.reshape(j.h, j.w, 3))
    res = np.empty(n3, np.uint8)
    _native.check(_native.lib().hdll_b200_trace(ctx.handle, index, 16 | 3, res.ctypes.data, n3), "decode trace")
    res = res.reshape(3, j.h, j.w)
    trace["m_star"] = tuple(((px[..., c].astype(np.int16) - res[c]) & 255).astype(np.uint8) for c in range(3))


def _decode(streams, sdr_only: bool, device: int = 0, trace: dict | None = None):
    import torch

    jobs = []
    for st in streams:
        if not sdr_only and st.sdr_only:
            raise StreamError("stream has no enhancement sections; only SDR is decodable")
        jobs.append(_Job(st, sdr_only))
    for j in jobs:
        if not j.ok_to_run:
            j.raise_first(0)
    dev = torch.device("cuda", device)
    ch = 3 if sdr_only else 4
    outs = [torch.empty(j.h * j.w * ch, dtype=torch.uint8, device=dev) for j in jobs]
    arr = (_native.DecodeImage * len(jobs))(*[j.struct() for j in jobs])
    ptrs = (ctypes.c_void_p * len(jobs))(*[o.data_ptr() for o in outs])
    status = np.zeros(len(jobs), np.uint32)
    ctx = _native.context(device)
    stream = torch.cuda.current_stream(dev)
    with ctx.lock:  # the trace reads this batch's planes
        _native.check(_native.lib().hdll_b200_decode_batch(ctx.handle, arr, len(jobs), ptrs,
                                                           status.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                                           stream.cuda_stream), "decode")
        results = []
        for j, o, s in zip(jobs, outs, status):
            j.raise_first(int(s))
            results.append(o.cpu().numpy().reshape(j.h, j.w, ch))
        if trace is not None and not sdr_only:
            _decode_trace(ctx, 0, jobs[0], results[0], trace)
    return results


def decode_hdr_batch(streams, device: int = 0) -> list:
    """decode_hdr for every stream of a batch in one device pass."""
    out = []
    for st, px in zip(streams, _decode(streams, False, device)):
        out.append(RadianceImage(st.width, st.height, px, list(st.header_vars), st.resolution_orientation))
    return out


def decode_hdr(stream: DualLayerStream, trace: dict | None = None, device: int = 0) -> RadianceImage:
    """Reconstruct the original Radiance image (container.py:238-280); `trace`
    receives the decoded S and M* like the reference's hook."""
    px = _decode([stream], False, device, trace)[0]
    return RadianceImage(stream.width, stream.height, px, list(stream.header_vars), stream.resolution_orientation)


def decode_sdr(stream: DualLayerStream, device: int = 0) -> SdrImage:
    """Decode the base layer only (container.py:233-235)."""
    return SdrImage.from_array(_decode([stream], True, device)[0])
