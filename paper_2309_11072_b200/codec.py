"""GPU coder plugins and the reference's coder registry.

The reference registers coders with `register_lossless_coder(id, coder,
replace)` / `register_lossy_coder(...)` (codec_core.py:295-303, :509-517); a
coder exposes `encode(...)` returning the body bytes and `decode(body...)`, and
the framing (length, id, CRC-32) is added and checked by lossless_encode /
lossless_decode / lossy_encode / lossy_decode (codec_core.py:306-331,
:520-548).  `MedRicePlaneCoderB200` and `BlockDctCoderB200` encode and decode
on the B200 with byte-identical bodies, so a user of the reference can swap
them in:

    import hdll
    from paper_2309_11072_b200.codec import BlockDctCoderB200, MedRicePlaneCoderB200
    hdll.register_lossless_coder(1, MedRicePlaneCoderB200(), replace=True)
    hdll.register_lossy_coder(1, BlockDctCoderB200(sdr_type=hdll.SdrImage), replace=True)

The reference's own `encode` decodes its base payload through the registered
lossy coder (container.py:172 -> codec_core.py:536-548) and `decode_hdr`
decodes every payload through the registry, so both coders implement
`decode` (the GPU decoder, `hdll_b200_decode_batch`, csrc/decode.cu).

This module also restates the registry itself (same names, arguments and
errors as codec_core.py), with the B200 coders registered as id 1: the
framed-payload API of the reference runs on this package alone.  Stored coders
(id 2) are out of scope; any registered object with the
coder interface works.
"""

from __future__ import annotations

import ctypes
import struct
import zlib

import numpy as np

from . import _native
from .container import (ChecksumError, CorruptPayloadError, LosslessCoderSpec, LossyCoderSpec, SdrImage,
                        UnknownCoderError)

__all__ = ["MedRicePlaneCoderB200", "BlockDctCoderB200", "register_lossless_coder", "register_lossy_coder",
           "lossless_encode", "lossless_decode", "lossy_encode", "lossy_decode", "payload_coder_id"]


def _as_plane_u8(plane) -> np.ndarray:
    """_util.as_plane_u8 (_util.py:14-24)."""
    arr = np.asarray(plane)
    if arr.ndim != 2:
        raise ValueError(f"plane must be 2-D, got shape {arr.shape}")
    if arr.dtype != np.uint8:
        vals = np.asarray(arr, dtype=np.int64)
        if ((vals < 0) | (vals > 255)).any():
            raise ValueError("plane samples must be in [0, 255]")
        arr = vals.astype(np.uint8)
    return np.ascontiguousarray(arr)


def _decode_body(body: bytes, kind: str, quality: int, device: int, crc: int | None = None) -> np.ndarray:
    """One coder body -> its decoded plane (h, w) or image (h, w, 3) on the GPU.
    Validation and messages follow _MedRicePlaneCoder.decode / _BlockDctCoder.decode
    (codec_core.py:267-277, :455-476).  With `crc`, the CRC-32 of the decoded
    bytes is checked on the device as lossless_decode / lossy_decode check it
    (ChecksumError)."""
    import torch

    if len(body) < 8:
        raise CorruptPayloadError(f"{kind} body shorter than its dimensions")
    w, h = struct.unpack_from("<II", body, 0)
    if w == 0 or h == 0:
        raise CorruptPayloadError(f"zero {kind} dimension")
    bits = bytes(body[8:])
    k = 0 if kind == "image" else 1
    im = _native.DecodeImage()
    im.width, im.height, im.quality = w, h, int(quality)
    im.sdr_only = 1 if kind == "image" else 2
    im.body[k] = ctypes.cast(ctypes.c_char_p(bits), ctypes.c_void_p) if bits else None
    im.body_len[k] = len(bits)
    im.crc[k] = 0 if crc is None else int(crc)
    ch = 3 if kind == "image" else 1
    dev = torch.device("cuda", device)
    out = torch.empty(h * w * ch, dtype=torch.uint8, device=dev)
    ptrs = (ctypes.c_void_p * 1)(out.data_ptr())
    status = np.zeros(1, np.uint32)
    _native.check(_native.lib().hdll_b200_decode_batch(
        _native.context(device).handle, ctypes.byref(im), 1, ptrs,
        status.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
        torch.cuda.current_stream(dev).cuda_stream), "decode")
    st = int(status[0])
    if st & (_native.DEC_BAD << k):
        raise CorruptPayloadError("corrupt DCT bitstream" if kind == "image" else "corrupt plane bitstream")
    if crc is not None and st & (_native.DEC_CRC << k):
        raise ChecksumError(f"{'image' if kind == 'image' else 'plane'} payload failed its CRC-32 check")
    arr = out.cpu().numpy()
    return arr.reshape(h, w, 3) if kind == "image" else arr.reshape(h, w)


class MedRicePlaneCoderB200:
    """Lossless coder id 1 (MED + context-adaptive Rice, codec_core.py:260-277) on the B200."""

    def __init__(self, device: int = 0):
        self.device = device

    def encode_with_crc(self, plane):
        plane = _as_plane_u8(plane)
        h, w = plane.shape
        if h == 0 or w == 0:
            raise ValueError("cannot encode an empty plane")
        cap = 8 + 8 * h * w + 64
        body = np.empty(cap, np.uint8)
        blen = ctypes.c_uint64(0)
        crc = ctypes.c_uint32(0)
        ctx = _native.context(self.device)
        _native.check(_native.lib().hdll_b200_lossless_encode_plane(
            ctx.handle, plane.ctypes.data, w, h, body.ctypes.data, cap, ctypes.byref(blen), ctypes.byref(crc)),
            "lossless_encode_plane")
        return body[: blen.value].tobytes(), crc.value

    def encode(self, plane) -> bytes:
        """codec_core.py:263-265 contract: (h, w) uint8 plane -> body (<II w, h> + bits)."""
        return self.encode_with_crc(plane)[0]

    def decode(self, body: bytes) -> np.ndarray:
        """codec_core.py:267-277 contract: body -> (h, w) uint8 plane."""
        return _decode_body(body, "plane", 85, self.device)

    def decode_checked(self, body: bytes, crc: int) -> np.ndarray:
        """decode + the CRC-32 check of lossless_decode, both on the device."""
        return _decode_body(body, "plane", 85, self.device, crc)


class BlockDctCoderB200:
    """Lossy coder id 1 (8x8 block DCT, codec_core.py:427-489) on the B200.

    `sdr_type`: the SdrImage class `decode` returns (default this package's;
    pass `hdll.SdrImage` when registering into the reference, whose
    SdrImage.__eq__ checks its own type)."""

    def __init__(self, device: int = 0, sdr_type=None):
        self.device = device
        self.sdr_type = sdr_type or SdrImage

    def encode_with_crc(self, image, quality: int):
        rgb = np.ascontiguousarray(image.as_array(), dtype=np.uint8)
        h, w = rgb.shape[:2]
        cap = 8 + 3 * ((w + 7) // 8) * ((h + 7) // 8) * 544 + 64
        body = np.empty(cap, np.uint8)
        dec = np.empty((h, w, 3), np.uint8)
        blen = ctypes.c_uint64(0)
        crc = ctypes.c_uint32(0)
        ctx = _native.context(self.device)
        _native.check(_native.lib().hdll_b200_lossy_encode(
            ctx.handle, rgb.ctypes.data, w, h, int(quality), body.ctypes.data, cap, ctypes.byref(blen),
            dec.ctypes.data, ctypes.byref(crc)), "lossy_encode")
        return body[: blen.value].tobytes(), dec, crc.value

    def encode(self, image, quality: int):
        """codec_core.py:430-453 contract: (body, decoded raw RGB bytes)."""
        body, dec, _ = self.encode_with_crc(image, quality)
        return body, dec.tobytes()

    def decode(self, body: bytes, quality: int):
        """codec_core.py:455-476 contract: body -> SdrImage (the _reconstruct of
        the decoded coefficients)."""
        return self.sdr_type.from_array(_decode_body(body, "image", quality, self.device))

    def decode_checked(self, body: bytes, quality: int, crc: int):
        """decode + the CRC-32 check of lossy_decode, both on the device."""
        return self.sdr_type.from_array(_decode_body(body, "image", quality, self.device, crc))


# --------------------------------------------------------------------------
# the registry and the framed-payload API (codec_core.py:225-331, :505-548)
# --------------------------------------------------------------------------
_LOSSLESS_CODERS: dict = {1: MedRicePlaneCoderB200()}
_LOSSY_CODERS: dict = {1: BlockDctCoderB200()}


def _frame(coder_id: int, crc: int, body: bytes) -> bytes:
    return struct.pack("<IBI", 5 + len(body), coder_id, crc) + body


def _unframe(payload: bytes):
    """codec_core.py:234-244."""
    if len(payload) < 9:
        raise CorruptPayloadError("payload shorter than its framing")
    (length,) = struct.unpack_from("<I", payload, 0)
    if 4 + length != len(payload):
        raise CorruptPayloadError(f"payload length field {length} does not match {len(payload) - 4} bytes")
    (crc,) = struct.unpack_from("<I", payload, 5)
    return payload[4], crc, payload[9:]


def payload_coder_id(payload: bytes) -> int:
    """Coder id named by a framed payload (codec_core.py:247-249)."""
    return _unframe(payload)[0]


def register_lossless_coder(coder_id: int, coder, replace: bool = False) -> None:
    """codec_core.py:298-303."""
    if not 0 <= coder_id <= 255:
        raise ValueError("coder_id must fit one byte")
    if coder_id in _LOSSLESS_CODERS and not replace:
        raise ValueError(f"lossless coder id {coder_id} already registered")
    _LOSSLESS_CODERS[coder_id] = coder


def register_lossy_coder(coder_id: int, coder, replace: bool = False) -> None:
    """codec_core.py:512-517."""
    if not 0 <= coder_id <= 255:
        raise ValueError("coder_id must fit one byte")
    if coder_id in _LOSSY_CODERS and not replace:
        raise ValueError(f"lossy coder id {coder_id} already registered")
    _LOSSY_CODERS[coder_id] = coder


def lossless_encode(plane, spec: LosslessCoderSpec = LosslessCoderSpec()) -> bytes:
    """Losslessly code a 2-D uint8 plane into a framed payload (codec_core.py:306-313).
    The B200 coder returns the CRC-32 it computed on the device; a user coder's
    body is framed with zlib's CRC of the plane bytes, as the reference does."""
    plane = _as_plane_u8(plane)
    coder = _LOSSLESS_CODERS.get(spec.coder_id)
    if coder is None:
        raise UnknownCoderError(f"unknown lossless coder id {spec.coder_id}")
    if hasattr(coder, "encode_with_crc"):
        body, crc = coder.encode_with_crc(plane)
    else:
        body, crc = coder.encode(plane), zlib.crc32(plane.tobytes()) & 0xFFFFFFFF
    return _frame(spec.coder_id, crc, body)


def lossless_decode(payload: bytes, spec: LosslessCoderSpec = LosslessCoderSpec()) -> np.ndarray:
    """Decode a framed plane payload and verify its CRC (codec_core.py:316-331)."""
    coder_id, crc, body = _unframe(payload)
    if coder_id != spec.coder_id:
        raise UnknownCoderError(f"payload coded with id {coder_id}, spec says {spec.coder_id}")
    coder = _LOSSLESS_CODERS.get(coder_id)
    if coder is None:
        raise UnknownCoderError(f"unknown lossless coder id {coder_id}")
    if hasattr(coder, "decode_checked"):
        return coder.decode_checked(body, crc)
    plane = coder.decode(body)
    if zlib.crc32(np.ascontiguousarray(plane).tobytes()) & 0xFFFFFFFF != crc:
        raise ChecksumError("plane payload failed its CRC-32 check")
    return plane


def lossy_encode(image, spec: LossyCoderSpec = LossyCoderSpec()) -> bytes:
    """Code an SDR image into a framed payload (codec_core.py:520-533); the CRC
    covers the bytes the decoder will produce."""
    if image.width <= 0 or image.height <= 0:
        raise ValueError("cannot encode an empty image")
    coder = _LOSSY_CODERS.get(spec.coder_id)
    if coder is None:
        raise UnknownCoderError(f"unknown lossy coder id {spec.coder_id}")
    if hasattr(coder, "encode_with_crc"):
        body, _, crc = coder.encode_with_crc(image, spec.quality)
    else:
        body, raw = coder.encode(image, spec.quality)
        crc = zlib.crc32(raw) & 0xFFFFFFFF
    return _frame(spec.coder_id, crc, body)


def lossy_decode(payload: bytes, spec: LossyCoderSpec = LossyCoderSpec()):
    """codec_core.py:536-548."""
    coder_id, crc, body = _unframe(payload)
    if coder_id != spec.coder_id:
        raise UnknownCoderError(f"payload coded with id {coder_id}, spec says {spec.coder_id}")
    coder = _LOSSY_CODERS.get(coder_id)
    if coder is None:
        raise UnknownCoderError(f"unknown lossy coder id {coder_id}")
    if hasattr(coder, "decode_checked"):
        return coder.decode_checked(body, spec.quality, crc)
    image = coder.decode(body, spec.quality)
    if zlib.crc32(image.as_array().tobytes()) & 0xFFFFFFFF != crc:
        raise ChecksumError("image payload failed its CRC-32 check")
    return image
