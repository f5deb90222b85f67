"""GPU coder plugins behind the reference's coder registry interface.

The reference registers coders with `register_lossless_coder(id, coder,
replace)` / `register_lossy_coder(...)` (codec_core.py:295-303, :509-517);
a coder exposes `encode(...)` returning the body bytes and the framing
(length, id, CRC-32) is added by lossless_encode / lossy_encode
(codec_core.py:306-313, :520-533).  `MedRicePlaneCoderB200` and
`BlockDctCoderB200` produce byte-identical bodies on the B200, so a user of the
reference can swap them in:

    import hdll
    from paper_2309_11072_b200.codec import MedRicePlaneCoderB200
    hdll.register_lossless_coder(1, MedRicePlaneCoderB200(), replace=True)

`lossless_encode` / `lossy_encode` here return the complete framed payloads.
Decoding stays with the reference (out of scope for this build).
"""

from __future__ import annotations

import ctypes
import struct

import numpy as np

from . import _native
from .container import LosslessCoderSpec, LossyCoderSpec, SdrImage, UnknownCoderError

__all__ = ["MedRicePlaneCoderB200", "BlockDctCoderB200", "lossless_encode", "lossy_encode"]


def _as_plane_u8(plane) -> np.ndarray:
    arr = np.asarray(plane)
    if arr.ndim != 2:
        raise ValueError(f"plane must be 2-D, got shape {arr.shape}")
    if arr.dtype != np.uint8:
        vals = np.asarray(arr, dtype=np.int64)
        if ((vals < 0) | (vals > 255)).any():
            raise ValueError("plane samples must be in [0, 255]")
        arr = vals.astype(np.uint8)
    return np.ascontiguousarray(arr)


class MedRicePlaneCoderB200:
    """Lossless coder id 1 (MED + context-adaptive Rice) on the B200."""

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
        return self.encode_with_crc(plane)[0]


class BlockDctCoderB200:
    """Lossy coder id 1 (8x8 block DCT) on the B200."""

    def __init__(self, device: int = 0):
        self.device = device

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


def lossless_encode(plane, spec: LosslessCoderSpec = LosslessCoderSpec()) -> bytes:
    if spec.coder_id != 1:
        raise UnknownCoderError(f"unknown lossless coder id {spec.coder_id}")
    body, crc = MedRicePlaneCoderB200().encode_with_crc(plane)
    return struct.pack("<IBI", 5 + len(body), spec.coder_id, crc) + body


def lossy_encode(image: SdrImage, spec: LossyCoderSpec = LossyCoderSpec()) -> bytes:
    if image.width <= 0 or image.height <= 0:
        raise ValueError("cannot encode an empty image")
    if spec.coder_id != 1:
        raise UnknownCoderError(f"unknown lossy coder id {spec.coder_id}")
    body, _, crc = BlockDctCoderB200().encode_with_crc(image, spec.quality)
    return struct.pack("<IBI", 5 + len(body), spec.coder_id, crc) + body
