"""Radiance `.hdr` read / write with the scanlines coded on the GPU
(reference radiance_io.py:119-326).

The text header and the resolution line are parsed here exactly as
`parse_hdr` does (radiance_io.py:119-164); the binary scanlines go through
`hdll_b200_hdr_decode` / `hdll_b200_hdr_encode` (csrc/hdrio.cu).  Output bytes
of `write_hdr` equal the reference's; `parse_hdr` returns the same image and
raises `RadianceFormatError` with the reference's messages.
"""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np

from . import _native
from .container import RadianceImage

__all__ = ["RadianceFormatError", "parse_hdr", "write_hdr", "read_hdr_file", "write_hdr_file"]

RGBE_FORMAT = "32-bit_rle_rgbe"
_SIGNATURES = (b"#?RADIANCE", b"#?RGBE")
_RESOLUTION_RE = re.compile(r"^\s*([+-][XY])\s+(\d+)\s+([+-][XY])\s+(\d+)\s*$")


class RadianceFormatError(ValueError):
    """Malformed or unsupported Radiance file data (radiance_io.py:49-50)."""


_MESSAGES = {
    17: "truncated new-RLE scanline", 18: "truncated new-RLE run", 19: "RLE run overflows scanline width",
    20: "zero-length literal packet", 21: "RLE literal overflows scanline width", 22: "truncated new-RLE literal",
    23: "truncated scanline data", 24: "repeat marker before any pixel",
    25: "old-RLE repeat overflows scanline width",
}


def _header(data: bytes):
    """radiance_io.py:121-164: header vars, orientation, dimensions, scanline offset."""
    if not any(data.startswith(sig) for sig in _SIGNATURES):
        raise RadianceFormatError("missing #?RADIANCE / #?RGBE signature")
    nl = data.find(b"\n")
    if nl < 0:
        raise RadianceFormatError("header is not newline-terminated")
    pos = nl + 1
    header_vars: list[tuple[str, str]] = []
    while True:
        nl = data.find(b"\n", pos)
        if nl < 0:
            raise RadianceFormatError("header not terminated by a blank line")
        line = data[pos:nl].decode("latin-1")
        pos = nl + 1
        if line == "":
            break
        if "=" in line and not line.startswith("#"):
            key, value = line.split("=", 1)
            header_vars.append((key, value))
        else:
            header_vars.append(("", line))
    fmt = next((v for k, v in header_vars if k == "FORMAT"), None)
    if fmt is not None and fmt != RGBE_FORMAT:
        raise RadianceFormatError(f"unsupported FORMAT {fmt!r} (only {RGBE_FORMAT})")
    nl = data.find(b"\n", pos)
    if nl < 0:
        raise RadianceFormatError("missing resolution line")
    m = _RESOLUTION_RE.match(data[pos:nl].decode("latin-1"))
    pos = nl + 1
    if not m or m.group(1)[1] == m.group(3)[1]:
        raise RadianceFormatError("resolution line does not match the -Y H +X W family")
    height, width = int(m.group(2)), int(m.group(4))
    orientation = f"{m.group(1)} {m.group(3)}"
    if width <= 0 or height <= 0:
        raise RadianceFormatError("zero image dimension in resolution line")
    return header_vars, orientation, width, height, pos


def parse_hdr(data: bytes, device: int = 0, keep_on_device: bool = False) -> RadianceImage:
    """Decode the bytes of a `.hdr` file; the scanlines expand on the GPU.
    keep_on_device: the image's pixels stay a CUDA tensor (feeds encode without
    a host round trip)."""
    import torch

    header_vars, orientation, width, height, pos = _header(data)
    body = data[pos:]
    dev = torch.device("cuda", device)
    out = torch.empty(height * width * 4, dtype=torch.uint8, device=dev)
    used = ctypes.c_uint64(0)
    detail = (ctypes.c_int64 * 2)()
    stream = torch.cuda.current_stream(dev)
    rc = _native.lib().hdll_b200_hdr_decode(_native.context(device).handle, ctypes.c_char_p(body), len(body), width,
                                            height, out.data_ptr(), ctypes.byref(used), detail, stream.cuda_stream)
    if rc == 16:
        raise RadianceFormatError(f"new-RLE scanline length {detail[0]} does not match width {detail[1]}")
    if rc in _MESSAGES:
        raise RadianceFormatError(_MESSAGES[rc])
    _native.check(rc, "hdr_decode")
    px = out.view(height, width, 4)
    if not keep_on_device:
        px = px.cpu().numpy()
    return RadianceImage(width, height, px, header_vars, orientation)


def write_hdr(image: RadianceImage, rle: bool = True, device: int = 0) -> bytes:
    """Encode a RadianceImage as `.hdr` bytes (radiance_io.py:245-286); the
    scanline packets are coded on the GPU."""
    import torch

    if image.width <= 0 or image.height <= 0:
        raise RadianceFormatError("cannot write image with zero dimension")
    pixels = image.pixels
    is_tensor = isinstance(pixels, torch.Tensor)
    shape = tuple(pixels.shape)
    dtype_ok = pixels.dtype == (torch.uint8 if is_tensor else np.uint8)
    if shape != (image.height, image.width, 4) or not dtype_ok:
        raise RadianceFormatError(f"pixels must be uint8 with shape ({image.height}, {image.width}, 4)")
    parts = image.resolution_orientation.split()
    if len(parts) != 2 or any(not re.fullmatch(r"[+-][XY]", p) for p in parts) or parts[0][1] == parts[1][1]:
        raise RadianceFormatError(f"bad resolution orientation {image.resolution_orientation!r}")
    head = bytearray(b"#?RADIANCE\n")
    for key, value in image.header_vars:
        line = value if key == "" else f"{key}={value}"
        head += line.encode("latin-1") + b"\n"
    head += b"\n"
    head += f"{parts[0]} {image.height} {parts[1]} {image.width}\n".encode("latin-1")
    dev = torch.device("cuda", device)
    d_px = pixels.to(dev).contiguous() if is_tensor else torch.from_numpy(np.ascontiguousarray(pixels)).to(dev)
    w, h = image.width, image.height
    cap = 4 * h * (1 + w + (w + 127) // 128) + 4 * h * w
    out = np.empty(cap, np.uint8)
    n = ctypes.c_uint64(0)
    stream = torch.cuda.current_stream(dev)
    _native.check(_native.lib().hdll_b200_hdr_encode(_native.context(device).handle, d_px.data_ptr(), w, h,
                                                     int(bool(rle)), out.ctypes.data, cap, ctypes.byref(n),
                                                     stream.cuda_stream), "hdr_encode")
    return bytes(head) + out[: n.value].tobytes()


def read_hdr_file(path, device: int = 0) -> RadianceImage:
    return parse_hdr(Path(path).read_bytes(), device)


def write_hdr_file(path, image: RadianceImage, rle: bool = True, device: int = 0) -> None:
    Path(path).write_bytes(write_hdr(image, rle=rle, device=device))
