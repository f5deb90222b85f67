#!/usr/bin/env python3
"""Golden vectors for the .hdr scanline coder, produced by the REAL reference
(radiance_io.write_hdr / parse_hdr).  Build container only:

    python tests/golden/make_hdr_golden.py

Writes tests/golden/hdr_golden.npz: for every case the input pixels, the
reference's file bytes (write cases) or the hand-built file bytes and the
reference's decoded pixels (read cases: flat, old-RLE repeats, mixed), and the
reference's error message for malformed files.
"""

from __future__ import annotations

import json
import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def main() -> int:
    scratch = Path(tempfile.mkdtemp(prefix="hdll_ref_"))
    shutil.copytree("/root/reference/pkg", scratch / "pkg")
    sys.path.insert(0, str(scratch / "pkg" / "src"))
    from hdll.radiance_io import RadianceFormatError, RadianceImage, parse_hdr, write_hdr

    rng = np.random.default_rng(77)
    arrays: dict[str, np.ndarray] = {}
    meta = []

    def image(h, w, kind):
        if kind == "noise":
            px = rng.integers(0, 256, (h, w, 4), dtype=np.uint8)
        elif kind == "runs":  # runs of every length around the 4 / 127 / 128 thresholds
            px = np.zeros((h, w, 4), np.uint8)
            for y in range(h):
                x = 0
                while x < w:
                    ln = int(rng.choice([1, 2, 3, 4, 5, 126, 127, 128, 129, 255, 300]))
                    px[y, x:x + ln] = rng.integers(0, 256, 4, dtype=np.uint8)
                    x += ln
        else:  # smooth: long constant exponent, slowly varying mantissas
            yy, xx = np.mgrid[0:h, 0:w]
            px = np.stack([(xx // 7) % 256, (yy // 5) % 256, ((xx + yy) // 9) % 256,
                           np.full_like(xx, 130)], -1).astype(np.uint8)
        return px

    for name, h, w, kind, rle in [("noise_64x96", 64, 96, "noise", True), ("runs_20x700", 20, 700, "runs", True),
                                  ("smooth_48x333", 48, 333, "smooth", True), ("narrow_9x7", 9, 7, "noise", True),
                                  ("flat_12x40", 12, 40, "runs", False), ("w8_5x8", 5, 8, "runs", True),
                                  ("wide_3x40000", 3, 40000, "runs", True)]:
        px = image(h, w, kind)
        hv = [("FORMAT", "32-bit_rle_rgbe"), ("", "# a comment"), ("EXPOSURE", "1.0")]
        data = write_hdr(RadianceImage(w, h, px, hv, "-Y +X"), rle=rle)
        back = parse_hdr(data)
        assert np.array_equal(back.pixels, px)
        arrays[f"{name}.px"] = px
        arrays[f"{name}.file"] = np.frombuffer(data, np.uint8)
        meta.append({"name": name, "kind": "write", "rle": rle, "h": h, "w": w, "header_vars": hv})

    def read_case(name, data: bytes):
        try:
            img = parse_hdr(data)
            arrays[f"{name}.px"] = img.pixels
            err = None
            info = {"h": img.height, "w": img.width, "header_vars": img.header_vars,
                    "orientation": img.resolution_orientation}
        except RadianceFormatError as e:
            err, info = str(e), {}
        arrays[f"{name}.file"] = np.frombuffer(data, np.uint8)
        meta.append({"name": name, "kind": "read", "error": err, **info})

    hdr = b"#?RADIANCE\nFORMAT=32-bit_rle_rgbe\n\n-Y 3 +X 10\n"
    px = [bytes([10 + i, 20, 30, 128]) for i in range(10)]
    flat = b"".join(px)
    read_case("flat_rows", hdr + flat * 3)
    # old-RLE: a pixel then (1,1,1,n) repeats, a repeat run spanning scanlines via prev
    old = px[0] + b"\x01\x01\x01\x04" + px[1] + b"\x01\x01\x01\x03" + px[2]  # 1 + 4 + 1 + 3 + 1 = 10
    old2 = b"\x01\x01\x01\x0a"  # the whole second scanline repeats the previous pixel
    old3 = px[3] + b"\x01\x01\x01\x01" + b"\x01\x01\x01\x00" + px[4] * 8  # shifted repeat counts: 1 + 0<<8
    read_case("old_rle", hdr + old + old2 + old3)
    new = write_hdr(RadianceImage(10, 1, np.frombuffer(flat, np.uint8).reshape(1, 10, 4).copy(), [], "-Y +X"))
    new_line = new[new.index(b"+X 10\n") + 6:]
    read_case("mixed_new_old", b"#?RADIANCE\n\n-Y 3 +X 10\n" + new_line + old2 + flat)
    read_case("orient_+x", b"#?RGBE\n\n+X 10 -Y 3\n" + flat * 3)
    read_case("err_repeat_first", hdr + b"\x01\x01\x01\x02" + flat)
    read_case("err_trunc", hdr + flat * 2 + flat[:7])
    read_case("err_len", hdr + b"\x02\x02\x00\x09" + flat * 3)
    read_case("err_zero_lit", b"#?RADIANCE\n\n-Y 1 +X 10\n\x02\x02\x00\x0a\x00" + flat)
    read_case("err_run_overflow", b"#?RADIANCE\n\n-Y 1 +X 10\n\x02\x02\x00\x0a\x8b\x05" + flat)
    read_case("err_lit_overflow", b"#?RADIANCE\n\n-Y 1 +X 10\n\x02\x02\x00\x0a\x0b" + flat)
    read_case("err_trunc_lit", b"#?RADIANCE\n\n-Y 1 +X 10\n\x02\x02\x00\x0a\x0a\x01\x02")
    read_case("err_trunc_run", b"#?RADIANCE\n\n-Y 1 +X 10\n\x02\x02\x00\x0a\x8a")
    read_case("err_trunc_line", b"#?RADIANCE\n\n-Y 1 +X 10\n\x02\x02\x00\x0a\x85\x07")
    read_case("err_repeat_overflow", hdr + px[0] + b"\x01\x01\x01\x0a" + flat * 2)
    read_case("err_signature", b"#?NOPE\n\n-Y 1 +X 10\n" + flat)
    read_case("err_format", b"#?RADIANCE\nFORMAT=32-bit_rle_xyze\n\n-Y 1 +X 10\n" + flat)
    read_case("err_resolution", b"#?RADIANCE\n\n-Y 1 -Y 10\n" + flat)

    np.savez_compressed(HERE / "hdr_golden.npz", **arrays)
    (HERE / "hdr_golden.json").write_text(json.dumps(meta, indent=1))
    print(len(meta), "cases")
    return 0


if __name__ == "__main__":
    sys.exit(main())
