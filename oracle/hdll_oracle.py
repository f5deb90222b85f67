"""CPU parity oracle for the hdll encoder hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and the
``--impl reference`` arm) may import this module, and only as the checker /
the timed CPU reference.  The product path (paper_2309_11072_b200) never imports
it and has no CPU fallback.

What it is: a restatement of ``hdll.container.encode`` (reference
/root/reference/pkg/src/hdll/container.py:131-230) that runs without the
reference installed:

* elementwise float stages that the reference writes as numpy ufunc calls
  (rgbe_to_float, tone_map, srgb_quantize, gaussian_kernel) are restated with
  the same numpy ufuncs in the same order, so on one host they produce the
  reference's bits (numpy's log/exp/power are not correctly rounded and are
  host-ISA dependent);
* every loop (DCT coder, MED/Rice plane coder, CRC-32, scipy correlate1d,
  numpy pairwise sum, OpenBLAS ddot, fit_region, estimate) is restated in C
  in oracle/hdll_oracle.c with the reference's exact operation order.

Pinning: tests/test_oracle.py checks this oracle against the reference's own
golden digests (pkg/tests/fixtures/fixtures.json, regenerated images committed
under tests/golden/) and against golden vectors produced by running the real
reference in the build container (tests/golden/make_golden.py).

``blas_kernel`` (0 = OpenBLAS SKYLAKEX, 1 = HASWELL) and ``blas_threads`` are
parity parameters of the sigma>0 regression sums: the
reference's np.dot bits depend on them for regions above 10,000 pixels.
"""

from __future__ import annotations

import ctypes
import json
import math
import os
import struct
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SO = _HERE / "_build" / "libhdll_oracle.so"
_lib = None

MAGIC = b"HDLL"
VERSION = 1


def build() -> Path:
    """Compile the C restatement (gcc; no reference sources involved)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not _SO.exists() or _SO.stat().st_mtime < (_HERE / "hdll_oracle.c").stat().st_mtime:
            build()
        L = ctypes.CDLL(str(_SO))
        u8p = ctypes.POINTER(ctypes.c_uint8)
        dp = ctypes.POINTER(ctypes.c_double)
        L.ho_crc32.restype = ctypes.c_uint32
        L.ho_crc32.argtypes = [u8p, ctypes.c_size_t]
        L.ho_encode_plane.restype = ctypes.c_uint64
        L.ho_encode_plane.argtypes = [u8p, ctypes.c_int, ctypes.c_int, u8p]
        L.ho_decode_plane.restype = ctypes.c_int
        L.ho_decode_plane.argtypes = [u8p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, u8p]
        L.ho_lossy_encode.restype = ctypes.c_uint64
        L.ho_lossy_encode.argtypes = [u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int, u8p, u8p,
                                      ctypes.POINTER(ctypes.c_int64)]
        L.ho_lossy_decode.restype = ctypes.c_int
        L.ho_lossy_decode.argtypes = [u8p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int, u8p]
        L.ho_quant_tables.restype = None
        L.ho_quant_tables.argtypes = [ctypes.c_int, dp, dp]
        L.ho_prefilter.restype = None
        L.ho_prefilter.argtypes = [u8p, ctypes.c_int, ctypes.c_int, dp, ctypes.c_int, dp]
        L.ho_pairwise_sum.restype = ctypes.c_double
        L.ho_pairwise_sum.argtypes = [dp, ctypes.c_size_t]
        L.ho_ddot.restype = ctypes.c_double
        L.ho_ddot.argtypes = [dp, dp, ctypes.c_size_t, ctypes.c_int, ctypes.c_int]
        L.ho_fit.restype = ctypes.c_int
        L.ho_fit.argtypes = [ctypes.c_void_p, ctypes.c_void_p, u8p, ctypes.c_size_t, ctypes.c_int,
                             ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float),
                             ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_uint32)]
        L.ho_estimate.restype = None
        L.ho_estimate.argtypes = [dp, u8p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_float),
                                  ctypes.POINTER(ctypes.c_float), u8p]
        _lib = L
    return _lib


def _p(a: np.ndarray, ctype=ctypes.c_uint8):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


# --------------------------------------------------------------------------
# numpy restatements of the reference's elementwise float stages
# --------------------------------------------------------------------------

def rgbe_to_float(px: np.ndarray) -> np.ndarray:
    """rgbe.py:70-90: ldexp((M + 0.5) / 256, E - 128); all-zero quad -> 0."""
    mant = px[..., :3].astype(np.float64)
    expo = px[..., 3].astype(np.int64) - 128
    out = np.ldexp((mant + 0.5) / 256.0, expo[..., None])
    out[~px.any(axis=-1)] = 0.0
    return out


def tone_map(hdr: np.ndarray, key=0.18, white_point=None, gamma=2.2, epsilon=1e-6) -> np.ndarray:
    """tonemap.py:74-118 restated with the same numpy ufunc sequence.
    Returns the (H, W, 3) uint8 SDR image."""
    h, w = hdr.shape[:2]
    lum = 0.2126 * hdr[..., 0] + 0.7152 * hdr[..., 1] + 0.0722 * hdr[..., 2]
    if not (lum > 0).any():
        return np.zeros((h, w, 3), np.uint8)
    log_avg = np.exp(np.mean(np.log(epsilon + lum)))
    scaled = key * lum / log_avg
    white = white_point if white_point is not None else scaled.max()
    disp = scaled * (1.0 + scaled / (white * white)) / (1.0 + scaled)
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.where(lum > 0, disp / lum, 0.0)
    v = np.power(np.clip(hdr * ratio[..., None], 0.0, None), 1.0 / gamma)
    x = 255.0 * np.clip(v, 0.0, 1.0)
    return np.trunc(x + np.copysign(0.5, x)).astype(np.uint8)


def gaussian_taps(sigma: float) -> np.ndarray:
    """estimator.py:120-127 restated: normalised Gaussian, radius ceil(3 sigma)."""
    radius = math.ceil(3.0 * sigma)
    xs = np.arange(-radius, radius + 1, dtype=np.float64)
    wts = np.exp(-0.5 * (xs / sigma) ** 2)
    return wts / wts.sum()


def tmo_record(key=0.18, white_point=None, gamma=2.2, epsilon=1e-6) -> bytes:
    """container.py:206-214: sorted-key JSON of the TMO parameters."""
    return json.dumps({"key": key, "white_point": white_point, "gamma": gamma,
                       "epsilon": epsilon}, sort_keys=True).encode("ascii")


# --------------------------------------------------------------------------
# C-backed loops
# --------------------------------------------------------------------------

def crc32(data) -> int:
    arr = np.frombuffer(bytes(data), np.uint8) if not isinstance(data, np.ndarray) else np.ascontiguousarray(data).view(np.uint8).ravel()
    return int(lib().ho_crc32(_p(arr), arr.size))


def _frame(coder_id: int, crc: int, body: bytes) -> bytes:
    return struct.pack("<IBI", 5 + len(body), coder_id, crc) + body


def plane_bits(plane: np.ndarray) -> bytes:
    plane = np.ascontiguousarray(plane, np.uint8)
    h, w = plane.shape
    buf = np.zeros(h * w * 8 + 128, np.uint8)
    nbits = lib().ho_encode_plane(_p(plane), h, w, _p(buf))
    return buf[: (nbits + 7) // 8].tobytes()


def lossless_payload(plane: np.ndarray) -> bytes:
    """lossless_encode with coder id 1 (codec_core.py:306-313)."""
    plane = np.ascontiguousarray(plane, np.uint8)
    h, w = plane.shape
    body = struct.pack("<II", w, h) + plane_bits(plane)
    return _frame(1, crc32(plane), body)


def decode_plane(bits: bytes, h: int, w: int) -> np.ndarray:
    arr = np.frombuffer(bits, np.uint8).copy() if bits else np.zeros(1, np.uint8)
    out = np.zeros((h, w), np.uint8)
    st = lib().ho_decode_plane(_p(arr), len(bits), h, w, _p(out))
    if st:
        raise ValueError(f"corrupt plane bitstream (status {st})")
    return out


def lossy_encode(sdr: np.ndarray, quality: int):
    """Block-DCT coder id 1 (codec_core.py:430-453).  Returns (framed payload,
    decoded S (H,W,3) u8, zigzag coefficients (3, nblocks, 64) int64)."""
    sdr = np.ascontiguousarray(sdr, np.uint8)
    h, w = sdr.shape[:2]
    ph, pw = (h + 7) // 8 * 8, (w + 7) // 8 * 8
    buf = np.zeros(ph * pw * 3 * 12 + 1024, np.uint8)
    dec = np.zeros((h, w, 3), np.uint8)
    zz = np.zeros((3, (ph // 8) * (pw // 8), 64), np.int64)
    nbits = lib().ho_lossy_encode(_p(sdr), h, w, quality, _p(buf), _p(dec), _p(zz, ctypes.c_int64))
    body = struct.pack("<II", w, h) + buf[: (nbits + 7) // 8].tobytes()
    return _frame(1, crc32(dec), body), dec, zz


def lossy_decode_bits(bits: bytes, h: int, w: int, quality: int) -> np.ndarray:
    arr = np.frombuffer(bits, np.uint8).copy() if bits else np.zeros(1, np.uint8)
    out = np.zeros((h, w, 3), np.uint8)
    st = lib().ho_lossy_decode(_p(arr), len(bits), h, w, quality, _p(out))
    if st:
        raise ValueError(f"corrupt DCT bitstream (status {st})")
    return out


def quant_tables(quality: int):
    lq = np.zeros(64)
    cq = np.zeros(64)
    lib().ho_quant_tables(quality, _p(lq, ctypes.c_double), _p(cq, ctypes.c_double))
    return lq.reshape(8, 8), cq.reshape(8, 8)


def prefilter(plane: np.ndarray, taps: np.ndarray) -> np.ndarray:
    plane = np.ascontiguousarray(plane, np.uint8)
    h, w = plane.shape
    out = np.zeros((h, w), np.float64)
    taps = np.ascontiguousarray(taps, np.float64)
    lib().ho_prefilter(_p(plane), h, w, _p(taps, ctypes.c_double), (taps.size - 1) // 2,
                       _p(out, ctypes.c_double))
    return out


def pairwise_sum(a: np.ndarray) -> float:
    a = np.ascontiguousarray(a, np.float64)
    return float(lib().ho_pairwise_sum(_p(a, ctypes.c_double), a.size))


def ddot(x: np.ndarray, y: np.ndarray, kernel: int = 0, threads: int = 1) -> float:
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    return float(lib().ho_ddot(_p(x, ctypes.c_double), _p(y, ctypes.c_double), x.size, kernel, threads))


def fit(sstar, mants, e, global_regression=False, blas_kernel=0, blas_threads=1):
    """fit_slrme (estimator.py:172-214).  Returns (a32 (3,256) f32, b32, counts (256,))
    and raises ValueError like RegressionTable for non-finite float32 params."""
    n = e.size
    ss = [np.ascontiguousarray(s, np.float64).ravel() for s in sstar]
    mm = [np.ascontiguousarray(m, np.uint8).ravel() for m in mants]
    e = np.ascontiguousarray(e, np.uint8).ravel()
    sp = (ctypes.c_void_p * 3)(*[s.ctypes.data for s in ss])
    mp = (ctypes.c_void_p * 3)(*[m.ctypes.data for m in mm])
    a32 = np.zeros((3, 256), np.float32)
    b32 = np.zeros((3, 256), np.float32)
    counts = np.zeros(256, np.uint32)
    bad = lib().ho_fit(sp, mp, _p(e), n, int(global_regression), blas_kernel, blas_threads,
                       _p(a32, ctypes.c_float), _p(b32, ctypes.c_float), _p(counts, ctypes.c_uint32))
    if bad:
        raise ValueError("regression parameters must be finite")
    return a32, b32, counts


def estimate(sstar_c: np.ndarray, e: np.ndarray, a32_c: np.ndarray, b32_c: np.ndarray) -> np.ndarray:
    s = np.ascontiguousarray(sstar_c, np.float64)
    e = np.ascontiguousarray(e, np.uint8)
    out = np.zeros(e.shape, np.uint8)
    a = np.ascontiguousarray(a32_c, np.float32)
    b = np.ascontiguousarray(b32_c, np.float32)
    lib().ho_estimate(_p(s, ctypes.c_double), _p(e), e.size, _p(a, ctypes.c_float), _p(b, ctypes.c_float), _p(out))
    return out


# --------------------------------------------------------------------------
# The encode pipeline (container.py:131-230) and serialisation (:306-340)
# --------------------------------------------------------------------------

def header_block(header_vars, orientation: str) -> bytes:
    lines = [v if k == "" else f"{k}={v}" for k, v in header_vars]
    lines.append(orientation)
    return "\n".join(lines).encode("latin-1")


def encode(pixels: np.ndarray, quality: int = 85, sigma: float = 1.0, slrme: bool = True,
           global_regression: bool = False, tmo: dict | None = None, header_vars=(),
           orientation: str = "-Y +X", blas_kernel: int = 0, blas_threads: int = 1,
           trace: dict | None = None) -> bytes:
    """Serialized HDLL v1 stream for an (H, W, 4) RGBE array, default coders 1/1."""
    pixels = np.ascontiguousarray(pixels, np.uint8)
    h, w = pixels.shape[:2]
    if h <= 0 or w <= 0:
        raise ValueError("cannot encode an empty image")
    if not 0.0 <= sigma <= 65.535:
        raise ValueError("sigma must be in [0, 65.535]")
    if not 1 <= quality <= 100:
        raise ValueError("quality must be in [1, 100]")
    sigma_milli = int(round(sigma * 1000.0))
    tmo = {**dict(key=0.18, white_point=None, gamma=2.2, epsilon=1e-6), **(tmo or {})}
    mants = [pixels[..., c].copy() for c in range(3)]
    e_plane = pixels[..., 3].copy()

    sdr = tone_map(rgbe_to_float(pixels), **tmo)
    base_payload, s_img, _zz = lossy_encode(sdr, quality)
    s_planes = [s_img[..., c].copy() for c in range(3)]

    entries = []
    if slrme:
        if sigma_milli == 0:
            sstar = [p.astype(np.float64) for p in s_planes]
        else:
            taps = gaussian_taps(sigma_milli / 1000.0)
            sstar = [prefilter(p, taps) for p in s_planes]
        a32, b32, counts = fit(sstar, mants, e_plane, global_regression, blas_kernel, blas_threads)
        m_star = [estimate(sstar[c], e_plane, a32[c], b32[c]) for c in range(3)]
        for c in range(3):
            for ex in np.flatnonzero(counts):
                entries.append((c, int(ex), float(a32[c, ex]), float(b32[c, ex]), int(counts[ex])))
    else:
        m_star = s_planes
    residuals = [((m.astype(np.int16) - ms.astype(np.int16)) & 255).astype(np.uint8)
                 for m, ms in zip(mants, m_star)]
    e_payload = lossless_payload(e_plane)
    res_payloads = [lossless_payload(r) for r in residuals]

    tmo_bytes = tmo_record(**tmo)
    out = bytearray(MAGIC)
    out += struct.pack("<BIIBBBBH", VERSION, w, h, 1 if slrme else 0, 1, quality, 1, sigma_milli)
    out += struct.pack("<H", len(tmo_bytes)) + tmo_bytes
    out += struct.pack("<H", len(entries))
    for ent in entries:
        out += struct.pack("<BBffI", *ent)
    blk = header_block(list(header_vars), orientation)
    out += struct.pack("<I", len(blk)) + blk
    out += base_payload + e_payload
    for p in res_payloads:
        out += p
    if trace is not None:
        trace.update(sdr=sdr, s=s_img, m_star=m_star, residuals=residuals, entries=entries,
                     base_payload=base_payload, e_payload=e_payload, residual_payloads=res_payloads)
    return bytes(out)


def decode_hdr(stream: bytes, blas_kernel: int = 0, blas_threads: int = 1) -> np.ndarray:
    """Round-trip verifier (container.py:238-280): stream bytes -> (H, W, 4) RGBE."""
    cur = 4
    assert stream[:4] == MAGIC
    ver, w, h, flags, lossy_id, quality, lossless_id, sigma_milli = struct.unpack_from("<BIIBBBBH", stream, cur)
    cur += 15
    (tl,) = struct.unpack_from("<H", stream, cur)
    cur += 2 + tl
    (ne,) = struct.unpack_from("<H", stream, cur)
    cur += 2
    a = np.zeros((3, 256), np.float32)
    b = np.zeros((3, 256), np.float32)
    for _ in range(ne):
        ch, ex, av, bv, _cnt = struct.unpack_from("<BBffI", stream, cur)
        cur += 14
        a[ch, ex] = av
        b[ch, ex] = bv
    (bl,) = struct.unpack_from("<I", stream, cur)
    cur += 4 + bl
    payloads = []
    while cur < len(stream):
        (ln,) = struct.unpack_from("<I", stream, cur)
        payloads.append(stream[cur + 9: cur + 4 + ln])
        cur += 4 + ln
    s = lossy_decode_bits(payloads[0][8:], h, w, quality)
    e_plane = decode_plane(payloads[1][8:], h, w)
    if flags & 1:
        if sigma_milli == 0:
            sstar = [s[..., c].astype(np.float64) for c in range(3)]
        else:
            taps = gaussian_taps(sigma_milli / 1000.0)
            sstar = [prefilter(np.ascontiguousarray(s[..., c]), taps) for c in range(3)]
        m_star = [estimate(sstar[c], e_plane, a[c], b[c]) for c in range(3)]
    else:
        m_star = [s[..., c] for c in range(3)]
    out = np.zeros((h, w, 4), np.uint8)
    for c in range(3):
        r = decode_plane(payloads[2 + c][8:], h, w)
        out[..., c] = ((m_star[c].astype(np.int16) + r.astype(np.int16)) & 255).astype(np.uint8)
    out[..., 3] = e_plane
    return out


if os.environ.get("HDLL_ORACLE_BUILD_ON_IMPORT"):
    build()
