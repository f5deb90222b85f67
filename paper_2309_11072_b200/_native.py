"""ctypes binding of the C ABI in include/hdll_b200.h (libhdll_b200.so).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is present, `lib()` / `context()` raise immediately.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["HDLL_B200_LIB"]) if os.environ.get("HDLL_B200_LIB") else _PKG / "libhdll_b200.so"

OK, E_ARG, E_EMPTY, E_NONFINITE, E_CUDA, E_INTERNAL, E_CAPACITY = range(7)

# every symbol include/hdll_b200.h declares (checked by tests/test_host.py)
EXPORTS = (
    "hdll_b200_ctx_create", "hdll_b200_ctx_destroy", "hdll_b200_stream_capacity",
    "hdll_b200_encode_batch_device", "hdll_b200_sync", "hdll_b200_encode_host", "hdll_b200_trace",
    "hdll_b200_lossless_encode_plane", "hdll_b200_lossy_encode", "hdll_b200_last_launch_count",
    "hdll_b200_stage_times", "hdll_b200_status_string",
    "hdll_b200_band_begin", "hdll_b200_band_layers", "hdll_b200_band_fit_sums", "hdll_b200_band_fit_coef",
    "hdll_b200_band_fit_local",
    "hdll_b200_band_fit_send", "hdll_b200_band_fit_owner",
    "hdll_b200_band_code", "hdll_b200_band_maps", "hdll_b200_band_emit", "hdll_b200_assemble_pieces",
    "hdll_b200_decode_batch", "hdll_b200_hdr_decode", "hdll_b200_hdr_encode",
)

DEC_BAD, DEC_CRC, DEC_NO_ENTRY = 1 << 0, 1 << 8, 1 << 13

BAND_PIECES, BAND_CTX = 7, 6


class Params(ctypes.Structure):
    _fields_ = [
        ("quality", ctypes.c_int32), ("sigma_milli", ctypes.c_int32), ("slrme", ctypes.c_int32),
        ("global_regression", ctypes.c_int32), ("blas_kernel", ctypes.c_int32),
        ("blas_threads", ctypes.c_int32), ("radius", ctypes.c_int32), ("want_trace", ctypes.c_int32),
        ("tmo_key", ctypes.c_double), ("tmo_white_point", ctypes.c_double),
        ("tmo_inv_gamma", ctypes.c_double), ("tmo_epsilon", ctypes.c_double),
        ("taps", ctypes.POINTER(ctypes.c_double)),
    ]


class Image(ctypes.Structure):
    _fields_ = [
        ("rgbe", ctypes.c_void_p), ("width", ctypes.c_uint32), ("height", ctypes.c_uint32),
        ("hdr_pre", ctypes.c_void_p), ("hdr_pre_len", ctypes.c_uint32),
        ("hdr_post", ctypes.c_void_p), ("hdr_post_len", ctypes.c_uint32),
        ("params", Params),
    ]


class DecodeImage(ctypes.Structure):
    _fields_ = [("width", ctypes.c_uint32), ("height", ctypes.c_uint32), ("quality", ctypes.c_int32),
                ("slrme", ctypes.c_int32), ("sigma_milli", ctypes.c_int32), ("radius", ctypes.c_int32),
                ("sdr_only", ctypes.c_int32), ("taps", ctypes.POINTER(ctypes.c_double)),
                ("a32", ctypes.POINTER(ctypes.c_float)), ("b32", ctypes.POINTER(ctypes.c_float)),
                ("body", ctypes.c_void_p * 5), ("body_len", ctypes.c_uint64 * 5), ("crc", ctypes.c_uint32 * 5)]


class Band(ctypes.Structure):
    _fields_ = [("row0", ctypes.c_uint32), ("row1", ctypes.c_uint32), ("crow0", ctypes.c_uint32),
                ("crow1", ctypes.c_uint32), ("node0", ctypes.c_uint64), ("node1", ctypes.c_uint64)]


_lib = None
_lock = threading.Lock()


def lib():
    """Load libhdll_b200.so (build it with `python -m paper_2309_11072_b200._build`)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"{LIB_PATH} is missing: the B200 extension is not built "
                    "(run `python -m paper_2309_11072_b200._build`); there is no CPU fallback")
            L = ctypes.CDLL(str(LIB_PATH))
            vp, u8p, u64p = ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64)
            L.hdll_b200_ctx_create.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int]
            L.hdll_b200_ctx_create.restype = ctypes.c_int
            L.hdll_b200_ctx_destroy.argtypes = [vp]
            L.hdll_b200_ctx_destroy.restype = None
            L.hdll_b200_stream_capacity.argtypes = [ctypes.c_uint32] * 4
            L.hdll_b200_stream_capacity.restype = ctypes.c_uint64
            L.hdll_b200_encode_batch_device.argtypes = [vp, ctypes.POINTER(Image), ctypes.c_int,
                                                        ctypes.POINTER(ctypes.c_void_p), u64p, vp, vp]
            L.hdll_b200_encode_batch_device.restype = ctypes.c_int
            L.hdll_b200_sync.argtypes = [vp]
            L.hdll_b200_sync.restype = ctypes.c_int
            L.hdll_b200_encode_host.argtypes = [vp, ctypes.POINTER(Image), u8p, ctypes.c_uint64, u64p]
            L.hdll_b200_encode_host.restype = ctypes.c_int
            L.hdll_b200_trace.argtypes = [vp, ctypes.c_int, ctypes.c_int, u8p, ctypes.c_uint64]
            L.hdll_b200_trace.restype = ctypes.c_int
            L.hdll_b200_lossless_encode_plane.argtypes = [vp, u8p, ctypes.c_uint32, ctypes.c_uint32, u8p,
                                                          ctypes.c_uint64, u64p, ctypes.POINTER(ctypes.c_uint32)]
            L.hdll_b200_lossless_encode_plane.restype = ctypes.c_int
            L.hdll_b200_lossy_encode.argtypes = [vp, u8p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int32, u8p,
                                                 ctypes.c_uint64, u64p, u8p, ctypes.POINTER(ctypes.c_uint32)]
            L.hdll_b200_lossy_encode.restype = ctypes.c_int
            L.hdll_b200_last_launch_count.argtypes = [vp]
            L.hdll_b200_last_launch_count.restype = ctypes.c_int
            L.hdll_b200_stage_times.argtypes = [vp, ctypes.POINTER(ctypes.c_float), ctypes.c_int]
            L.hdll_b200_stage_times.restype = ctypes.c_int
            L.hdll_b200_status_string.argtypes = [ctypes.c_int]
            L.hdll_b200_status_string.restype = ctypes.c_char_p
            dp, i64p = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)
            u32p, f32p = ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_float)
            i32p = ctypes.POINTER(ctypes.c_int32)
            sig = {
                "hdll_b200_band_begin": [vp, ctypes.POINTER(Image), ctypes.POINTER(Band), vp, dp, dp],
                "hdll_b200_band_layers": [vp, dp, ctypes.c_uint64, ctypes.c_double, u32p],
                "hdll_b200_band_fit_send": [vp, u32p, ctypes.c_int, vp, ctypes.c_uint64, u64p],
                "hdll_b200_band_fit_owner": [vp, vp, u64p, u32p, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32,
                                             f32p, f32p, u32p],
                "hdll_b200_band_fit_sums": [vp, i64p],
                "hdll_b200_band_fit_local": [vp, f32p, f32p, u32p],
                "hdll_b200_band_fit_coef": [vp, i64p, u32p, f32p, f32p, u32p],
                "hdll_b200_band_code": [vp, f32p, f32p, i32p, u32p, i64p, i32p, u64p, u64p],
                "hdll_b200_band_maps": [vp, i64p, i32p, i64p],
                "hdll_b200_band_emit": [vp, i64p, i32p, i32p, u64p, u64p],
                "hdll_b200_assemble_pieces": [vp, ctypes.POINTER(Image), u32p, f32p, f32p, u32p,
                                              ctypes.POINTER(ctypes.c_int32), u64p, u64p, vp, ctypes.c_uint64, vp, vp],
                "hdll_b200_decode_batch": [vp, ctypes.POINTER(DecodeImage), ctypes.c_int,
                                           ctypes.POINTER(ctypes.c_void_p), u32p, vp],
                "hdll_b200_hdr_decode": [vp, vp, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, vp, u64p, i64p, vp],
                "hdll_b200_hdr_encode": [vp, vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int32, vp, ctypes.c_uint64,
                                         u64p, vp],
            }
            for name, args in sig.items():
                getattr(L, name).argtypes = args
                getattr(L, name).restype = ctypes.c_int
            _lib = L
    return _lib


class Context:
    """One device context (workspace arena + entropy status) per CUDA device."""

    def __init__(self, device: int = 0):
        self.device = device
        # held by host code that reads a batch's results (stage times, traces)
        # after the call that launched it; each C call also locks the context
        self.lock = threading.RLock()
        self.handle = ctypes.c_void_p()
        rc = lib().hdll_b200_ctx_create(ctypes.byref(self.handle), device)
        if rc != OK:
            raise RuntimeError(f"hdll_b200_ctx_create(device={device}) failed: "
                               f"{lib().hdll_b200_status_string(rc).decode()} (no CUDA device?)")

    def close(self):
        if self.handle:
            lib().hdll_b200_ctx_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_contexts: dict[int, Context] = {}


_ctx_lock = threading.Lock()


def context(device: int = 0) -> Context:
    """The device's shared context (created once; the C side serialises calls on it)."""
    with _ctx_lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = _contexts[device] = Context(device)
    return ctx


def check(rc: int, what: str = "hdll_b200"):
    """Map C status codes onto the reference's exceptions."""
    if rc == OK:
        return
    msg = lib().hdll_b200_status_string(rc).decode()
    if rc == E_EMPTY:
        from .container import StreamError
        raise StreamError(msg)
    if rc in (E_ARG, E_NONFINITE):
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg} (status {rc})")
