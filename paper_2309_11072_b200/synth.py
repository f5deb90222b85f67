"""Seeded synthetic Radiance RGBE inputs for the BASELINE.json configs.

The paper's datasets (HDR-Eye, DML-HDR) are not available offline; these
generators stand in for them with the shapes, sizes and value distributions
BASELINE.json names.  Seeds are frozen here:
config c uses seed 1000*c + image_index.

`float_to_rgbe` restates the reference's float->RGBE conversion
(/root/reference/pkg/src/hdll/rgbe.py:16-67) so generated quads equal what the
reference produces for the same scene; tests/test_host.py pins that.
It is input preparation only -- not part of the encode hot path.
"""

from __future__ import annotations

import numpy as np

__all__ = ["float_to_rgbe", "config0_scene", "config1_scene", "config2_scene",
           "make_config", "CONFIG_NAMES", "config4_sizes"]


def float_to_rgbe(rgb) -> np.ndarray:
    """Nonnegative finite (..., 3) radiance -> canonical (..., 4) uint8 RGBE.

    Shared exponent e = ceil(log2(max component)) + 128, nudged until the top
    mantissa floor(max * 2^(136-e)) lies in [128, 255]; all-zero -> (0,0,0,0)
    (rgbe.py:16-67)."""
    v = np.asarray(rgb, dtype=np.float64)
    if v.ndim == 0 or v.shape[-1] != 3:
        raise ValueError(f"expected trailing dimension 3, got shape {v.shape}")
    if not np.isfinite(v).all():
        raise ValueError("radiance values must be finite")
    if (v < 0.0).any():
        raise ValueError("radiance values must be nonnegative")
    lead = v.shape[:-1]
    flat = v.reshape(-1, 3)
    top = flat.max(axis=-1)
    live = top > 0.0
    top_safe = np.where(live, top, 1.0)
    ex = np.ceil(np.log2(top_safe)).astype(np.int64) + 128
    for _ in range(3):  # power-of-two / log2 rounding overflow: step up
        hi = live & (np.floor(np.ldexp(top_safe, 136 - ex)) > 255)
        if not hi.any():
            break
        ex[hi] += 1
    for _ in range(3):  # step down while the top mantissa is below 128
        lo = live & (np.floor(np.ldexp(top_safe, 136 - ex)) < 128) & (ex > 0)
        if not lo.any():
            break
        ex[lo] -= 1
    if (live & ((ex < 0) | (ex > 255))).any():
        raise OverflowError("exponent outside [0, 255]; value not representable")
    ex = np.where(live, ex, 0)
    mant = np.clip(np.floor(np.ldexp(flat, (136 - ex)[:, None])), 0, 255)
    mant[~live] = 0
    out = np.empty((flat.shape[0], 4), np.uint8)
    out[:, :3] = mant
    out[:, 3] = ex
    return out.reshape(lead + (4,))


def _blobs(rng, h, w, count, out):
    """out *= 1 + sum_i (g_i - 1) exp(-d^2 / (2 s_i^2)), evaluated in a 5-sigma window."""
    mod = np.ones((h, w), np.float32)
    for _ in range(count):
        cy, cx = rng.uniform(0, h), rng.uniform(0, w)
        s = rng.uniform(20.0, 120.0)
        g = np.float32(2.0 ** rng.uniform(0.0, 10.0))
        y0, y1 = max(0, int(cy - 5 * s)), min(h, int(cy + 5 * s) + 1)
        x0, x1 = max(0, int(cx - 5 * s)), min(w, int(cx + 5 * s) + 1)
        if y0 >= y1 or x0 >= x1:
            continue
        dy = (np.arange(y0, y1, dtype=np.float32) - np.float32(cy)) ** 2
        dx = (np.arange(x0, x1, dtype=np.float32) - np.float32(cx)) ** 2
        inv = np.float32(-0.5 / (s * s))
        mod[y0:y1, x0:x1] += (g - 1) * (np.exp(dy * inv)[:, None] * np.exp(dx * inv)[None, :])
    out *= mod


def config0_scene(seed: int, h: int = 512, w: int = 768, log_sigma: float = 2.0, blobs: int = 16,
                  zero_frac: float = 0.0, highlight_frac: float = 0.0) -> np.ndarray:
    """fp32 scene: lum = exp(N(0, log_sigma)) x 16 Gaussian blobs (sigma 20-120 px,
    gain 2^U(0,10)), chroma U(0.5,1.5)^3, 1% multiplicative noise (BASELINE configs 0/1/3/4)."""
    rng = np.random.default_rng(seed)
    lum = np.exp(rng.standard_normal((h, w), dtype=np.float32) * np.float32(log_sigma))
    _blobs(rng, h, w, blobs, lum)
    chroma = rng.uniform(0.5, 1.5, 3).astype(np.float32)
    scene = lum[..., None] * chroma[None, None, :]
    scene *= 1 + np.float32(0.01) * rng.standard_normal((h, w, 3), dtype=np.float32)
    np.maximum(scene, 0, out=scene)
    if highlight_frac > 0:
        m = rng.random((h, w)) < highlight_frac
        hl = (2.0 ** rng.uniform(10.0, 20.0, int(m.sum()))).astype(np.float32)
        scene[m] = hl[:, None] * chroma[None, :] / chroma.max()
    if zero_frac > 0:
        scene[rng.random((h, w)) < zero_frac] = 0.0
    return scene


def config1_scene(seed: int, h: int = 1080, w: int = 1920) -> np.ndarray:
    """Config 1: config-0 generator with lum exp(N(0,3)), 2% exact zeros, 0.5% highlights <= 2^20."""
    return config0_scene(seed, h, w, log_sigma=3.0, zero_frac=0.02, highlight_frac=0.005)


def config2_scene(seed: int = 2000, h: int = 2160, w: int = 4096, lo: float = -30.0, hi: float = 30.0) -> np.ndarray:
    """Config 2: smooth wide-range field; log2 L = lo + (hi-lo) * rank(sum of 64 sinusoids)."""
    rng = np.random.default_rng(seed)
    ys = np.arange(h, dtype=np.float32)[:, None]
    xs = np.arange(w, dtype=np.float32)[None, :]
    field = np.zeros((h, w), np.float32)
    for _ in range(64):
        th = rng.uniform(0, 2 * np.pi)
        lam = 2.0 ** rng.uniform(5.0, 10.0)
        ph = rng.uniform(0, 2 * np.pi)
        k = np.float32(2 * np.pi / lam)
        field += np.sin((xs * np.float32(np.cos(th)) * k + np.float32(ph)) + ys * np.float32(np.sin(th)) * k)
    order = np.argsort(field, axis=None, kind="stable")
    u = np.empty(h * w, np.float64)
    u[order] = (np.arange(h * w, dtype=np.float64) + 0.5) / (h * w)
    lum = np.exp2(lo + (hi - lo) * u).reshape(h, w)
    chroma = rng.uniform(0.5, 1.5, 3)
    return (lum[..., None] * chroma[None, None, :]).astype(np.float64)


CONFIG_NAMES = {
    0: "c0_768x512",
    1: "c1_64x1920x1080",
    2: "c2_4096x2160_widerange",
    3: "c3_7680x4320",
    4: "c4_mixed_stream",
}

_C4_SIZES = ((512, 512), (512, 768), (768, 1024), (1080, 1920), (2160, 3840))


def config4_sizes(count: int = 1024, seed: int = 4000):
    """(h, w) of each image in config 4's mixed stream (uniform over 5 sizes)."""
    rng = np.random.default_rng(seed)
    return [_C4_SIZES[i] for i in rng.integers(0, len(_C4_SIZES), count)]


def make_config(config: int, index: int = 0, scale: float = 1.0) -> np.ndarray:
    """RGBE (H, W, 4) uint8 for image `index` of BASELINE config `config`.

    `scale` < 1 shrinks the image (parity tests at oracle-friendly sizes)."""
    def sz(h, w):
        return max(1, int(round(h * scale))), max(1, int(round(w * scale)))
    if config == 0:
        return float_to_rgbe(config0_scene(0 + index, *sz(512, 768)))
    if config == 1:
        return float_to_rgbe(config1_scene(1000 + index, *sz(1080, 1920)))
    if config == 2:
        return float_to_rgbe(config2_scene(2000 + index, *sz(2160, 4096)))
    if config == 21:  # variant 2b: spans E 2..255
        return float_to_rgbe(config2_scene(2000 + index, *sz(2160, 4096), lo=-127.0, hi=126.0))
    if config == 3:
        return float_to_rgbe(config0_scene(3000 + index, *sz(4320, 7680)))
    if config == 4:
        h, w = config4_sizes()[index]
        rng = np.random.default_rng(4000 + index)
        ls = float(rng.uniform(1.0, 4.0))
        nb = int(rng.integers(4, 65))
        return float_to_rgbe(config0_scene(4000 + index, *sz(h, w), log_sigma=ls, blobs=nb))
    raise ValueError(f"unknown config {config}")
