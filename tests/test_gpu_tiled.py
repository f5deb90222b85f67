"""Tile-sharded single-image encode on one B200.

The N band ranks run as threads of this process, each with its own device
context and stream (tiled.ThreadExchange); every exchange happens on the host
between phases, so no kernel waits on another rank.  The stream must equal
the single-GPU encode() stream, which the other GPU tests pin to the oracle,
and, for one case here, the oracle directly.
"""

import numpy as np
import pytest

import paper_2309_11072_b200 as P
from paper_2309_11072_b200 import container, synth, tiled

pytestmark = pytest.mark.gpu


def _image(w, h, seed):
    pix = synth.make_config(0, seed, scale=1.0)
    rng = np.random.default_rng(seed)
    # a (h, w) crop of a config-0 scene, tiled if needed
    reps = (-(-h // pix.shape[0]), -(-w // pix.shape[1]), 1)
    pix = np.tile(pix, reps)[:h, :w].copy()
    zero = rng.random((h, w)) < 0.02
    pix[zero] = 0
    return P.RadianceImage(w, h, pix, [("FORMAT", "32-bit_rle_rgbe")])


CASES = [
    # (w, h, world, sigma, global_regression)
    (64, 96, 1, 1.0, False),
    (64, 96, 2, 1.0, False),
    (64, 96, 3, 1.0, False),
    (100, 75, 2, 1.0, False),     # width and height not multiples of 8: DCT edge padding in the last band
    (64, 96, 4, 0.0, False),      # sigma = 0: S* = S
    (96, 64, 3, 1.0, True),       # global regression: one raster-order segment, owner 0
    (128, 200, 5, 2.0, False),    # radius 6 halo
    (40, 24, 3, 1.0, False),      # one block row per rank
    (257, 130, 4, 1.0, False),
]


@pytest.mark.parametrize("w,h,world,sigma,glob", CASES)
def test_tiled_equals_single_gpu(w, h, world, sigma, glob):
    im = _image(w, h, 3000 + w + h + world)
    ref = P.serialize(P.encode(im, sigma=sigma, global_regression=glob))
    got = tiled.encode_tiled(im, world, sigma=sigma, global_regression=glob, return_bytes=True)
    assert got == ref


def test_tiled_config0_vs_oracle():
    from oracle import hdll_oracle

    pix = synth.make_config(0, 0)
    h, w = pix.shape[:2]
    im = P.RadianceImage(w, h, pix, [("FORMAT", "32-bit_rle_rgbe")])
    got = tiled.encode_tiled(im, 4, return_bytes=True)
    ref = hdll_oracle.encode(pix, sigma=1.0, header_vars=[("FORMAT", "32-bit_rle_rgbe")])
    assert got == ref


def test_tiled_repeat_and_worlds():
    im = _image(200, 160, 7)
    ref = P.serialize(P.encode(im))
    for world in (2, 6, 20):
        assert tiled.encode_tiled(im, world, return_bytes=True) == ref
    assert tiled.encode_tiled(im, 2, return_bytes=True) == ref  # contexts reused


def test_tiled_too_many_ranks():
    im = _image(32, 16, 1)
    with pytest.raises(ValueError):
        tiled.encode_tiled(im, 3)
