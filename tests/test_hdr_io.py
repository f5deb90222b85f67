"""Radiance .hdr read / write against vectors made by the
reference's radiance_io (tests/golden/make_hdr_golden.py).  Header parsing is
host logic (CPU tests); the scanline coding runs on the GPU (gpu tests)."""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2309_11072_b200 import hdr_io

GOLDEN = Path(__file__).resolve().parent / "golden"
META = json.loads((GOLDEN / "hdr_golden.json").read_text())
ARR = np.load(GOLDEN / "hdr_golden.npz")
WRITE = [c for c in META if c["kind"] == "write"]
READ = [c for c in META if c["kind"] == "read"]
HEADER_ERRORS = ("missing #?RADIANCE", "unsupported FORMAT", "resolution line")


def _file(c):
    return ARR[c["name"] + ".file"].tobytes()


@pytest.mark.parametrize("case", READ, ids=[c["name"] for c in READ])
def test_header_parse(case):
    data = _file(case)
    err = case["error"]
    if err and err.startswith(HEADER_ERRORS):
        with pytest.raises(hdr_io.RadianceFormatError, match="^" + __import__("re").escape(err) + "$"):
            hdr_io._header(data)
        return
    hv, orient, w, h, pos = hdr_io._header(data)
    if not err:
        assert [list(x) for x in hv] == [list(x) for x in case["header_vars"]]
        assert orient == case["orientation"] and (w, h) == (case["w"], case["h"])


@pytest.mark.parametrize("case", WRITE, ids=[c["name"] for c in WRITE])
def test_header_of_written_files(case):
    hv, orient, w, h, pos = hdr_io._header(_file(case))
    assert (w, h, orient) == (case["w"], case["h"], "-Y +X")
    assert [list(x) for x in hv] == [list(x) for x in case["header_vars"]]


@pytest.mark.gpu
@pytest.mark.parametrize("case", WRITE, ids=[c["name"] for c in WRITE])
def test_write_matches_reference(case):
    from paper_2309_11072_b200 import RadianceImage

    px = ARR[case["name"] + ".px"]
    img = RadianceImage(case["w"], case["h"], px, [tuple(x) for x in case["header_vars"]], "-Y +X")
    assert hdr_io.write_hdr(img, rle=case["rle"]) == _file(case)
    back = hdr_io.parse_hdr(_file(case))
    assert np.array_equal(back.pixels, px)


@pytest.mark.gpu
@pytest.mark.parametrize("case", READ, ids=[c["name"] for c in READ])
def test_read_matches_reference(case):
    data = _file(case)
    if case["error"]:
        with pytest.raises(hdr_io.RadianceFormatError) as ei:
            hdr_io.parse_hdr(data)
        assert str(ei.value) == case["error"]
        return
    img = hdr_io.parse_hdr(data)
    assert np.array_equal(img.pixels, ARR[case["name"] + ".px"])


@pytest.mark.gpu
def test_file_to_stream_on_device():
    """parse on the GPU, keep the pixels in HBM, encode: the stream equals the host path's."""
    import paper_2309_11072_b200 as P

    case = next(c for c in WRITE if c["name"] == "smooth_48x333")
    img = hdr_io.parse_hdr(_file(case), keep_on_device=True)
    host = hdr_io.parse_hdr(_file(case))
    assert np.array_equal(img.pixels.cpu().numpy(), host.pixels)
    assert P.serialize(P.encode(host)) == P.serialize(P.encode(
        P.RadianceImage(host.width, host.height, img.pixels.cpu().numpy(), host.header_vars,
                        host.resolution_orientation)))
