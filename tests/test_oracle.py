"""Pin the CPU oracle (test infrastructure) against the reference's golden data.

* the reference's own published digests (pkg/tests/fixtures/fixtures.json:1-48,
  produced by pkg/tests/make_fixtures.py:22-60 at seed 123, size 96);
* golden vectors produced here by running the real reference
  (tests/golden/make_golden.py -> golden.json);
* the third-party summation orders (numpy pairwise sum, OpenBLAS ddot) against
  numpy itself when the host BLAS kernel is one the oracle models.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import golden_pixels
from oracle import hdll_oracle as O

# /root/reference/pkg/tests/fixtures/fixtures.json (stream_sha256, sdr_sha256,
# m_star_sha256 per image/mode): the reference's own golden vectors.
REF_FIXTURES = {
    "gradient_00.slrme": ("0133d6d3fd3b35810d050bd53ce2429ea2ec75e675c12b5b84729c3aea8e6ed7",
                          "f1d89bc6675590c6b7486172981c4d9945e8a0b59322f8daa2a12e9918b760da",
                          "5b352044ed6b4c26dc62f18894e732411911e914f6c5c7bc890a5569d93e28dc",
                          "2268567a33e3decf2164c97a151f8969733973eba10ace5e2de502f4e95a740e"),
    "gradient_00.noslrme": ("465fdb27ca2e3ebd7ae43eb80e226237eb1fbd75d3984a25c073318bad07ae49",
                            "f1d89bc6675590c6b7486172981c4d9945e8a0b59322f8daa2a12e9918b760da",
                            "b6df56cd639aa8fbae24d879d4961b5950885dcad8f677978383a901b059f8b6",
                            "2268567a33e3decf2164c97a151f8969733973eba10ace5e2de502f4e95a740e"),
    "steps_00.slrme": ("198b71f7965b99a25dd7e52cfdc0a8b573901049227ff5b7408b754977633dde",
                       "289e2ee3427b8036238c96b79f0d46fa75c0de73996c100aca560cac79fd4c2f",
                       "616048f1efe1c7bdd1e8c5b9028ba2000734c93835eb306a332127fe8c9346db",
                       "c4d0ec222a80536256c2f263afbc616c1d744ffae3a93f07700df2b1530965c8"),
    "steps_00.noslrme": ("a21f02f7bb51942327e9344bae2b0c46982300bc667f826b24ea24bd7098029e",
                         "289e2ee3427b8036238c96b79f0d46fa75c0de73996c100aca560cac79fd4c2f",
                         "196be574f64965c3467ff1cd81cd6b0a09005384e4e80d6615aae3fc34f4b67d",
                         "c4d0ec222a80536256c2f263afbc616c1d744ffae3a93f07700df2b1530965c8"),
    "affine_00.slrme": ("4996951e9c3c33ff30673849741648f59e3b3614adec6a2bc6887d5a726d8a81",
                        "2fa375ba20645d02d3d9b9e57c110e740f53820a49480e0ce78f84a402158199",
                        "d011b8209d4d3c82ae39c154ce9eea246f2e2f4c75fd8ca05e14be823b39d4e4",
                        "c092f2034000b8d71e3b4bf73bc181b5febaf05fc82ffc4ed5bf0eaaeb73b734"),
    "affine_00.noslrme": ("b70d37362c8d8bdfdcbd11f64d8a8c40ec1ea53d968288426ece60885c28e782",
                          "2fa375ba20645d02d3d9b9e57c110e740f53820a49480e0ce78f84a402158199",
                          "a784d6bbb89bf4126737646a1dd75f5c79f60af6275bed83f096068a6acaae4d",
                          "c092f2034000b8d71e3b4bf73bc181b5febaf05fc82ffc4ed5bf0eaaeb73b734"),
}


def sha(b) -> str:
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


def oracle_encode(case, px, trace=None):
    kw = dict(case["kwargs"])
    return O.encode(px, header_vars=[tuple(hv) for hv in case["header_vars"]],
                    orientation=case["orientation"], blas_kernel=max(case["blas_kernel"], 0),
                    blas_threads=case["blas_threads"], trace=trace, **kw)


def test_reference_fixture_digests(golden):
    """The oracle reproduces every digest the reference publishes (stream, SDR, M*, HDR)."""
    data, inputs = golden
    by_name = {c["name"]: c for c in data["cases"]}
    for key, (stream_sha, sdr_sha, mstar_sha, hdr_sha) in REF_FIXTURES.items():
        case = by_name[f"fixture_{key}"]
        px = golden_pixels(case, inputs)
        tr: dict = {}
        blob = oracle_encode(case, px, tr)
        assert sha(blob) == stream_sha, key
        assert sha(tr["s"]) == sdr_sha, key  # decode_sdr(stream) == encoder-side S
        assert sha(b"".join(np.ascontiguousarray(p).tobytes() for p in tr["m_star"])) == mstar_sha, key
        assert sha(O.decode_hdr(blob)) == hdr_sha, key


def _golden_cases():
    from conftest import load_golden
    data, _ = load_golden()
    return [c for c in data["cases"] if not c["name"].startswith("c0_full")]


@pytest.mark.parametrize("case", _golden_cases(), ids=lambda c: c["name"])
def test_oracle_matches_reference_golden(case, golden):
    _, inputs = golden
    px = golden_pixels(case, inputs)
    if case["error"]:
        with pytest.raises(ValueError):
            oracle_encode(case, px)
        return
    tr: dict = {}
    blob = oracle_encode(case, px, tr)
    assert sha(tr["sdr"]) == case["sdr_sha256"]
    assert sha(tr["s"]) == case["s_sha256"]
    assert sha(b"".join(np.ascontiguousarray(p).tobytes() for p in tr["m_star"])) == case["m_star_sha256"]
    assert sha(b"".join(np.ascontiguousarray(p).tobytes() for p in tr["residuals"])) == case["residuals_sha256"]
    assert [list(e) for e in tr["entries"]] == case["table"]
    assert len(blob) == case["stream_len"]
    assert sha(blob) == case["stream_sha256"]
    assert np.array_equal(O.decode_hdr(blob), px)


def test_oracle_full_config0(golden):
    """Full-size config 0 (768x512), sigma 1 and 0: stream digest equals the reference's."""
    data, inputs = golden
    for case in data["cases"]:
        if case["name"].startswith("c0_full"):
            blob = oracle_encode(case, golden_pixels(case, inputs))
            assert sha(blob) == case["stream_sha256"], case["name"]


def _blas_kernel():
    try:
        from threadpoolctl import threadpool_info
    except ImportError:
        return None
    arch = [i.get("architecture") for i in threadpool_info() if i["user_api"] == "blas"]
    return {"SkylakeX": 0, "Haswell": 1}.get(arch[0] if arch else None)


def test_pairwise_sum_model_matches_numpy():
    rng = np.random.default_rng(0)
    for n in list(range(0, 260)) + [1000, 4095, 100003, 1 << 20, 2073601]:
        a = rng.standard_normal(n) * np.exp(rng.uniform(-5, 5, n))
        assert O.pairwise_sum(a) == np.sum(a), n


def test_ddot_model_matches_numpy():
    kernel = _blas_kernel()
    if kernel is None:
        pytest.skip("host OpenBLAS kernel is not one the oracle models")
    from threadpoolctl import threadpool_limits
    rng = np.random.default_rng(1)
    for T in (1, 2, 3, 8):
        with threadpool_limits(limits=T, user_api="blas"):
            for n in list(range(1, 130)) + [10000, 10001, 12345, 40000, 100000]:
                x = rng.uniform(0, 255, n)
                y = rng.integers(0, 256, n).astype(np.float64)
                assert O.ddot(x, x, kernel, T) == np.dot(x, x), (T, n)
                assert O.ddot(x, y, kernel, T) == np.dot(x, y), (T, n)


def test_crc32_matches_zlib():
    import zlib
    rng = np.random.default_rng(2)
    for n in (0, 1, 7, 8, 9, 1000, 65537):
        b = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert O.crc32(b) == zlib.crc32(b)
