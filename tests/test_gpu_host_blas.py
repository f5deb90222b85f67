"""The host-library orders the parity contract models, checked on the GPU box's
own numpy: a reference run on this host would sum the
regression bins with this numpy's pairwise `sum` and this OpenBLAS's `ddot`.

These run with the GPU tests so the box that measures parity also proves that
the (kernel, thread count) model the B200 and the oracle use equals np.dot
here -- the CPU-suite copies in test_oracle.py only prove it for the build
container's host.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import hdll_oracle as O

pytestmark = pytest.mark.gpu


def test_host_blas_is_modelled():
    from paper_2309_11072_b200.container import host_blas
    hb = host_blas()
    print("host BLAS:", hb)
    assert hb["kernel"] is not None, f"OpenBLAS core type {hb['architecture']!r} has no ddot model"


def test_pairwise_sum_model_matches_host_numpy():
    rng = np.random.default_rng(0)
    for n in list(range(0, 200)) + [1000, 4095, 100003, 1 << 20]:
        a = rng.standard_normal(n) * np.exp(rng.uniform(-5, 5, n))
        assert O.pairwise_sum(a) == np.sum(a), n


@pytest.mark.parametrize("T", [1, 2, 3, 8])
def test_ddot_model_matches_host_numpy(T):
    from threadpoolctl import threadpool_limits

    from paper_2309_11072_b200.container import host_blas
    kernel = host_blas()["kernel"]
    if kernel is None:
        pytest.skip("host OpenBLAS kernel is not modelled")
    rng = np.random.default_rng(1 + T)
    with threadpool_limits(limits=T, user_api="blas"):
        for n in list(range(1, 100)) + [10000, 10001, 12345, 40000, 100000]:
            x = rng.uniform(0, 255, n)
            y = rng.integers(0, 256, n).astype(np.float64)
            assert O.ddot(x, x, kernel, T) == np.dot(x, x), (T, n)
            assert O.ddot(x, y, kernel, T) == np.dot(x, y), (T, n)
