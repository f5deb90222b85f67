from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
GOLDEN = REPO / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs on the GPU box)")


def load_golden():
    data = json.loads((GOLDEN / "golden.json").read_text())
    inputs = np.load(GOLDEN / "inputs.npz")
    return data, inputs


def golden_pixels(case, inputs):
    """RGBE input of a golden case: stored in inputs.npz or regenerated from synth."""
    if case["name"] in inputs.files:
        return inputs[case["name"]]
    from paper_2309_11072_b200 import synth  # noqa: F401  (used by eval)
    return eval(case["source"], {"synth": synth})


@pytest.fixture(scope="session")
def golden():
    return load_golden()
