"""bench.py --gpus N without torchrun: it re-launches itself through
torch.distributed.run with N ranks, shards ONE job over them (LPT, strong
scaling) or gives each rank its own images (--weak), and rank 0 prints one
JSON line.  Run here on CPU (gloo) with --dry-run, in which the ranks 'encode'
each image as the SHA-256 of its RGBE bytes: the gathered per-image list at
N = 2 must equal the one rank run, in image order."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _run(*args):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--dry-run", "--steps", "1", *args],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("cfg,images", [(4, 12), (1, 6)])
def test_spawn_world2_gathers_single_rank_streams(cfg, images):
    common = ["--config", str(cfg), "--images", str(images), "--scale", "0.05"]
    one = _run("--gpus", "1", *common)
    two = _run("--gpus", "2", *common)
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["scaling"] == "strong" and two["images_total"] == images
    assert two["stream_sha256"] == one["stream_sha256"]


def test_spawn_weak_scaling_gives_each_rank_its_images():
    two = _run("--gpus", "2", "--weak", "--config", "1", "--images", "3", "--scale", "0.05")
    one = _run("--gpus", "1", "--config", "1", "--images", "6", "--scale", "0.05")
    assert two["scaling"] == "weak" and two["images_total"] == 6
    assert two["stream_sha256"] == one["stream_sha256"]
