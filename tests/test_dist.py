"""Batch sharding across ranks (world_size 2, gloo on CPU): LPT assignment and
the gather of per-rank streams, with the oracle standing in for the GPU encoder."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from paper_2309_11072_b200 import dist as D


def test_lpt_balances_mixed_sizes():
    from paper_2309_11072_b200 import synth
    sizes = [h * w for h, w in synth.config4_sizes(1024)]
    for world in (1, 2, 4, 8):
        owner = D.lpt_assign(sizes, world)
        loads = [sum(s for s, o in zip(sizes, owner) if o == r) for r in range(world)]
        assert max(loads) - min(loads) <= max(sizes)
        assert sorted(sum((D.local_indices(sizes, r, world) for r in range(world)), [])) == list(range(1024))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from oracle import hdll_oracle as O
    from paper_2309_11072_b200 import RadianceImage, synth

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    imgs = []
    for i in range(5):
        px = synth.make_config(4, i, scale=0.04)
        imgs.append(RadianceImage(px.shape[1], px.shape[0], px))

    def enc(batch):
        return [O.encode(im.pixels) for im in batch]

    out = D.encode_sharded(imgs, enc)
    if rank == 0:
        q.put([len(b) for b in out] + [all(o == O.encode(im.pixels) for o, im in zip(out, imgs))])
    dist.barrier()
    dist.destroy_process_group()


def test_encode_sharded_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res[-1] is True and len(res) == 6
