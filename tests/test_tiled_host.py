"""Host logic of the tile-sharded encode (paper_2309_11072_b200/tiled.py), on CPU.

The device phases run in tests/test_gpu_tiled.py; here: band geometry, the
adaptive Rice state-map algebra the ranks use to chain their pieces, CRC
combination, owner ranges, and the torch.distributed exchange under gloo with
world size 2.
"""

import os
import socket
import zlib

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2309_11072_b200 import tiled


def test_crc32_combine_matches_zlib():
    rng = np.random.default_rng(1)
    for _ in range(50):
        a = rng.bytes(int(rng.integers(0, 5000)))
        b = rng.bytes(int(rng.integers(0, 5000)))
        assert tiled.crc32_combine(zlib.crc32(a), zlib.crc32(b), len(b)) == zlib.crc32(a + b)
    # a chain of bands, as rank 0 combines them
    parts = [rng.bytes(int(rng.integers(1, 3000))) for _ in range(7)]
    acc = zlib.crc32(parts[0])
    for p in parts[1:]:
        acc = tiled.crc32_combine(acc, zlib.crc32(p), len(p))
    assert acc == zlib.crc32(b"".join(parts))


def _pairwise_offsets_rec(n, L):
    if L == 0:
        return [0]
    n2 = n // 2
    n2 -= n2 % 8
    return _pairwise_offsets_rec(n2, L - 1) + [n2 + o for o in _pairwise_offsets_rec(n - n2, L - 1)]


@pytest.mark.parametrize("n", [1024, 4096, 6144, 393216, 7680 * 4320, 1234567])
def test_pairwise_offsets(n):
    L = tiled.pairwise_level(n)
    assert (n >> L) >= tiled.NODE_TARGET or L == 0
    offs = tiled.pairwise_offsets(n, L)
    assert list(offs[:-1]) == _pairwise_offsets_rec(n, L) and offs[-1] == n
    assert np.all(np.diff(offs) > 128)  # every node is split by numpy's recursion


@pytest.mark.parametrize("w,h,world,radius", [(64, 96, 3, 3), (100, 75, 2, 3), (40, 24, 3, 3), (7680, 4320, 8, 3),
                                              (7680, 4320, 3, 0), (128, 200, 5, 6), (257, 130, 4, 3),
                                              (33, 4000, 7, 197), (1920, 1080, 1, 3)])
def test_band_plan(w, h, world, radius):
    specs = tiled.band_plan(w, h, world, radius)
    L = tiled.pairwise_level(w * h)
    offs = tiled.pairwise_offsets(w * h, L)
    assert specs[0].row0 == 0 and specs[-1].row1 == h
    assert specs[0].node0 == 0 and specs[-1].node1 == 1 << L
    for a, b in zip(specs, specs[1:]):
        assert a.row1 == b.row0 and a.node1 == b.node0
    for s in specs:
        assert s.row0 % 8 == 0 and (s.row1 % 8 == 0 or s.row1 == h) and s.row0 < s.row1
        assert s.crow0 % 8 == 0 and (s.crow1 % 8 == 0 or s.crow1 == h)
        assert s.crow0 <= s.row0 and s.row1 <= s.crow1 <= h
        if s.row0 > 0:
            assert s.row0 - s.crow0 >= max(8, radius + 1)  # DC predictor block row, prefilter + plane halo
        if s.row1 < h:
            assert s.crow1 - s.row1 >= radius
        if s.node1 > s.node0:
            assert offs[s.node0] >= s.crow0 * w and offs[s.node1] <= s.crow1 * w
    # balanced to within one block row
    nbr = [(-(-s.row1 // 8)) - s.row0 // 8 for s in specs]
    assert max(nbr) - min(nbr) <= 1


def test_band_plan_rejects_too_many_ranks():
    with pytest.raises(ValueError):
        tiled.band_plan(32, 16, 3)


def test_owner_bounds():
    rng = np.random.default_rng(2)
    for world in (1, 2, 3, 8):
        h = np.bincount(rng.integers(90, 170, 100000), minlength=256)
        b = tiled.owner_bounds(h, world)
        assert len(b) == world + 1 and b[0] == 0 and b[-1] == 256 and b == sorted(b)
        loads = [h[b[o]: b[o + 1]].sum() for o in range(world)]
        assert sum(loads) == h.sum()
        assert max(loads) <= h.sum() / world + h.max()
    assert tiled.owner_bounds(np.zeros(256), 4) == [0, 256, 256, 256, 256]


def _halves_after(j):  # csrc/common.cuh halves_after
    return 1 if j >= 62 and (j - 62) % 32 == 0 else 0


def test_amap_chain_equals_sequential_state():
    """The adaptive Rice A of one context (_kernels.py:122-128) after a sequence
    of symbols, computed by composing per-piece maps, equals the sequential run."""
    rng = np.random.default_rng(3)
    for trial in range(200):
        n = int(rng.integers(1, 3000))
        u = rng.integers(0, 256 if trial % 3 else 8, n)
        a = 4
        for j in range(n):
            a = (a + int(u[j])) >> _halves_after(j)
        cuts = sorted(set(int(x) for x in rng.integers(0, n + 1, int(rng.integers(0, 6))))) + [n]
        comp, start = tiled.IDENTITY, 0
        for cut in cuts:
            m = tiled.IDENTITY
            for j in range(start, cut):
                m = tiled.amap_then(m, (int(u[j]), _halves_after(j), 0))
            # entering A of the piece from the composition so far
            assert tiled.amap_apply(comp, 4) >= 0
            comp = tiled.amap_then(comp, m)
            start = cut
        assert tiled.amap_apply(comp, 4) == a


def test_amap_then_is_associative_on_domain():
    rng = np.random.default_rng(4)
    def rand_map():
        m = tiled.IDENTITY
        for _ in range(int(rng.integers(0, 400))):
            m = tiled.amap_then(m, (int(rng.integers(0, 256)), int(rng.random() < 0.1), 0))
        return m
    for _ in range(60):
        f, g, k = rand_map(), rand_map(), rand_map()
        left = tiled.amap_then(tiled.amap_then(f, g), k)
        right = tiled.amap_then(f, tiled.amap_then(g, k))
        for a in list(range(0, tiled.A_DOMAIN, 97)) + [tiled.A_DOMAIN - 1]:
            want = tiled.amap_apply(k, tiled.amap_apply(g, tiled.amap_apply(f, a)))
            assert tiled.amap_apply(left, a) == want == tiled.amap_apply(right, a)


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_piece_roles(world):
    """Chains in stream order: Y by rank; Cb by rank then Cr by rank (they share
    contexts 3-5); each plane by rank.  First pieces are coded in phase 5, the
    rest in phase 7; A-maps only for pieces strictly inside a chain."""
    chains = tiled.piece_chains(world)
    assert chains[0] == [(r, 0) for r in range(world)]
    assert chains[1] == [(r, 1) for r in range(world)] + [(r, 2) for r in range(world)]
    assert sorted(x for ch in chains for x in ch) == [(r, p) for r in range(world) for p in range(tiled.PIECES)]
    first, need, emit = tiled.piece_roles(world)
    assert first[0].tolist() == [True, True, False, True, True, True, True]
    assert not first[1:].any()
    assert (emit == ~first).all()
    if world == 1:
        assert not need.any()  # one rank: phase 5 codes all but Cr, phase 7 codes Cr alone
        assert emit[0].tolist() == [False, False, True, False, False, False, False]
    else:
        assert need[0, 2] and need[world - 1, 1] and not need[world - 1, 2] and not need[0, 0]


def test_prefix_counts_and_entering_a_equal_sequential_state():
    """entering_a(out_a of the first pieces, maps) == the A a sequential coder
    has when it reaches each piece (maps composed in chain order)."""
    world = 3
    rng = np.random.default_rng(5)
    cnts = [rng.integers(0, 100, (tiled.PIECES, tiled.NCTX)) for _ in range(world)]
    in_cnt = tiled.prefix_counts(cnts, world)
    for ch in tiled.piece_chains(world):
        run = np.zeros(tiled.NCTX, np.int64)
        for r, p in ch:
            assert np.array_equal(in_cnt[r, p], run)
            run += cnts[r][p]
    # every piece's map: a random exact map (A + c) >> s of small shift
    maps = [np.zeros((tiled.PIECES, tiled.NCTX, 3), np.int64) for _ in range(world)]
    for r in range(world):
        for p in range(tiled.PIECES):
            for c in range(tiled.NCTX):
                maps[r][p, c] = (int(rng.integers(0, 300)), int(rng.integers(0, 3)), 0)
    # the sequential state: start at A = 4, apply each piece's map in chain order
    want = np.zeros((world, tiled.PIECES, tiled.NCTX), np.int64)
    out_a = [np.zeros((tiled.PIECES, tiled.NCTX), np.int64) for _ in range(world)]
    for ch in tiled.piece_chains(world):
        state = [4] * tiled.NCTX
        for i, (r, p) in enumerate(ch):
            want[r, p] = state
            state = [tiled.amap_apply(tuple(maps[r][p, c]), state[c]) for c in range(tiled.NCTX)]
            if i == 0:
                out_a[r][p] = state  # phase 5 reports the first piece's outgoing A
    got = tiled.entering_a(out_a, maps, world)
    first, _, _ = tiled.piece_roles(world)
    assert np.array_equal(got[~first], want[~first])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _exchange_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ex = tiled.TorchExchange()
        got = ex.allgather(np.arange(3) + 10 * rank)
        var = ex.allgather_var(np.arange(rank + 2, dtype=np.float64), [2, 3])
        red = ex.allreduce_sum(np.array([1, 2, 3], np.int64) * (rank + 1))
        # all-to-all with uneven chunks, as phase 3 sends fit samples to owners
        sizes = [[3, 5], [0, 7]]  # sizes[src][dst]
        send = torch.cat([torch.full((sizes[rank][d],), 16 * rank + d, dtype=torch.uint8) for d in range(world)])
        recv = ex.alltoall(send, sizes[rank], [sizes[s][rank] for s in range(world)])
        assert [v.tolist() for v in var] == [[0.0, 1.0], [0.0, 1.0, 2.0]]
        assert red.tolist() == [3, 6, 9]
        q.put((rank, [g.tolist() for g in got], recv.tolist()))
        ex.barrier()
    finally:
        dist.destroy_process_group()


def test_torch_exchange_gloo_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (g, v)) for r, g, v in (q.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert res[r][0] == [[10 * s + i for i in range(3)] for s in range(world)]
    assert res[0][1] == [0] * 3 + [16] * 0
    assert res[1][1] == [1] * 5 + [17] * 7
