"""Tile-sharded single-image encode (BASELINE config 3).

One image, N ranks, each coding a contiguous band of rows; the output stream
is byte-identical to `container.encode` on one GPU (and to the reference).
The device work of a band runs in seven phases of the C ABI
(include/hdll_b200.h, csrc/band.cu); between phases the ranks exchange:

  1. begin    -> allgather the rank's pairwise-tree node sums of log(eps+Lw)
                 and its max Lw (tonemap.py:97-104 reduce over the whole image)
  2. layers   -> allgather the band's exponent histogram
  3. fit_send -> all-to-all: each exponent bin's (S*, M) samples go to the rank
                 owning the bin, in band order = raster order (estimator.py:145-214)
  4. fit_owner-> allgather the owners' float32 coefficients and error bits
  5. code     -> allgather the per-piece context counts and the band CRCs
  6. maps     -> allgather the per-piece A-maps (adaptive Rice state transfer
                 functions, csrc/common.cuh AMap)
  7. emit     -> gather the piece bit streams on rank 0, which concatenates them
                 and serializes (container.py:306-340)

Host-side arithmetic mirrors the device: `amap_then`/`amap_apply` restate
common.cuh, `crc32_combine` is zlib's GF(2) combine.  The exchange is an
object with allgather / alltoall / gather_pieces: `TorchExchange` runs over
torch.distributed (NCCL on B200 ranks, gloo in the CPU tests);
`ThreadExchange` runs N ranks as threads of one process on one device (each
phase ends with a stream synchronize, so no kernel ever waits on another
rank's kernel).
"""

from __future__ import annotations

import ctypes
import os
import sys
import threading
import time
from dataclasses import dataclass

import numpy as np

from . import _native, container

__all__ = ["BandSpec", "band_plan", "owner_bounds", "amap_then", "amap_apply", "crc32_combine",
           "ThreadExchange", "TorchExchange", "encode_band", "encode_tiled", "encode_tiled_dist"]

NODE_TARGET = 1024  # csrc/encoder.cuh kNodeTarget
A_DOMAIN_BITS = 14  # csrc/common.cuh kADomainBits
A_DOMAIN = 1 << A_DOMAIN_BITS
PIECES, NCTX = _native.BAND_PIECES, _native.BAND_CTX


# ---------------------------------------------------------------------------
# geometry
# ---------------------------------------------------------------------------
def pairwise_level(n: int) -> int:
    """Depth L of the cut of numpy's pairwise tree (csrc/encoder.cuh pairwise_level)."""
    L = 0
    while (n >> (L + 1)) >= NODE_TARGET:
        L += 1
    return L


def pairwise_offsets(n: int, L: int) -> np.ndarray:
    """Start offsets of the 2^L depth-L nodes, plus n (csrc/pairwise.cuh pairwise_node)."""
    off = np.zeros(1, np.int64)
    size = np.array([n], np.int64)
    for _ in range(L):
        n2 = size // 2
        n2 -= n2 % 8
        off = np.stack([off, off + n2], 1).reshape(-1)
        size = np.stack([n2, size - n2], 1).reshape(-1)
    return np.append(off, n)


@dataclass(frozen=True)
class BandSpec:
    row0: int
    row1: int
    crow0: int
    crow1: int
    node0: int
    node1: int


def band_plan(width: int, height: int, world: int, radius: int = 0) -> list[BandSpec]:
    """Contiguous bands of whole DCT block rows (8 rows), balanced by block rows.

    Each band holds the rows it codes plus the halo it recomputes: one block row
    above (DC predictor, codec_core.py:441-450) and the prefilter radius plus
    the plane coder's row above (estimator.py:130-142, _kernels.py:131-143),
    widened to the pixels of its tone-map nodes."""
    nby = (height + 7) // 8
    if not 1 <= world <= nby:
        raise ValueError(f"cannot split {nby} block rows over {world} ranks")
    n = width * height
    offs = pairwise_offsets(n, pairwise_level(n))
    out = []
    for r in range(world):
        row0 = 8 * (r * nby // world)
        row1 = min(height, 8 * ((r + 1) * nby // world))
        node0 = int(np.searchsorted(offs[:-1], row0 * width, "left"))
        node1 = int(np.searchsorted(offs[:-1], row1 * width, "left")) if r + 1 < world else len(offs) - 1
        need = max(8, radius + 1)
        crow0 = 0 if row0 == 0 else max(0, (row0 - need) // 8 * 8)
        last = row1 + radius
        if node1 > node0:
            last = max(last, -(-int(offs[node1]) // width))
            crow0 = min(crow0, int(offs[node0]) // width // 8 * 8)
        crow1 = min(height, -(-last // 8) * 8)
        out.append(BandSpec(row0, row1, crow0, crow1, node0, node1))
    return out


def owner_bounds(hist_total, world: int) -> list[int]:
    """Exponent ranges of the fit owners: contiguous, balanced by sample count."""
    h = np.asarray(hist_total, np.int64)
    total = int(h.sum())
    bounds = [0]
    acc = 0
    for e in range(256):
        acc += int(h[e])
        while len(bounds) < world and acc * world >= len(bounds) * total and total > 0:
            bounds.append(e + 1)
    while len(bounds) < world:
        bounds.append(256)
    bounds.append(256)
    return bounds


def fit_chunk_bytes(m: int) -> int:
    """Bytes of one owner chunk: [3][m] f64 S* then [3][m] u8 M, 8-byte padded (band.cu)."""
    return 24 * m + ((3 * m + 7) & ~7)


# ---------------------------------------------------------------------------
# adaptive Rice state maps (csrc/common.cuh), CRC combine (zlib)
# ---------------------------------------------------------------------------
def _make_step(c: int, s: int):
    q = c >> s
    t = min(A_DOMAIN, max(0, ((q + 1) << s) - c))
    return (q, -1, t)


def amap_apply(m, a: int) -> int:
    c, s, t = m
    return (a + c) >> s if s >= 0 else c + (1 if a >= t else 0)


def amap_then(f, g):
    """g after f (common.cuh amap_then)."""
    fc, fs, ft = f
    gc, gs, gt = g
    if fs < 0:
        v0, v1 = amap_apply(g, fc), amap_apply(g, fc + 1)
        return (v0, -1, A_DOMAIN if v1 == v0 else ft)
    if gs < 0:
        t = (gt << fs) - fc
        if gt >= A_DOMAIN:
            t = A_DOMAIN
        return (gc, -1, min(A_DOMAIN, max(0, t)))
    c, s = fc + (gc << fs), fs + gs
    if s >= A_DOMAIN_BITS:
        return _make_step(c, s)
    return (c, s, 0)


IDENTITY = (0, 0, 0)

_CRC_POLY = 0xEDB88320


def _multmodp(a: int, b: int) -> int:
    m, p = 1 << 31, 0
    while True:
        if a & m:
            p ^= b
            if (a & (m - 1)) == 0:
                break
        m >>= 1
        b = (b >> 1) ^ _CRC_POLY if b & 1 else b >> 1
    return p


_X2N = [1 << 30]  # x^(2^k) mod P, zlib's x2n_table
for _k in range(31):
    _X2N.append(_multmodp(_X2N[-1], _X2N[-1]))


def _x2nmodp(n: int, k: int) -> int:
    p = 1 << 31
    while n:
        if n & 1:
            p = _multmodp(_X2N[k & 31], p)
        n >>= 1
        k += 1
    return p


def crc32_combine(crc1: int, crc2: int, len2: int) -> int:
    """zlib.crc32(A + B) from crc32(A), crc32(B) and len(B)."""
    return _multmodp(_x2nmodp(len2, 3), crc1) ^ crc2


# ---------------------------------------------------------------------------
# exchanges
# ---------------------------------------------------------------------------
class _DevBytes:
    """A device byte range seen as a torch tensor (zero copy)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}


def _dev_tensor(ptr: int, nbytes: int, device):
    import torch

    if nbytes == 0:
        return torch.empty(0, dtype=torch.uint8, device=device)
    return torch.as_tensor(_DevBytes(ptr, nbytes), device=device)


class ThreadExchange:
    """N ranks as threads of one process (one device); see the module docstring."""

    def __init__(self, world: int):
        self.world = world
        self._bar = threading.Barrier(world)
        self._slots = [None] * world

    def view(self, rank: int):
        return _ThreadView(self, rank)


class _ThreadView:
    pieces_in_place = True  # gather_pieces hands rank 0 the other ranks' device pointers

    def __init__(self, ex: ThreadExchange, rank: int):
        self.ex, self.rank, self.world = ex, rank, ex.world

    def _swap(self, obj):
        self.ex._slots[self.rank] = obj
        self.ex._bar.wait()
        out = list(self.ex._slots)
        self.ex._bar.wait()
        return out

    def allgather(self, arr: np.ndarray):
        return [np.array(a, copy=True) for a in self._swap(np.asarray(arr))]

    def allgather_var(self, arr: np.ndarray, counts):
        return self.allgather(arr)

    def allreduce_sum(self, arr: np.ndarray):
        parts = self._swap(np.asarray(arr))
        out = np.zeros_like(parts[0])
        for p in parts:
            out += p
        return out

    def alltoall(self, send, send_bytes, recv_bytes):
        import torch

        posts = self._swap((send, list(send_bytes)))
        parts = []
        for s, (buf, sizes) in enumerate(posts):
            off = sum(sizes[: self.rank])
            parts.append(buf[off: off + sizes[self.rank]])
            assert sizes[self.rank] == recv_bytes[s]
        out = torch.cat(parts) if parts else send[:0]
        torch.cuda.synchronize(send.device)
        self._swap(None)  # every rank has copied its slices before the buffers go
        return out

    def gather_pieces(self, ptrs, nbytes, device):
        posts = self._swap(list(ptrs))
        return posts if self.rank == 0 else None, []

    def barrier(self):
        self._swap(None)


class TorchExchange:
    """torch.distributed exchange (NCCL on GPUs, gloo on CPU).

    The small per-phase summaries travel as flat tensors (one
    all_gather_into_tensor / all_reduce each; on NCCL staged through the
    device), not pickled objects."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        nccl = dist.get_backend(group) == "nccl"
        self.dev = (torch.device("cuda", torch.cuda.current_device()) if device is None else device) if nccl else None

    def _t(self, arr: np.ndarray):
        import torch

        t = torch.from_numpy(np.ascontiguousarray(arr).reshape(-1).view(np.uint8).copy())
        return t.to(self.dev) if self.dev is not None else t

    def allgather(self, arr: np.ndarray):
        """arr has the same dtype and shape on every rank"""
        import torch

        arr = np.ascontiguousarray(arr)
        if self.world == 1:
            return [arr.copy()]
        t = self._t(arr)
        out = torch.empty(self.world * t.numel(), dtype=torch.uint8, device=t.device)
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        raw = out.cpu().numpy()
        n = t.numel()
        return [raw[r * n:(r + 1) * n].view(arr.dtype).reshape(arr.shape).copy() for r in range(self.world)]

    def allgather_var(self, arr: np.ndarray, counts):
        """1-D arr of counts[rank] elements (every rank knows all counts): padded to the largest"""
        arr = np.asarray(arr)
        m = max(1, max(int(c) for c in counts))
        pad = np.zeros(m, arr.dtype)
        pad[: arr.size] = arr
        return [g[: int(c)] for g, c in zip(self.allgather(pad), counts)]

    def allreduce_sum(self, arr: np.ndarray):
        import torch

        arr = np.ascontiguousarray(arr)
        if self.world == 1:
            return arr.copy()
        t = torch.from_numpy(arr.copy())
        if self.dev is not None:
            t = t.to(self.dev)
        self.dist.all_reduce(t, group=self.group)
        return t.cpu().numpy().reshape(arr.shape)

    def alltoall(self, send, send_bytes, recv_bytes):
        import torch

        out = torch.empty(int(sum(recv_bytes)), dtype=torch.uint8, device=send.device)
        self.dist.all_to_all_single(out, send[: int(sum(send_bytes))], output_split_sizes=[int(x) for x in recv_bytes],
                                    input_split_sizes=[int(x) for x in send_bytes], group=self.group)
        if send.is_cuda:
            torch.cuda.synchronize(send.device)
        return out

    def gather_pieces(self, ptrs, nbytes, device):
        """Rank 0 receives every rank's piece streams; returns (device pointers per rank, keep-alive)."""
        import torch

        if self.world == 1:
            return [list(ptrs)], []
        sizes = self.allgather(np.asarray(nbytes, np.int64))
        if self.rank != 0:
            for p, n in zip(ptrs, nbytes):
                if n:
                    self.dist.send(_dev_tensor(int(p), int(n), device), dst=0, group=self.group)
            return None, []
        keep, out = [], [list(ptrs)]
        for r in range(1, self.world):
            got = []
            for n in sizes[r]:
                t = torch.empty(max(int(n), 16), dtype=torch.uint8, device=device)
                if n:
                    self.dist.recv(t[: int(n)], src=r, group=self.group)
                keep.append(t)
                got.append(t.data_ptr())
            out.append(got)
        return out, keep

    def barrier(self):
        self.dist.barrier(group=self.group)


# ---------------------------------------------------------------------------
# one rank
# ---------------------------------------------------------------------------
def _ptr(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def piece_chains(world: int):
    """The coder chains over the ranks' pieces, in stream order.  Pieces 0-2 are
    a band's Y, Cb, Cr slices of the base-layer DCT stream, 3-6 its E, R, G, B
    plane rows.  Y (contexts 0-2) and Cb, Cr (contexts 3-5) share no state
    (codec_core.py:439-450), so the DCT stream is two chains: Y of every rank,
    and Cb of every rank followed by Cr of every rank."""
    R = range(world)
    return ([[(r, 0) for r in R], [(r, 1) for r in R] + [(r, 2) for r in R]]
            + [[(r, 3 + k) for r in R] for k in range(4)])


def piece_roles(world: int):
    """Per (rank, piece): `first` -- it starts its chain, nothing enters it, so
    it is coded in phase 5 from the reset state; `need_map` -- a later piece
    composes its A-map (neither the chain's first nor its last); `emit` -- coded
    in phase 7 once its entering state is known."""
    first = np.zeros((world, PIECES), bool)
    need = np.zeros((world, PIECES), bool)
    for ch in piece_chains(world):
        for i, (r, p) in enumerate(ch):
            first[r, p] = i == 0
            need[r, p] = 0 < i < len(ch) - 1
    return first, need, ~first


def prefix_counts(cnts, world: int) -> np.ndarray:
    """Context counts entering every piece: the counts of the earlier pieces of its chain."""
    in_cnt = np.zeros((world, PIECES, NCTX), np.int64)
    for ch in piece_chains(world):
        run = np.zeros(NCTX, np.int64)
        for r, p in ch:
            in_cnt[r, p] = run
            run = run + np.asarray(cnts[r][p], np.int64)
    return in_cnt


def entering_a(out_a, maps, world: int) -> np.ndarray:
    """A entering every piece: the chain's first piece's outgoing A (phase 5),
    then the A-maps of the pieces between (phase 6) applied in order."""
    in_a = np.full((world, PIECES, NCTX), 4, np.int32)  # AdaptiveRiceState A = 4 (_kernels.py:114-128)
    for ch in piece_chains(world):
        r0, p0 = ch[0]
        state = [int(v) for v in out_a[r0][p0]]
        for i, (r, p) in enumerate(ch[1:], start=1):
            in_a[r, p] = state
            if i < len(ch) - 1:
                state = [amap_apply(tuple(int(x) for x in maps[r][p, c]), state[c]) for c in range(NCTX)]
    return in_a


_DIAG: dict = {}
last_phase_ms: dict = {}  # host wall time of the last encode_band's phases (each ends in a device sync)


def encode_band(ex, prep, rows_ptr: int, spec: BandSpec, ctx, stream_handle: int, device, out=None):
    """Run one rank's band of a tile-sharded encode.  rows_ptr: device RGBE rows
    [spec.crow0, spec.crow1).  Rank 0 returns the serialized stream (bytes), or,
    given `out` = (device uint8 buffer of stream_capacity bytes, device int64[1]),
    leaves it there and returns its length."""
    import torch

    L = _native.lib()
    h = ctx.handle
    W, H = prep.w, prep.h
    world, rank = ex.world, ex.rank
    specs = ex.specs
    im = container._image_struct(prep, rows_ptr)
    bd = _native.Band(spec.row0, spec.row1, spec.crow0, spec.crow1, spec.node0, spec.node1)
    diag = bool(os.environ.get("HDLL_B200_BAND_TIMING"))
    if diag:  # diagnostic: is device work pending when the encode starts?
        t_s = time.perf_counter()
        gap = 1e3 * (t_s - _DIAG.get("exit", t_s))
        torch.cuda.synchronize()
        t_1 = time.perf_counter()
        torch.cuda.synchronize()
        t_2 = time.perf_counter()
        print(f"encode_band entry: host gap {gap:.3f} ms, device sync {1e3 * (t_1 - t_s):.3f} ms, "
              f"again {1e3 * (t_2 - t_1):.3f} ms", file=sys.stderr)
    t_ph = [time.perf_counter()]
    names_ph = []

    def mark(name):
        t_ph.append(time.perf_counter())
        names_ph.append(name)

    # 1. tone-map node sums and max Lw
    nodes = np.zeros(1 + max(1, spec.node1 - spec.node0), np.float64)
    mx = ctypes.c_double(0.0)
    _native.check(L.hdll_b200_band_begin(h, ctypes.byref(im), ctypes.byref(bd), stream_handle,
                                         _ptr(nodes[1:], ctypes.c_double), ctypes.byref(mx)), "band_begin")
    nodes[0] = mx.value
    mark("begin_device")
    got = ex.allgather_var(nodes[: 1 + spec.node1 - spec.node0], [1 + s.node1 - s.node0 for s in specs])
    nodes_all = np.ascontiguousarray(np.concatenate([g[1:] for g in got]))
    maxlw = float(max(g[0] for g in got))
    mark("begin_exchange")
    # 2. layers -> histogram
    hist = np.zeros(256, np.uint32)
    _native.check(L.hdll_b200_band_layers(h, _ptr(nodes_all, ctypes.c_double), nodes_all.size, maxlw,
                                          _ptr(hist, ctypes.c_uint32)), "band_layers")
    mark("layers")
    A32 = np.zeros(768, np.float32)
    B32 = np.zeros(768, np.float32)
    status = 0
    if prep.slrme and prep.sigma_milli == 0:
        # 3-4, sigma = 0: every sum is an exact integer -- all-reduce the bin table
        # (counts, sums of x, x^2, x*y, y: 3328 int64) and fit on every rank
        sums = np.zeros(4 * 768, np.int64)
        _native.check(L.hdll_b200_band_fit_sums(h, _ptr(sums, ctypes.c_int64)), "band_fit_sums")
        tot = ex.allreduce_sum(np.concatenate([hist.astype(np.int64), sums]))
        hist_total = tot[:256]
        sums_t = np.ascontiguousarray(tot[256:])
        hist_u = np.ascontiguousarray(hist_total.astype(np.uint32))
        st = ctypes.c_uint32(0)
        _native.check(L.hdll_b200_band_fit_coef(h, _ptr(sums_t, ctypes.c_int64), _ptr(hist_u, ctypes.c_uint32),
                                                _ptr(A32, ctypes.c_float), _ptr(B32, ctypes.c_float),
                                                ctypes.byref(st)), "band_fit_coef")
        status = st.value
    elif world == 1:
        # 3-4 on one rank: its band is the image, its sorted samples all there are
        hist_total = hist.astype(np.int64)
        st = ctypes.c_uint32(0)
        _native.check(L.hdll_b200_band_fit_local(h, _ptr(A32, ctypes.c_float), _ptr(B32, ctypes.c_float),
                                                 ctypes.byref(st)), "band_fit_local")
        status = st.value
    else:
        hists = np.stack(ex.allgather(hist)).astype(np.uint32)
        hist_total = hists.astype(np.int64).sum(0)
        # 3. fit samples to their owners
        glob = bool(prep.params.global_regression)
        bounds = [0] + [256] * world if glob else owner_bounds(hist_total, world)

        def chunk(hs, o):
            if not prep.slrme:
                return 0
            if glob:
                return int(hs.astype(np.int64).sum()) if o == 0 else 0
            return int(hs[bounds[o]: bounds[o + 1]].astype(np.int64).sum())

        send_b = [fit_chunk_bytes(chunk(hist, o)) for o in range(world)]
        send = torch.empty(max(16, sum(send_b)), dtype=torch.uint8, device=device)
        send_bytes = np.zeros(world, np.uint64)
        lo_arr = np.asarray(bounds, np.uint32)
        _native.check(L.hdll_b200_band_fit_send(h, _ptr(lo_arr, ctypes.c_uint32), world, send.data_ptr(),
                                                send.numel(), _ptr(send_bytes, ctypes.c_uint64)), "band_fit_send")
        assert [int(x) for x in send_bytes] == send_b
        recv_b = [fit_chunk_bytes(chunk(hists[s], rank)) for s in range(world)]
        recv = ex.alltoall(send, send_b, recv_b)
        # 4. owner fit -> table
        a32 = np.zeros(768, np.float32)
        b32 = np.zeros(768, np.float32)
        st = ctypes.c_uint32(0)
        rb = np.asarray(recv_b, np.uint64)
        hflat = np.ascontiguousarray(hists.reshape(-1))
        recv_ptr = recv.data_ptr() if recv.numel() else send.data_ptr()
        _native.check(L.hdll_b200_band_fit_owner(h, recv_ptr, _ptr(rb, ctypes.c_uint64), _ptr(hflat, ctypes.c_uint32),
                                                 world, bounds[rank], bounds[rank + 1], _ptr(a32, ctypes.c_float),
                                                 _ptr(b32, ctypes.c_float), ctypes.byref(st)), "band_fit_owner")
        tabs = ex.allgather(np.concatenate([a32.view(np.uint32), b32.view(np.uint32), [st.value]]).astype(np.uint32))
        for o, t in enumerate(tabs):
            status |= int(t[-1])
            for c in range(3):
                sl = slice(c * 256 + bounds[o], c * 256 + bounds[o + 1])
                A32[sl] = t[:768].view(np.float32)[sl]
                B32[sl] = t[768:1536].view(np.float32)[sl]
    if status & 1:  # kErrNonFinite: RegressionTable's ValueError (estimator.py:66-67)
        raise ValueError("regression parameters must be finite")
    mark("fit")
    # 5. estimate, CRCs, piece counts; the pieces that start their chains are coded now
    first, need, emit = piece_roles(world)
    crc = np.zeros(5, np.uint32)
    cnt = np.zeros((PIECES, NCTX), np.int64)
    out_a = np.zeros((PIECES, NCTX), np.int32)
    bits = np.zeros(PIECES, np.uint64)
    ptrs = np.zeros(PIECES, np.uint64)
    fr = np.ascontiguousarray(first[rank].astype(np.int32))
    _native.check(L.hdll_b200_band_code(h, _ptr(A32, ctypes.c_float), _ptr(B32, ctypes.c_float),
                                        _ptr(fr, ctypes.c_int32), _ptr(crc, ctypes.c_uint32),
                                        _ptr(cnt, ctypes.c_int64), _ptr(out_a, ctypes.c_int32),
                                        _ptr(bits, ctypes.c_uint64), _ptr(ptrs, ctypes.c_uint64)), "band_code")
    meta = ex.allgather(np.concatenate([cnt.reshape(-1), out_a.reshape(-1).astype(np.int64), crc.astype(np.int64)]))
    nc = PIECES * NCTX
    cnts = [m[:nc].reshape(PIECES, NCTX) for m in meta]
    outs_a = [m[nc:2 * nc].reshape(PIECES, NCTX) for m in meta]
    crc_all = [m[2 * nc:] for m in meta]
    in_cnt = prefix_counts(cnts, world)
    mark("code")
    # 6. A-maps of the pieces between a chain's first and last (none for one rank)
    maps_all = None
    if need.any():
        maps = np.zeros((PIECES, NCTX, 3), np.int64)
        mine = np.ascontiguousarray(in_cnt[rank])
        nd = np.ascontiguousarray(need[rank].astype(np.int32))
        if nd.any():
            _native.check(L.hdll_b200_band_maps(h, _ptr(mine, ctypes.c_int64), _ptr(nd, ctypes.c_int32),
                                                _ptr(maps, ctypes.c_int64)), "band_maps")
        maps_all = ex.allgather(maps)
    mark("maps")
    # 7. code the remaining pieces from their entering state, gather on rank 0
    if emit[rank].any():
        in_a = entering_a(outs_a, maps_all, world)
        ina = np.ascontiguousarray(in_a[rank])
        inc = np.ascontiguousarray(in_cnt[rank])
        em = np.ascontiguousarray(emit[rank].astype(np.int32))
        bits7 = np.zeros(PIECES, np.uint64)
        _native.check(L.hdll_b200_band_emit(h, _ptr(inc, ctypes.c_int64), _ptr(ina, ctypes.c_int32),
                                            _ptr(em, ctypes.c_int32), _ptr(bits7, ctypes.c_uint64),
                                            _ptr(ptrs, ctypes.c_uint64)), "band_emit")
        bits = np.where(emit[rank], bits7, bits)
    mark("emit")
    bits_all = ex.allgather(bits.astype(np.int64)) if world > 1 else [bits.astype(np.int64)]
    nbytes = [int((int(b) + 31) // 32 * 4) for b in bits]
    all_ptrs, keep = ex.gather_pieces([int(p) for p in ptrs], nbytes, device)
    # ThreadExchange: rank 0 reads the other ranks' pieces in place, so they
    # wait until it has assembled.  TorchExchange sends them (stream-ordered on
    # NCCL's stream before the next encode's first collective), no barrier.
    in_place = getattr(ex, "pieces_in_place", False)
    if rank != 0:
        if in_place:
            ex.barrier()
        return None
    order = [[(r, c) for c in range(3) for r in range(world)]] + [[(r, 3 + k) for r in range(world)] for k in range(4)]
    npieces = np.asarray([len(ch) for ch in order], np.int32)
    pp = np.asarray([all_ptrs[r][p] for ch in order for r, p in ch], np.uint64)
    pb = np.asarray([bits_all[r][p] for ch in order for r, p in ch], np.uint64)
    # CRCs of the whole image, band by band (codec_core.py:252-253)
    crc_full = np.zeros(5, np.uint32)
    for j in range(5):
        acc = None
        for r in range(world):
            ln = (specs[r].row1 - specs[r].row0) * W * (3 if j == 0 else 1)
            acc = int(crc_all[r][j]) if acc is None else crc32_combine(acc, int(crc_all[r][j]), ln)
        crc_full[j] = acc
    hist_u32 = np.ascontiguousarray(np.asarray(hist_total).astype(np.uint32))
    cap = container.stream_capacity(prep)
    if out is not None:
        d_out, d_len = out
    else:
        d_out = torch.empty(cap, dtype=torch.uint8, device=device)
        d_len = torch.zeros(1, dtype=torch.int64, device=device)
    imf = container._image_struct(prep, 0)
    _native.check(L.hdll_b200_assemble_pieces(h, ctypes.byref(imf), _ptr(crc_full, ctypes.c_uint32),
                                              _ptr(A32, ctypes.c_float), _ptr(B32, ctypes.c_float),
                                              _ptr(hist_u32, ctypes.c_uint32), _ptr(npieces, ctypes.c_int32),
                                              _ptr(pp, ctypes.c_uint64), _ptr(pb, ctypes.c_uint64), d_out.data_ptr(),
                                              cap, d_len.data_ptr(), stream_handle), "assemble_pieces")
    n = int(d_len.item())
    if diag:
        t_s = time.perf_counter()
        torch.cuda.synchronize()
        print(f"encode_band exit device sync {1e3 * (time.perf_counter() - t_s):.3f} ms", file=sys.stderr)
        _DIAG["exit"] = time.perf_counter()
    mark("gather_assemble")
    last_phase_ms.clear()
    last_phase_ms.update({k: round((t1 - t0) * 1e3, 3) for k, t0, t1 in zip(names_ph, t_ph, t_ph[1:])})
    res = n if out is not None else bytes(d_out[:n].cpu().numpy())
    del keep
    if in_place:
        ex.barrier()
    return res


# ---------------------------------------------------------------------------
# drivers
# ---------------------------------------------------------------------------
_thread_ctx: dict = {}


def encode_tiled(image, world: int, device: int = 0, quality: int = 85, sigma: float = 1.0, slrme: bool = True,
                 global_regression: bool = False, lossy_coder: int = 1, lossless_coder: int = 1, tmo=None,
                 blas_kernel=None, blas_threads=None, return_bytes: bool = False):
    """Tile-sharded encode of one image by `world` band ranks run as threads on
    one device (each with its own context and stream).  Same stream as encode()."""
    import torch

    prep = container._prepare(image, quality, sigma, slrme, global_regression, lossy_coder, lossless_coder, tmo,
                              blas_kernel, blas_threads, False)
    specs = band_plan(prep.w, prep.h, world, prep.params.radius if slrme and prep.sigma_milli else 0)
    ex = ThreadExchange(world)
    dev = torch.device("cuda", device)
    results, errors = [None] * world, [None] * world

    def run(r):
        try:
            torch.cuda.set_device(dev)
            ctx = _thread_ctx.get((device, r))
            if ctx is None:
                ctx = _thread_ctx[(device, r)] = _native.Context(device)
            s = specs[r]
            rows = torch.from_numpy(prep.pixels[s.crow0: s.crow1]).to(dev)
            stream = torch.cuda.Stream(dev)
            view = ex.view(r)
            view.specs = specs
            results[r] = encode_band(view, prep, rows.data_ptr(), s, ctx, stream.cuda_stream, dev)
        except BaseException as e:  # noqa: BLE001 -- re-raised in the caller
            errors[r] = e
            ex._bar.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for e in errors:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in errors:
        if e is not None:
            raise e
    data = results[0]
    return data if return_bytes else container.deserialize(data)


def encode_tiled_dist(image, group=None, device=None, quality: int = 85, sigma: float = 1.0, slrme: bool = True,
                      global_regression: bool = False, tmo=None, blas_kernel=None, blas_threads=None):
    """Tile-sharded encode over the ranks of a torch.distributed group (one GPU
    per rank).  Every rank passes the same image; each uploads only its band's
    rows.  Rank 0 returns the serialized stream, the others None."""
    import torch

    ex = TorchExchange(group)
    prep = container._prepare(image, quality, sigma, slrme, global_regression, 1, 1, tmo, blas_kernel,
                              blas_threads, False)
    specs = band_plan(prep.w, prep.h, ex.world, prep.params.radius if slrme and prep.sigma_milli else 0)
    ex.specs = specs
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    s = specs[ex.rank]
    rows = torch.from_numpy(prep.pixels[s.crow0: s.crow1]).to(dev)
    ctx = _native.context(dev.index)
    stream = torch.cuda.current_stream(dev)
    return encode_band(ex, prep, rows.data_ptr(), s, ctx, stream.cuda_stream, dev)
