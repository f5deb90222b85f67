"""Multi-GPU batch sharding (BASELINE configs 1 and 4).

Images are independent units: each rank encodes its own images with no
data-path collective.  Assignment is LPT (longest processing time first) on
pixel count, which balances the mixed-size stream of config 4.  Streams can be
gathered to rank 0 in the caller's original order.

The plumbing is torch.distributed (NCCL on the GPU box, gloo in the CPU tests);
nothing here touches pixel data on the host beyond what the caller passes in.
"""

from __future__ import annotations

import heapq

__all__ = ["lpt_assign", "local_indices", "gather_streams", "encode_sharded"]


def lpt_assign(sizes, world: int) -> list[int]:
    """owner rank of every image: largest first onto the least-loaded rank
    (ties broken by the lower rank, then the lower image index)."""
    heap = [(0, r) for r in range(world)]
    owner = [0] * len(sizes)
    for i in sorted(range(len(sizes)), key=lambda i: (-int(sizes[i]), i)):
        load, r = heapq.heappop(heap)
        owner[i] = r
        heapq.heappush(heap, (load + int(sizes[i]), r))
    return owner


def local_indices(sizes, rank: int, world: int) -> list[int]:
    owner = lpt_assign(sizes, world)
    return [i for i, o in enumerate(owner) if o == rank]


def gather_streams(local: dict, n_total: int, group=None, dst: int = 0):
    """Gather {image index: stream bytes} from every rank; rank `dst` returns the
    list of all streams in original order, other ranks return None."""
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [local[i] for i in range(n_total)]
    rank = dist.get_rank(group)
    parts = [None] * dist.get_world_size(group) if rank == dst else None
    dist.gather_object(local, parts, dst=dst, group=group)
    if rank != dst:
        return None
    merged = {}
    for p in parts:
        merged.update(p)
    return [merged[i] for i in range(n_total)]


def encode_sharded(images, encode_fn, group=None, dst: int = 0):
    """Encode `images` across the ranks of `group` and gather to `dst`.

    `encode_fn(list_of_images) -> list_of_stream_bytes` runs on the local shard
    (paper_2309_11072_b200.encode_batch on a GPU rank)."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    sizes = [im.width * im.height for im in images]
    mine = local_indices(sizes, rank, world)
    out = encode_fn([images[i] for i in mine]) if mine else []
    return gather_streams(dict(zip(mine, out)), len(images), group, dst)
