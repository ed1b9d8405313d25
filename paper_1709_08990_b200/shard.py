"""Multi-GPU sharding of segmented batches.

Batches of independent arrays (configs 4 and 5) shard with no collective on the
data path: every segment carries its own delta base, so rank r decodes a
contiguous range of segments on its own GPU.  Ranges are cut at equal
cumulative cost (cost of a segment = its algorithmic bytes, cmp + 4n), which
keeps the max-over-ranks time -- the one that sets whole-job throughput --
close to the mean.  Single arrays (configs 2, 3) are replicas only.

The optional gather of decoded segments to one device (timed separately) uses
torch.distributed (NCCL over NVLink on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np


def partition_by_cost(costs: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Split segments [0, len(costs)) into `world` contiguous ranges of ~equal total cost.

    Rank r gets the segments whose cumulative-cost midpoint falls in
    [r/world, (r+1)/world) of the total; ranges are contiguous, disjoint and
    cover every segment."""
    costs = np.asarray(costs, dtype=np.float64)
    n = costs.size
    if world <= 1 or n == 0:
        return [(0, n)] + [(n, n)] * max(0, world - 1)
    csum = np.cumsum(costs)
    total = csum[-1]
    mid = csum - costs / 2.0
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(mid, total * r / world, side="left")))
    cuts.append(n)
    for i in range(1, len(cuts)):  # monotone
        cuts[i] = max(cuts[i], cuts[i - 1])
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def shard_segments(lens: np.ndarray, comp_bytes: np.ndarray | None, world: int) -> list[tuple[int, int]]:
    """Cost = cmp + 4n when compressed sizes are known, else 4n."""
    lens = np.asarray(lens, dtype=np.float64)
    cost = 4.0 * lens + (np.asarray(comp_bytes, dtype=np.float64) if comp_bytes is not None else 0.0)
    return partition_by_cost(cost, world)


def gather_to_root(tensor, world: int, rank: int, root: int = 0):
    """Gather every rank's decoded shard (1-D tensor, possibly different lengths) on `root`.

    Uses torch.distributed point-to-point (NCCL send/recv over NVLink on the
    GPU box); returns the list of shards on root, None elsewhere."""
    import torch
    import torch.distributed as dist
    sizes = [torch.zeros(1, dtype=torch.int64, device=tensor.device) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([tensor.numel()], dtype=torch.int64, device=tensor.device))
    if rank == root:
        out = []
        for r in range(world):
            if r == root:
                out.append(tensor)
            else:
                buf = torch.empty(int(sizes[r].item()), dtype=tensor.dtype, device=tensor.device)
                dist.recv(buf, src=r)
                out.append(buf)
        return out
    dist.send(tensor, dst=root)
    return None
