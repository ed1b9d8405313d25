"""Multi-GPU sharding host logic on CPU: cost-balanced contiguous
segment ranges, and a world_size-2 gloo run where every rank generates and codes
its own shard (bench.Batch) and the root gathers -- the same code path bench.py
uses with NCCL on the box.  The per-segment codec here is the CPU oracle (test
infrastructure); tests/test_multirank_gpu.py runs the product kernels."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1709_08990_b200.shard import gather_to_root, partition_by_cost, shard_segments


def test_partition_covers_and_balances():
    rng = np.random.default_rng(0)
    for world in (1, 2, 3, 4, 8):
        for nseg in (0, 1, 5, 1000):
            costs = rng.integers(1, 2000, nseg).astype(np.float64)
            parts = partition_by_cost(costs, world)
            assert len(parts) == world
            assert parts[0][0] == 0 and parts[-1][1] == nseg
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c and a <= b
            if nseg >= 100 * world:
                loads = [costs[a:b].sum() for a, b in parts]
                assert max(loads) <= costs.sum() / world + costs.max() + 1e-9


def test_shard_segments_uses_compressed_bytes():
    lens = np.array([100, 100, 100, 100], np.uint32)
    comp = np.array([400, 0, 0, 0], np.uint64)
    parts = shard_segments(lens, comp, 2)
    assert parts[0] == (0, 1) and parts[1] == (1, 4)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results, cfg=4, scale=0.0005):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    # this rank generates and codes only its own shard (bench.Batch), no data-path collective
    wl = bench.Batch(cfg, rank, world, scale)
    es, eoff = wl.host_segments()
    enc = np.zeros(int(eoff[-1]) + 16, np.uint8)
    lens = np.zeros(wl.nseg, np.uint64)
    oracle.encode_batch(es, wl.values, enc, lens, True)
    ds = np.zeros(wl.nseg, bench.DECODE_SEG_DTYPE)
    ds["src_offset"], ds["src_bytes"], ds["dst_offset"] = eoff[:-1], lens, wl.offs[:-1]
    ds["n"], ds["prev"] = wl.lens, wl.prevs
    out = np.zeros(max(1, wl.n), np.uint32)
    assert oracle.decode_batch(ds, enc, out, True) == oracle.OK
    mine = torch.from_numpy(out[:wl.n].view(np.int32).copy())
    shards = gather_to_root(mine, world, rank)
    if rank == 0:
        whole = bench.Batch(cfg, 0, 1, scale)
        full = torch.cat(shards).numpy().view(np.uint32)
        results.put(bool(np.array_equal(full, whole.values)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(240)
def test_gloo_two_rank_shard_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(200)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True
