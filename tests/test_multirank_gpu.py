"""The sharded batch path with the product kernels, on the one GPU a gpurun lease
has: two ranks (gloo plumbing) share cuda:0, each generates only its shard
(bench.Batch), runs the batch kernels on it, checks every segment's bytes
against the oracle, and the root gathers the decoded shards and compares them
with the whole workload.  The kernels of different ranks never wait on each
other (no data-path collective: SURVEY.md §8(e)), so sharing one GPU is safe.
Also: `bench.py --gpus 2` launches its own ranks and reports n_gpus = 2."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, q, cfg, scale):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import bench
    import oracle
    from paper_1709_08990_b200.device import DeviceCodec
    from paper_1709_08990_b200.shard import gather_to_root
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dev = DeviceCodec(0)
    wl = bench.Batch(cfg, rank, world, scale)
    wl.setup(dev, torch)
    wl.decode()
    torch.cuda.synchronize()
    wl.verify(torch)
    es, eoff = wl.host_segments()
    want = np.zeros(int(eoff[-1]) + 16, np.uint8)
    lens = np.zeros(wl.nseg, np.uint64)
    oracle.encode_batch(es, wl.values, want, lens, True)
    ok = bool(np.array_equal(wl.enc_lens, lens))
    got = wl.d_c.cpu().numpy()
    ln = lens.astype(np.int64)
    pk = np.zeros(wl.nseg, np.int64)
    np.cumsum(ln[:-1], out=pk[1:])
    idx = np.arange(int(ln.sum()), dtype=np.int64) + np.repeat(eoff[:-1].astype(np.int64) - pk, ln)
    ok = ok and bool(np.array_equal(got[idx], want[idx]))
    shards = gather_to_root(wl.d_o.cpu(), world, rank)
    if rank == 0:
        whole = bench.Batch(cfg, 0, 1, scale)
        ok = ok and bool(np.array_equal(torch.cat(shards).numpy().view(np.uint32), whole.values))
    flags = [None] * world
    dist.all_gather_object(flags, ok)
    if rank == 0:
        q.put(all(flags))
    dist.barrier()
    dev.close()
    dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("cfg,scale", [(4, 0.02), (5, 1 / 64)])
def test_two_ranks_share_gpu0(cfg, scale):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q, cfg, scale)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(500)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


@pytest.mark.timeout(900)
def test_bench_spawns_its_own_ranks():
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--workload", "cfg4", "--scale", "0.02",
                          "--steps", "3", "--warmup", "3", "--no-cpu"], cwd=ROOT, capture_output=True, text=True,
                         timeout=800)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["workload"] == "cfg4"
    assert line["config"]["parallelism"].startswith("segment shards x2")
    assert line["gather"]["ok"] is True and line["gather"]["ms"] > 0
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
