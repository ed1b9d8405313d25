"""Dev tool: varint-GB encode / decode throughput on the BASELINE configs' arrays (device
buffers, L2 flushed between steps, CUDA events), checked against the input.
Usage: python tools/bench_gb.py [CFG ...]   (2: delta, sorted ids; 3: plain, mixed widths)"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1709_08990_b200 import gen  # noqa: E402
from paper_1709_08990_b200.device import DeviceCodec  # noqa: E402

dev = DeviceCodec(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
drain = torch.ones(64 << 20, dtype=torch.int32, device="cuda")


def timed(fn, reps=12):
    ts = []
    for it in range(reps):
        flush.fill_(it)
        drain.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


for cfg in [int(a) for a in sys.argv[1:]] or [2, 3]:
    v = gen.config_array(cfg)
    n = v.size
    delta = cfg in (2, 5)
    d_v = torch.from_numpy(v.view(np.int32)).cuda()
    d_c = torch.empty((n + 3) // 4 + 4 * n, dtype=torch.uint8, device="cuda")
    d_len = torch.zeros(1, dtype=torch.int64, device="cuda")
    d_o = torch.empty_like(d_v)
    te = timed(lambda: dev.gb_encode(d_v, d_c, d_len, delta=delta))
    m = int(d_len.item())
    td = timed(lambda: dev.gb_decode(d_c, n, d_o, in_len=m, delta=delta))
    dev.check()
    ok = torch.equal(d_o, d_v)
    print(f"cfg{cfg} n={n} delta={delta} bytes={m} ({m / n:.2f} B/int): encode {te:8.1f} us "
          f"({n / te / 1e3:6.1f} Gint/s)  decode {td:8.1f} us ({n / td / 1e3:6.1f} Gint/s)  ok={ok}")
