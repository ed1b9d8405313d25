"""Dev tool: time encoded_sizes_batch on cfg4/cfg5 (scale) against encode_batch."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1709_08990_b200.device import DeviceCodec  # noqa: E402

cfg, scale = int(sys.argv[1]), float(sys.argv[2])
wl = bench.Batch(cfg, 0, 1, scale)
dev = DeviceCodec(0)
wl.setup(dev, torch)
d_sz = torch.zeros(wl.nseg, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, fn in (("sizes", lambda: dev.encoded_sizes_batch(wl.d_esegs, wl.nseg, wl.d_v, d_sz, delta=True)),
                 ("encode", wl.encode)):
    ts = []
    for it in range(6):
        flush.fill_(it)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if it >= 2:
            ts.append(e0.elapsed_time(e1))
    print(f"cfg{cfg} {name}: {sorted(ts)[len(ts) // 2]:.3f} ms")
dev.check()
assert torch.equal(d_sz, wl.d_lens)
