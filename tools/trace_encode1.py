"""Dev tool: per-tile timeline of the one-pass encode (svb_encode1_kernel, %globaltimer).
Usage: python tools/trace_encode1.py CFG [FLAGS]   (cfg3 needs FLAGS 0x1000: one-pass plain)
Per tile (thread 0 / warp 0 / scanner): 0 producer issued the input copy, 1 consumers start
waiting for it, 2 input landed, 3 tile aggregate published (scanner), 4 offset posted
(scanner, one round later), 6/7 consumer starts/ends waiting for that offset, 5 stored."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1709_08990_b200 import gen  # noqa: E402
from paper_1709_08990_b200._native import lib  # noqa: E402
from paper_1709_08990_b200.device import DeviceCodec  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
flags = int(sys.argv[2], 0) if len(sys.argv) > 2 else 0
delta = cfg == 2
v = gen.config_array(cfg)
n = v.size
dev = DeviceCodec(0)
lib.bcgpu_debug_set_flags.argtypes = [C.c_void_p, C.c_uint32]
lib.bcgpu_debug_set_flags(dev._ctx, flags)
d_v = torch.from_numpy(v.view(np.int32)).cuda()
d_c = torch.empty((n + 3) // 4 + 4 * n, dtype=torch.uint8, device="cuda")
d_len = torch.zeros(1, dtype=torch.int64, device="cuda")
tiles = (n + 8191) // 8192
trace = torch.zeros(tiles * 8, dtype=torch.int64, device="cuda")
f = lib.bcgpu_debug_set_trace
f.argtypes = [C.c_void_p, C.c_void_p]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
drain = torch.ones(64 << 20, dtype=torch.int32, device="cuda")
for it in range(4):
    flush.fill_(it)
    drain.sum()
    f(dev._ctx, trace.data_ptr() if it == 3 else None)
    dev.encode(d_v, d_c, d_len, delta=delta)
    torch.cuda.synchronize()
f(dev._ctx, None)
t = trace.cpu().numpy().reshape(tiles, 8).astype(np.int64)
t0 = t[:, 0][t[:, 0] > 0].min()
print(f"cfg{cfg} tiles={tiles} span={(t[:, 5].max() - t0) / 1e3:.1f} us")
for name, a, b in [("issue->landed", 0, 2), ("wait for data", 1, 2), ("landed->published", 2, 3),
                   ("published->offset", 3, 4), ("consumer waits offset", 6, 7), ("offset->stored", 7, 5),
                   ("landed->stored", 2, 5)]:
    d = (t[:, b] - t[:, a]) / 1e3
    print(f"  {name:22s} p10={np.percentile(d, 10):6.2f} p50={np.median(d):6.2f} p90={np.percentile(d, 90):6.2f} max={d.max():6.2f} us")
print("  stored times (us) at 10/50/90%:", np.percentile((t[:, 5] - t0) / 1e3, [10, 50, 90]).round(2))
