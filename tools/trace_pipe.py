"""Dev tool: per-sub-tile timestamps of the pipelined decode (issue, wait-begin, wait-end, done)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1709_08990_b200 import gen  # noqa: E402
from paper_1709_08990_b200._native import lib  # noqa: E402
from paper_1709_08990_b200.device import DeviceCodec  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
delta = cfg == 2
v = gen.config_array(cfg)
n = v.size
dev = DeviceCodec(0)
d_v = torch.from_numpy(v.view(np.int32)).cuda()
d_c = torch.empty((n + 3) // 4 + 4 * n, dtype=torch.uint8, device="cuda")
d_len = torch.zeros(1, dtype=torch.int64, device="cuda")
dev.encode(d_v, d_c, d_len, delta=delta)
m = int(d_len.item())
d_o = torch.empty_like(d_v)
nsub = ((n + 3) // 4 + 255) // 256
trace = torch.zeros(nsub * 4, dtype=torch.int64, device="cuda")
lib.bcgpu_debug_set_trace.argtypes = [C.c_void_p, C.c_void_p]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(4):
    flush.fill_(it)
    lib.bcgpu_debug_set_trace(dev._ctx, trace.data_ptr() if it == 3 else None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dev.decode(d_c, n, d_o, in_len=m, delta=delta)
    e1.record()
    torch.cuda.synchronize()
    print(f"iter {it}: {e0.elapsed_time(e1) * 1e3:.1f} us")
lib.bcgpu_debug_set_trace(dev._ctx, None)
assert torch.equal(d_o, d_v)
t = trace.cpu().numpy().reshape(nsub, 4).astype(np.int64)
ok = t[:, 0] > 0
lat = (t[ok, 2] - t[ok, 0]) / 1e3
wait = (t[:, 2] - t[:, 1]) / 1e3
comp = (t[:, 3] - t[:, 2]) / 1e3
for nm, a in [("issue->data ready", lat), ("exposed wait", wait), ("compute+store", comp)]:
    print(f"  {nm:18s} p50={np.median(a):.2f} us p90={np.percentile(a, 90):.2f} mean={a.mean():.2f}")
