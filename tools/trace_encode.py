"""Dev tool: per-tile phase timestamps of the single-array encode kernel (%globaltimer).
Phases: 0 start, 1 input staged (TMA), 2 lengths+scan, 3 ctrl stored + packed, 4 CTA sync,
5 offset look-back done, 6 written out."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1709_08990_b200 import gen  # noqa: E402
from paper_1709_08990_b200._native import lib  # noqa: E402
from paper_1709_08990_b200.device import DeviceCodec  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
delta = cfg == 2
v = gen.config_array(cfg)
n = v.size
dev = DeviceCodec(0)
d_v = torch.from_numpy(v.view(np.int32)).cuda()
d_c = torch.empty((n + 3) // 4 + 4 * n, dtype=torch.uint8, device="cuda")
d_len = torch.zeros(1, dtype=torch.int64, device="cuda")
tiles = (n + 8191) // 8192
trace = torch.zeros(tiles * 8, dtype=torch.int64, device="cuda")
lib.bcgpu_debug_set_flags.argtypes = [C.c_void_p, C.c_uint32]
lib.bcgpu_debug_set_flags(dev._ctx, flags)
f = lib.bcgpu_debug_set_trace
f.argtypes = [C.c_void_p, C.c_void_p]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(4):
    flush.fill_(it)
    f(dev._ctx, trace.data_ptr() if it == 3 else None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dev.encode(d_v, d_c, d_len, delta=delta)
    e1.record()
    torch.cuda.synchronize()
    print(f"iter {it}: {e0.elapsed_time(e1) * 1e3:.1f} us")
f(dev._ctx, None)
t = trace.cpu().numpy().reshape(tiles, 8).astype(np.int64)
names = ["stage(TMA)", "lengths+scan", "ctrl-store+pack(+w0 look-back)", "cta-sync", "sync"]
for k in range(1, 6):
    d = (t[:, k] - t[:, k - 1]) / 1e3
    print(f"  {names[k - 1]:16s} p50={np.median(d):7.2f} us p90={np.percentile(d, 90):7.2f}")
st = t[1:, 7].astype(np.uint64)
polls = (st >> 56) & 0xFF
bad = (st >> 48) & 0xFF
first = ((st >> 24) & 0xFFFFFF) / 1e3
total = (st & 0xFFFFFF) / 1e3
for nm, a in [("polls", polls), ("bad polls", bad), ("first poll us", first), ("look-back us", total)]:
    a = a.astype(np.float64)
    print(f"  {nm:14s} p50={np.median(a):.2f} p90={np.percentile(a, 90):.2f} max={a.max():.2f}")
