"""Dev tool: per-tile phase timestamps of the single-array decode kernel (%globaltimer).

Phases (svb_decode_ct_kernel): 0 start, 1 ctrl+scan done, 2 offset look-back done,
3 data staged, 4 expanded, 5 sums synced, 6 carry look-back done, 7 stored."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1709_08990_b200 import gen  # noqa: E402
from paper_1709_08990_b200._native import lib  # noqa: E402
from paper_1709_08990_b200.device import DeviceCodec  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nostore = len(sys.argv) > 2 and sys.argv[2] == "nostore"
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
tiles = (n + 8191) // 8192
trace = torch.zeros(tiles * 8, dtype=torch.int64, device="cuda")
lib.bcgpu_debug_set_flags.argtypes = [C.c_void_p, C.c_uint32]
f = lib.bcgpu_debug_set_trace
f.argtypes = [C.c_void_p, C.c_void_p]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(4):
    flush.fill_(it)
    f(dev._ctx, trace.data_ptr() if it == 3 else None)
    lib.bcgpu_debug_set_flags(dev._ctx, 1 if nostore else 0)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    dev.decode(d_c, n, d_o, in_len=m, delta=delta)
    ev1.record()
    torch.cuda.synchronize()
    print(f"iter {it}: {ev0.elapsed_time(ev1) * 1e3:.1f} us")
f(dev._ctx, None)
lib.bcgpu_debug_set_flags(dev._ctx, 0)
if not nostore:
    assert torch.equal(d_o, d_v)
t = trace.cpu().numpy().reshape(tiles, 8).astype(np.int64)
t0 = t[:, 0].min()
names = ["ctrl+scan", "offset-lookback", "stage(TMA)", "expand", "sum-sync", "carry-lookback", "store"]
cols = [1, 2, 3, 4, 5, 6, 7] if delta else [1, 2, 3, 4, 7]
prev = 0
print(f"tiles={tiles} kernel span={(t[:, 7].max() - t0) / 1e3:.1f} us")
for c in cols:
    d = (t[:, c] - t[:, prev]) / 1e3
    print(f"  {names[c - 1]:16s} p50={np.median(d):7.2f} us  p90={np.percentile(d, 90):7.2f}  max={d.max():7.2f}")
    prev = c
life = (t[:, 7] - t[:, 0]) / 1e3
print(f"  lifetime p50={np.median(life):.2f} us p90={np.percentile(life, 90):.2f}")
starts = np.sort(t[:, 0] - t0) / 1e3
print("  start times (us) of tiles 0,100,500,1000,4000,last:", [round(float(starts[i]), 1) for i in [0, 100, 500, 1000, 4000, -1] if i < len(starts)])
# concurrency: tiles alive at the middle of the kernel
mid = t0 + (t[:, 7].max() - t0) // 2
print("  alive at mid:", int(((t[:, 0] <= mid) & (t[:, 7] >= mid)).sum()))
# order check: does tile i start after tile i-1?
print("  start-order inversions:", int((np.diff(t[:, 0]) < 0).sum()))
if not delta:
    sp, rd = t[:, 5] & 0xFFFFFFFF, t[:, 6] & 0xFFFFFFFF
    pr = (t[:, 5] >> 32) / 1e3
    print(f"  private strong-load probe (us): p50={np.median(pr):.2f} p90={np.percentile(pr, 90):.2f}")
    fp = (t[:, 6] >> 32) / 1e3
    print(f"  first poll round trip (us): p50={np.median(fp):.2f} p90={np.percentile(fp, 90):.2f}")
    print(f"  offset look-back spins p50={np.median(sp)} p90={np.percentile(sp, 90)} max={sp.max()}; "
          f"rounds p50={np.median(rd)} p90={np.percentile(rd, 90)} max={rd.max()}")
    ctrl_end = t[:, 1]
    late = (ctrl_end[:-1] - ctrl_end[1:]) / 1e3
    print(f"  pred ctrl-done minus own ctrl-done: p50={np.median(late):.2f} us p90={np.percentile(late, 90):.2f} max={late.max():.2f}")
    lag = (t[:, 2] - t[:, 1]) / 1e3
    ok = sp == 0
    print(f"  look-back time when no spin needed: p50={np.median(lag[ok]) if ok.any() else -1:.2f} us (n={ok.sum()})")
