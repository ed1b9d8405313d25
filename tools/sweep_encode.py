"""Dev tool: time the single-array encode under debug flag settings.  Usage:
python tools/sweep_encode.py CFG FLAGS...   (16: two-read path; 32|h<<6: slot path with L2 hints h)"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1709_08990_b200 import gen  # noqa: E402
from paper_1709_08990_b200._native import lib  # noqa: E402
from paper_1709_08990_b200.device import DeviceCodec  # noqa: E402

cfg = int(sys.argv[1])
delta = cfg == 2
v = gen.config_array(cfg)
n = v.size
dev = DeviceCodec(0)
d_v = torch.from_numpy(v.view(np.int32)).cuda()
d_c = torch.empty((n + 3) // 4 + 4 * n, dtype=torch.uint8, device="cuda")
d_len = torch.zeros(1, dtype=torch.int64, device="cuda")
lib.bcgpu_debug_set_flags.argtypes = [C.c_void_p, C.c_uint32]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
drain = torch.ones(64 << 20, dtype=torch.int32, device="cuda")
ref = None
for arg in sys.argv[2:]:
    flags = int(arg, 0)
    lib.bcgpu_debug_set_flags(dev._ctx, flags)
    ts = []
    for it in range(12):
        flush.fill_(it)
        drain.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dev.encode(d_v, d_c, d_len, delta=delta)
        e1.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    m = int(d_len.item())
    h = hash(bytes(d_c[:m].cpu().numpy()))
    ref = ref or h
    print(f"flags=0x{flags:04x} encode median {np.median(ts):7.1f} us  min {min(ts):7.1f}  same={h == ref}")
lib.bcgpu_debug_set_flags(dev._ctx, 0)
