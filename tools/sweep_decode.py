"""Dev tool: time the cfg2 delta decode under debug flag settings (stage count / pool factor
of the sums pass).  Usage: python tools/sweep_decode.py FLAGS..."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1709_08990_b200 import gen  # noqa: E402
from paper_1709_08990_b200._native import lib  # noqa: E402
from paper_1709_08990_b200.device import DeviceCodec  # noqa: E402

v = gen.config_array(2)
n = v.size
dev = DeviceCodec(0)
d_v = torch.from_numpy(v.view(np.int32)).cuda()
d_c = torch.empty((n + 3) // 4 + 4 * n, dtype=torch.uint8, device="cuda")
d_len = torch.zeros(1, dtype=torch.int64, device="cuda")
dev.encode(d_v, d_c, d_len, delta=True)
m = int(d_len.item())
d_o = torch.empty_like(d_v)
lib.bcgpu_debug_set_flags.argtypes = [C.c_void_p, C.c_uint32]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
drain = torch.ones(64 << 20, dtype=torch.int32, device="cuda")
for arg in sys.argv[1:]:
    flags = int(arg, 0)
    lib.bcgpu_debug_set_flags(dev._ctx, flags)
    ts = []
    for it in range(15):
        flush.fill_(it)
        drain.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dev.decode(d_c, n, d_o, in_len=m, delta=True)
        e1.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    ok = torch.equal(d_o, d_v)
    print(f"flags=0x{flags:06x} decode median {np.median(ts):7.1f} us  min {min(ts):7.1f}  ok={ok}")
lib.bcgpu_debug_set_flags(dev._ctx, 0)
