"""Dev tool: time the batch encode/decode of cfg4/cfg5 (optionally scaled) under debug flags.
Usage: python tools/sweep_batch.py CFG SCALE FLAGS..."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1709_08990_b200._native import lib  # noqa: E402
from paper_1709_08990_b200.device import DeviceCodec  # noqa: E402

cfg, scale = int(sys.argv[1]), float(sys.argv[2])
wl = bench.Batch(cfg, 0, 1, scale)
dev = DeviceCodec(0)
wl.setup(dev, torch)
lib.bcgpu_debug_set_flags.argtypes = [C.c_void_p, C.c_uint32]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
drain = torch.ones(64 << 20, dtype=torch.int32, device="cuda")
ref = wl.d_lens.clone()
for arg in sys.argv[3:]:
    flags = int(arg, 0)
    lib.bcgpu_debug_set_flags(dev._ctx, flags)
    te, td = [], []
    for it in range(6):
        for fn, ts in ((wl.encode, te), (wl.decode, td)):
            flush.fill_(it)
            drain.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if it >= 2:
                ts.append(e0.elapsed_time(e1))
    dev.check()
    bad = (wl.d_o != wl.d_v).nonzero().flatten()
    ok = (int(bad.numel()), int(bad[0]) if bad.numel() else -1, torch.equal(wl.d_lens, ref))
    print(f"cfg{cfg} x{scale} flags=0x{flags:04x} encode {np.median(te):7.3f} ms  decode {np.median(td):7.3f} ms  ok={ok}")
lib.bcgpu_debug_set_flags(dev._ctx, 0)
