"""Dev tool: batched seek / select throughput on the cfg2 stream (64M sorted ints), device API."""
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
rng = np.random.default_rng(1)
for q in (1, 1 << 10, 1 << 20):
    tg = torch.from_numpy(rng.integers(0, int(v[-1]), q, dtype=np.int64).astype(np.uint32).view(np.int32)).cuda()
    ix = torch.from_numpy(rng.integers(0, n, q, dtype=np.int64)).cuda()
    oi = torch.empty(q, dtype=torch.int64, device="cuda")
    ov = torch.empty(q, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for name, fn in (("seek", lambda: lib.bcgpu_svb_seek_batch_device(dev._ctx, d_c.data_ptr(), m, n, 0, tg.data_ptr(), q,
                                                                       oi.data_ptr(), ov.data_ptr(), s)),
                     ("select", lambda: lib.bcgpu_svb_select_batch_device(dev._ctx, d_c.data_ptr(), m, n, 0,
                                                                           ix.data_ptr(), q, ov.data_ptr(), s))):
        for _ in range(3):
            assert fn() == 0
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"{name:6s} q={q:8d}: {ms * 1e3:8.1f} us per call (metadata pass + queries), {q / ms / 1e3:8.2f} Mqueries/s")
    if q == 1 << 20:
        got = oi.cpu().numpy()
        want = np.searchsorted(v, tg.cpu().numpy().view(np.uint32), side="left")
        assert np.array_equal(got, want), "seek mismatch"
        assert np.array_equal(ov.cpu().numpy().view(np.uint32), v[ix.cpu().numpy()]), "select mismatch"
print("verified")
