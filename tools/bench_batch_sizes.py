"""Dev tool: batch encode/decode time vs segment length (fixed total integers), to separate the
per-segment cost from the per-integer cost.  Usage: python tools/bench_batch_sizes.py [TOTAL_M] L..."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1709_08990_b200.device import DECODE_SEG_DTYPE, ENCODE_SEG_DTYPE, DeviceCodec, segments_to_tensor  # noqa

total = int(float(sys.argv[1]) * (1 << 20))
dev = DeviceCodec(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=5):
    ts = []
    for it in range(reps + 2):
        flush.fill_(it)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if it >= 2:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


for L in map(int, sys.argv[2:]):
    nseg = total // L
    n = nseg * L
    rng = np.random.default_rng(L)
    gaps = rng.integers(1, 1 << 15, n, dtype=np.uint64).astype(np.uint32)  # ~2-byte deltas
    vals = np.cumsum(gaps.reshape(nseg, L), axis=1, dtype=np.uint64).astype(np.uint32).ravel()
    lens = np.full(nseg, L, np.uint64)
    cap = (L + 3) // 4 + 4 * L
    es = np.zeros(nseg, ENCODE_SEG_DTYPE)
    es["src_offset"] = np.arange(nseg, dtype=np.uint64) * L
    es["dst_capacity"], es["dst_offset"], es["n"] = cap, np.arange(nseg, dtype=np.uint64) * cap, L
    d_v = torch.from_numpy(vals.view(np.int32)).cuda()
    d_c = torch.empty(nseg * cap + 16, dtype=torch.uint8, device="cuda")
    d_l = torch.zeros(nseg, dtype=torch.int64, device="cuda")
    d_es = segments_to_tensor(es, "cuda")
    te = timed(lambda: dev.encode_batch(d_es, nseg, d_v, d_c, d_l, delta=True, max_seg_n=L))
    ls = d_l.cpu().numpy().astype(np.uint64)
    ds = np.zeros(nseg, DECODE_SEG_DTYPE)
    ds["src_offset"], ds["src_bytes"], ds["dst_offset"], ds["n"] = es["dst_offset"], ls, es["src_offset"], L
    d_ds = segments_to_tensor(ds, "cuda")
    d_o = torch.empty_like(d_v)
    td = timed(lambda: dev.decode_batch(d_ds, nseg, d_c, d_o, delta=True, max_seg_n=L))
    dev.check()
    assert torch.equal(d_o, d_v)
    cmp = float(ls.sum())
    roof = (cmp + 4 * n) / 6.55e12 * 1e3
    print(f"L={L:6d} nseg={nseg:8d} encode {te:7.3f} ms ({n / te / 1e6:6.1f} Gint/s, {te * 1e6 / nseg:7.1f} ns/seg, "
          f"frac {roof / te:.2f})  decode {td:7.3f} ms ({n / td / 1e6:6.1f} Gint/s, {td * 1e6 / nseg:7.1f} ns/seg, "
          f"frac {roof / td:.2f})")
