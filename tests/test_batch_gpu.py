"""GPU parity of the segmented batch kernels (codec.hpp:85-90 per segment; SPEC.md:555
chained chunks) against the pinned CPU oracle: short segments decode segment-resident
(svb_batch3.cu), long ones on the tile pipeline (svb_batch2.cu).  Covers every 16-B phase of
the input streams and every 4-B phase of the outputs, the n = 1920 / 1921 boundary between
the two kernels, gaps between streams, malformed segments (each errc the reference maps,
SURVEY.md §8(b)) and the max_seg_n contract.  Bit-exact: integer work, no tolerance."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

SMALL_N = 1920  # kBatchSmallN (svb_kernels.cuh)


@pytest.fixture(scope="module")
def dev():
    from paper_1709_08990_b200.device import DeviceCodec
    return DeviceCodec(0)


def _values(rng, n, delta, small=False):
    if small:  # every delta (or value) < 256: the all-one-byte encode path
        g = rng.integers(0, 256, n, dtype=np.uint64)
        return (np.cumsum(g) if delta else g).astype(np.uint32)
    if delta:
        gaps = rng.choice(np.array([1, 200, 70_000, 1 << 24], np.uint64), n, p=[0.4, 0.3, 0.2, 0.1])
        return np.cumsum(gaps * rng.integers(1, 3, n, dtype=np.uint64)).astype(np.uint32)
    k = rng.integers(0, 4, n)
    lo = np.where(k == 0, 0, 1 << (8 * k)).astype(np.uint64)
    span = ((1 << (8 * (k + 1))) - lo).astype(np.uint64)
    return (lo + rng.integers(0, 2**62, n, dtype=np.uint64) % span).astype(np.uint32)


def _layout(rng, sizes, encs, gap_in, gap_out):
    """Streams and outputs placed with random gaps (any 16-B / 4-B phase)."""
    src, dst, p, q = [], [], 0, 0
    for n, e in zip(sizes, encs):
        p += int(rng.integers(0, 33)) if gap_in else 0
        q += int(rng.integers(0, 7)) if gap_out else 0
        src.append(p)
        dst.append(q)
        p += len(e)
        q += n
    return np.array(src, np.uint64), np.array(dst, np.uint64), p, q


def _run(dev, sizes, delta, rng, *, gap_in=True, gap_out=True, hint=None, corrupt=None):
    import torch
    from paper_1709_08990_b200.device import DECODE_SEG_DTYPE, segments_to_tensor
    vals = [_values(rng, n, delta) for n in sizes]
    prevs = rng.integers(0, 2**32, len(sizes), dtype=np.uint64).astype(np.uint32)
    encs = [oracle.encode(v, delta=delta, prev=int(p)) for v, p in zip(vals, prevs)]
    src, dst, in_len, out_len = _layout(rng, sizes, encs, gap_in, gap_out)
    blob = np.full(in_len + 64, 0xA5, np.uint8)
    for s, e in zip(src, encs):
        blob[int(s):int(s) + len(e)] = np.frombuffer(e, np.uint8)
    segs = np.zeros(len(sizes), DECODE_SEG_DTYPE)
    segs["src_offset"], segs["src_bytes"] = src, [len(e) for e in encs]
    segs["dst_offset"], segs["n"], segs["prev"] = dst, sizes, prevs
    if corrupt is not None:
        corrupt(segs)
    d_in = torch.from_numpy(blob).cuda()
    sentinel = -7
    d_out = torch.full((out_len + 8,), sentinel, dtype=torch.int32, device="cuda")
    d_segs = segments_to_tensor(segs, "cuda")
    dev.decode_batch(d_segs, len(sizes), d_in, d_out, delta=delta,
                     max_seg_n=max(sizes) if hint is None else hint)
    return vals, dst, d_out, sentinel


def _check(dev, vals, dst, d_out, sentinel):
    dev.check()
    got = d_out.cpu().numpy()
    covered = np.zeros(got.size, bool)
    for v, d in zip(vals, dst):
        d = int(d)
        assert np.array_equal(got[d:d + v.size].view(np.uint32), v), f"segment at {d}, n={v.size}"
        covered[d:d + v.size] = True
    assert np.all(got[~covered] == sentinel), "write outside the segments' outputs"


@pytest.mark.parametrize("delta", [True, False])
def test_short_segments_every_phase(dev, delta):
    rng = np.random.default_rng(11 + delta)
    sizes = list(range(1, 140)) + list(rng.integers(1, SMALL_N + 1, 600))
    vals, dst, d_out, s = _run(dev, sizes, delta, rng)
    _check(dev, vals, dst, d_out, s)


@pytest.mark.parametrize("delta", [True, False])
def test_boundary_between_kernels(dev, delta):
    rng = np.random.default_rng(21 + delta)
    sizes = [SMALL_N - 1, SMALL_N, SMALL_N + 1, 1024, 1025, 4096 + 3, 96 * 4, 97 * 4, 128 * 3, 128 * 3 + 1,
             70_000, 1, 2, 3, 4] * 6
    rng.shuffle(sizes)
    for hint in (None, 0):
        vals, dst, d_out, s = _run(dev, sizes, delta, rng, hint=hint)
        _check(dev, vals, dst, d_out, s)


def test_contiguous_lists(dev):
    """cfg4 layout: streams back to back, outputs back to back."""
    from paper_1709_08990_b200 import gen
    rng = np.random.default_rng(5)
    lb = gen.posting_lists(4000, 9, cap_total=4000 * 1875)
    sizes = [int(x) for x in lb.lengths]
    vals, dst, d_out, s = _run(dev, sizes, True, rng, gap_in=False, gap_out=False)
    _check(dev, vals, dst, d_out, s)


def test_hint_contradicted_by_long_segment(dev):
    from paper_1709_08990_b200.codec import GpuError
    rng = np.random.default_rng(3)
    sizes = [100, 5000, 7]
    _run(dev, sizes, True, rng, hint=200)
    with pytest.raises(GpuError, match="(?i)invalid"):
        dev.check()


@pytest.mark.parametrize("which", ["short", "long"])
@pytest.mark.parametrize("kind", ["truncated_ctrl", "truncated_data", "trailing", "empty_with_bytes"])
def test_malformed_segment_status(dev, which, kind):
    from paper_1709_08990_b200.codec import CodecError, errc
    rng = np.random.default_rng(17)
    n_bad = 300 if which == "short" else 9000
    sizes = [50, n_bad, 2500, 9]

    def corrupt(segs):
        if kind == "truncated_ctrl":
            segs["src_bytes"][1] = (n_bad + 3) // 4 - 1
        elif kind == "truncated_data":
            segs["src_bytes"][1] -= 1
        elif kind == "trailing":
            segs["src_bytes"][1] += 1
        else:
            segs["n"][1] = 0
    _run(dev, sizes, True, rng, corrupt=corrupt, hint=0)
    with pytest.raises(CodecError) as ei:
        dev.check()
    want = errc.trailing_bytes if kind in ("trailing", "empty_with_bytes") else errc.truncated
    assert ei.value.code == want


@pytest.mark.parametrize("ring_kb", [0, 8, 9, 13])
def test_ring_wraps_many_segments_per_warp(dev, ring_kb):
    """~70 segments per warp (one CTA per SM via the debug occupancy cap), so every warp's
    ring wraps many times, including allocations that end exactly at the ring's end."""
    import ctypes as C
    from paper_1709_08990_b200._native import lib
    lib.bcgpu_debug_set_flags.argtypes = [C.c_void_p, C.c_uint32]
    rng = np.random.default_rng(100 + ring_kb)
    sizes = list(rng.choice(np.array([1, 5, 64, 700, 1500, 1920]), 40_000, p=[.1, .2, .2, .2, .2, .1]))
    lib.bcgpu_debug_set_flags(dev._ctx, (ring_kb << 16) | (1 << 12))
    try:
        vals, dst, d_out, s = _run(dev, sizes, True, rng, gap_in=False)
        _check(dev, vals, dst, d_out, s)
    finally:
        lib.bcgpu_debug_set_flags(dev._ctx, 0)


def _run_encode(dev, sizes, delta, rng, *, gap_in=True, gap_out=True, hint=None, cap_short=None, small=None):
    import torch
    from paper_1709_08990_b200.device import ENCODE_SEG_DTYPE, segments_to_tensor
    vals = [_values(rng, n, delta, small=small is not None and rng.random() < small) for n in sizes]
    prevs = rng.integers(0, 2**32, len(sizes), dtype=np.uint64).astype(np.uint32)
    want = [oracle.encode(v, delta=delta, prev=int(p)) for v, p in zip(vals, prevs)]
    caps = [(n + 3) // 4 + 4 * n for n in sizes]
    src, dst, p, q = [], [], 0, 0
    for n, c in zip(sizes, caps):
        p += int(rng.integers(0, 7)) if gap_in else 0
        q += int(rng.integers(0, 33)) if gap_out else 0
        src.append(p)
        dst.append(q)
        p += n
        q += c
    segs = np.zeros(len(sizes), ENCODE_SEG_DTYPE)
    segs["src_offset"], segs["dst_capacity"], segs["dst_offset"] = src, caps, dst
    segs["n"], segs["prev"] = sizes, prevs
    if cap_short is not None:
        segs["dst_capacity"][cap_short] -= 1
    flat = np.zeros(p + 4, np.uint32)
    for s_, v in zip(src, vals):
        flat[s_:s_ + v.size] = v
    d_in = torch.from_numpy(flat.view(np.int32)).cuda()
    d_out = torch.full((q + 64,), 0x5A, dtype=torch.uint8, device="cuda")
    d_lens = torch.full((len(sizes),), -1, dtype=torch.int64, device="cuda")
    dev.encode_batch(segments_to_tensor(segs, "cuda"), len(sizes), d_in, d_out, d_lens, delta=delta,
                     max_seg_n=max(sizes) if hint is None else hint)
    return want, dst, d_out, d_lens


def _check_encode(dev, want, dst, d_out, d_lens):
    dev.check()
    got = d_out.cpu().numpy()
    lens = d_lens.cpu().numpy()
    assert np.array_equal(lens, [len(w) for w in want])
    covered = np.zeros(got.size, bool)
    for i, (w, d) in enumerate(zip(want, dst)):
        assert got[d:d + len(w)].tobytes() == w, f"segment {i} n-bytes={len(w)} dst={d}"
        covered[d:d + len(w)] = True
    assert np.all(got[~covered] == 0x5A), "write outside the segments' streams"


@pytest.mark.parametrize("delta", [True, False])
def test_encode_short_segments_every_phase(dev, delta):
    rng = np.random.default_rng(31 + delta)
    sizes = list(range(1, 140)) + list(rng.integers(1, SMALL_N + 1, 600))
    _check_encode(dev, *_run_encode(dev, sizes, delta, rng))


@pytest.mark.parametrize("delta", [True, False])
def test_encode_boundary_between_kernels(dev, delta):
    rng = np.random.default_rng(41 + delta)
    sizes = [SMALL_N - 1, SMALL_N, SMALL_N + 1, 1024, 1025, 4096 + 3, 96 * 4, 97 * 4, 128 * 3, 128 * 3 + 1,
             70_000, 1, 2, 3, 4, 0] * 6
    rng.shuffle(sizes)
    for hint in (None, 0):
        _check_encode(dev, *_run_encode(dev, sizes, delta, rng, hint=hint))


def test_encode_small_values_and_wide_values(dev):
    """All-one-byte deltas, all-four-byte values, and alternating widths (every pack shape)."""
    import torch
    from paper_1709_08990_b200.device import ENCODE_SEG_DTYPE, segments_to_tensor
    rng = np.random.default_rng(7)
    vals = [np.arange(1000, dtype=np.uint32) * 3, np.full(777, 0xF1F2F3F4, np.uint32),
            np.tile(np.array([1, 300, 70000, 1 << 30], np.uint32), 300), rng.integers(0, 2**32, 1920, dtype=np.uint64).astype(np.uint32)]
    for delta in (False, True):
        want = [oracle.encode(v, delta=delta, prev=0) for v in vals]
        caps = [(v.size + 3) // 4 + 4 * v.size for v in vals]
        segs = np.zeros(len(vals), ENCODE_SEG_DTYPE)
        segs["src_offset"] = np.concatenate([[0], np.cumsum([v.size for v in vals])[:-1]])
        segs["dst_capacity"] = caps
        segs["dst_offset"] = np.concatenate([[0], np.cumsum(caps)[:-1]]) + 3
        segs["n"] = [v.size for v in vals]
        d_in = torch.from_numpy(np.concatenate(vals).view(np.int32)).cuda()
        d_out = torch.zeros(sum(caps) + 64, dtype=torch.uint8, device="cuda")
        d_lens = torch.zeros(len(vals), dtype=torch.int64, device="cuda")
        dev.encode_batch(segments_to_tensor(segs, "cuda"), len(vals), d_in, d_out, d_lens, delta=delta, max_seg_n=1920)
        dev.check()
        got = d_out.cpu().numpy()
        for w, d in zip(want, segs["dst_offset"]):
            assert got[int(d):int(d) + len(w)].tobytes() == w


def test_encode_capacity_too_small(dev):
    from paper_1709_08990_b200.codec import GpuError
    rng = np.random.default_rng(9)
    want, dst, d_out, d_lens = _run_encode(dev, [10, 500, 20], True, rng, cap_short=1, hint=0)
    with pytest.raises(GpuError, match="(?i)invalid"):
        dev.check()
    # the short segment writes nothing and reports length 0 (callers packing by the lengths
    # stay in bounds); the others are encoded as usual
    lens = d_lens.cpu().numpy()
    assert lens[1] == 0 and lens[0] == len(want[0]) and lens[2] == len(want[2])


@pytest.mark.parametrize("ring_kb", [0, 8, 9, 13, 23])
def test_encode_ring_wraps_many_segments_per_warp(dev, ring_kb):
    import ctypes as C
    from paper_1709_08990_b200._native import lib
    lib.bcgpu_debug_set_flags.argtypes = [C.c_void_p, C.c_uint32]
    rng = np.random.default_rng(200 + ring_kb)
    sizes = list(rng.choice(np.array([1, 5, 64, 700, 1500, 1920]), 40_000, p=[.1, .2, .2, .2, .2, .1]))
    lib.bcgpu_debug_set_flags(dev._ctx, (ring_kb << 24) | (1 << 12))
    try:
        _check_encode(dev, *_run_encode(dev, sizes, True, rng, gap_out=False))
    finally:
        lib.bcgpu_debug_set_flags(dev._ctx, 0)


@pytest.mark.parametrize("delta", [True, False])
def test_encode_one_byte_blocks(dev, delta):
    """Segments (and long-segment pieces) whose 384-integer blocks are all one-byte, at every
    data phase, including pieces that end exactly on a block (n = 384 k)."""
    rng = np.random.default_rng(51 + delta)
    sizes = [384, 768, 1152, 1536, 1920, 383, 385, 1024, 3 * 1024, 5000, 65536, 130_000, 7] * 4
    rng.shuffle(sizes)
    _check_encode(dev, *_run_encode(dev, sizes, delta, rng, small=0.8))


@pytest.mark.parametrize("delta", [True, False])
def test_many_segments_dynamic_chunks(dev, delta):
    """Batches with at least 32 segments per resident warp take the ticket path: warps draw
    chunks of 8 consecutive segments instead of a fixed stride (svb_batch3.cu).  160K segments
    of 0..300 integers (some empty, one long), every byte and every integer against the oracle,
    run twice on one context: the ticket words must be zero again after a launch."""
    import torch
    from paper_1709_08990_b200.device import DECODE_SEG_DTYPE, ENCODE_SEG_DTYPE, segments_to_tensor
    rng = np.random.default_rng(77 + delta)
    nseg = 160_000
    lens = rng.integers(0, 301, nseg).astype(np.uint32)
    lens[12345] = 5000  # one segment in pieces (encode) / on the tile pipeline (decode)
    offs = np.zeros(nseg + 1, np.uint64)
    np.cumsum(lens, out=offs[1:])
    n = int(offs[-1])
    vals = _values(rng, n, delta)
    prevs = rng.integers(0, 2**32, nseg, dtype=np.uint64).astype(np.uint32)
    caps = (lens.astype(np.uint64) + 3) // 4 + 4 * lens.astype(np.uint64)
    eoff = np.zeros(nseg + 1, np.uint64)
    np.cumsum(caps + rng.integers(0, 5, nseg).astype(np.uint64), out=eoff[1:])
    es = np.zeros(nseg, ENCODE_SEG_DTYPE)
    es["src_offset"], es["dst_capacity"], es["dst_offset"], es["n"], es["prev"] = offs[:-1], caps, eoff[:-1], lens, prevs
    want = np.full(int(eoff[-1]) + 16, 0xA5, np.uint8)
    want_lens = np.zeros(nseg, np.uint64)
    oracle.encode_batch(es, vals, want, want_lens, delta)
    d_es = segments_to_tensor(es, "cuda")
    d_v = torch.from_numpy(vals.view(np.int32)).cuda()
    for _ in range(2):
        d_c = torch.full((int(eoff[-1]) + 16,), 0xA5, dtype=torch.uint8, device="cuda")
        d_lens = torch.zeros(nseg, dtype=torch.int64, device="cuda")
        dev.encode_batch(d_es, nseg, d_v, d_c, d_lens, delta=delta)
        dev.check()
        assert np.array_equal(d_lens.cpu().numpy().astype(np.uint64), want_lens)
        assert np.array_equal(d_c.cpu().numpy(), want)
        ds = np.zeros(nseg, DECODE_SEG_DTYPE)
        ds["src_offset"], ds["src_bytes"], ds["dst_offset"], ds["n"], ds["prev"] = eoff[:-1], want_lens, offs[:-1], lens, prevs
        d_ds = segments_to_tensor(ds, "cuda")
        d_o = torch.full((n + 4,), -1, dtype=torch.int32, device="cuda")
        dev.decode_batch(d_ds, nseg, d_c, d_o, delta=delta)
        dev.check()
        got = d_o.cpu().numpy().view(np.uint32)
        assert np.array_equal(got[:n], vals)
        assert (got[n:] == 0xFFFFFFFF).all()
