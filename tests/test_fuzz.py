"""Randomised parity: hypothesis draws sizes, value shapes, delta/prev and buffer offsets (and, for
batches, segment lengths, layouts and ring sizes), and
every encode / decode path the library dispatches between (one-pass, slot, two-read, sums +
pooled decode) must reproduce the pinned oracle byte for byte."""
import ctypes as C
import os

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle

pytestmark = pytest.mark.gpu

# debug flags of the ctx (bcgpu_capi.cu): which path runs
ENCODE_PATHS = {"default": 0, "two_read": 16, "slots": 32, "one_pass_plain": 4096, "two_read_plain": 0x80000,
                "scanner_delta": 0x100000}
DECODE_PATHS = {"default": 0, "sums_pooled": 0x400, "scan_dense": 0x400000}


@pytest.fixture(scope="module")
def env():
    import torch
    from paper_1709_08990_b200._native import lib
    from paper_1709_08990_b200.device import DeviceCodec
    lib.bcgpu_debug_set_flags.argtypes = [C.c_void_p, C.c_uint32]
    return torch, lib, DeviceCodec(0)


def _values(kind, n, seed):
    rng = np.random.default_rng(seed)
    if kind == "classes":
        k = rng.integers(0, 4, n)
        return (rng.integers(0, 2**32, n, dtype=np.uint64) >> (8 * (3 - k)).astype(np.uint64)).astype(np.uint32)
    if kind == "sorted_small":
        return np.cumsum(rng.integers(0, 200, n, dtype=np.uint64)).astype(np.uint32)
    if kind == "sorted_wide":
        return np.cumsum(rng.integers(0, 1 << 22, n, dtype=np.uint64)).astype(np.uint32)  # wraps mod 2^32
    if kind == "constant":
        return np.full(n, rng.integers(0, 2**32), np.uint32)
    return rng.integers(0, 256, n, dtype=np.uint64).astype(np.uint32)


@settings(max_examples=int(os.environ.get("FUZZ_EXAMPLES", "200")), deadline=None, suppress_health_check=list(HealthCheck))
@given(n=st.one_of(st.integers(0, 3000), st.integers(3000, 400_000), st.sampled_from([8192, 65536, 1 << 20])),
       kind=st.sampled_from(["classes", "sorted_small", "sorted_wide", "constant", "bytes"]),
       delta=st.booleans(), prev=st.integers(0, 2**32 - 1), seed=st.integers(0, 2**31),
       in_off=st.sampled_from([0, 1, 2, 3, 4]), out_off=st.integers(0, 17),
       enc=st.sampled_from(sorted(ENCODE_PATHS)), dec=st.sampled_from(sorted(DECODE_PATHS)))
def test_fuzz_roundtrip(env, n, kind, delta, prev, seed, in_off, out_off, enc, dec):
    torch, lib, dev = env
    v = _values(kind, n, seed)
    if not delta:
        prev = 0
    want = oracle.encode(v, delta=delta, prev=prev)
    src = torch.zeros(n + 8, dtype=torch.int32, device="cuda")
    if n:
        src[in_off:in_off + n] = torch.from_numpy(v.view(np.int32)).cuda()
    cap = (n + 3) // 4 + 4 * n
    outb = torch.zeros(cap + 32, dtype=torch.uint8, device="cuda")
    olen = torch.zeros(1, dtype=torch.int64, device="cuda")
    try:
        lib.bcgpu_debug_set_flags(dev._ctx, ENCODE_PATHS[enc])
        dev.encode(src[in_off:in_off + n], outb[out_off:out_off + cap], olen, delta=delta, prev=prev)
        dev.check()
        m = int(olen.item())
        assert m == len(want)
        assert outb[out_off:out_off + m].cpu().numpy().tobytes() == want
        lib.bcgpu_debug_set_flags(dev._ctx, DECODE_PATHS[dec])
        dst = torch.zeros(n + 8, dtype=torch.int32, device="cuda")
        last = torch.zeros(1, dtype=torch.int32, device="cuda")
        dev.decode(outb[out_off:out_off + m], n, dst[in_off:in_off + n], delta=delta, base=prev, last=last)
        dev.check()
        assert np.array_equal(dst[in_off:in_off + n].cpu().numpy().view(np.uint32), v)
        if delta:
            assert (int(last.item()) & 0xFFFFFFFF) == (int(v[-1]) if n else prev)
    finally:
        lib.bcgpu_debug_set_flags(dev._ctx, 0)


def _status(P, fn):
    """0 when fn() succeeds, else the bcgpu status of the CodecError (errc + 1)."""
    try:
        fn()
        return 0
    except P.CodecError as e:
        return int(e.code) + 1


@settings(max_examples=int(os.environ.get("FUZZ_EXAMPLES", "200")), deadline=None, suppress_health_check=list(HealthCheck))
@given(n=st.one_of(st.integers(0, 3000), st.integers(3000, 300_000)),
       kind=st.sampled_from(["classes", "sorted_small", "sorted_wide", "constant", "bytes"]),
       delta=st.booleans(), seed=st.integers(0, 2**31), in_off=st.sampled_from([0, 1, 3]),
       out_off=st.integers(0, 17))
def test_fuzz_varint_gb(env, n, kind, delta, seed, in_off, out_off):
    """varint-GB (svb_gb.cu) through the device API at any buffer offsets, against the oracle."""
    torch, lib, dev = env
    v = _values(kind, n, seed)
    payload = oracle.delta_encode(v, 0) if delta else v
    want = oracle.gb_encode(payload)
    src = torch.zeros(n + 8, dtype=torch.int32, device="cuda")
    if n:
        src[in_off:in_off + n] = torch.from_numpy(v.view(np.int32)).cuda()
    cap = (n + 3) // 4 + 4 * n
    outb = torch.zeros(cap + 32, dtype=torch.uint8, device="cuda")
    olen = torch.zeros(1, dtype=torch.int64, device="cuda")
    dev.gb_encode(src[in_off:in_off + n], outb[out_off:out_off + cap], olen, delta=delta)
    dev.check()
    m = int(olen.item())
    assert m == len(want) and outb[out_off:out_off + m].cpu().numpy().tobytes() == want
    dst = torch.zeros(n + 8, dtype=torch.int32, device="cuda")
    dev.gb_decode(outb[out_off:out_off + m], n, dst[in_off:in_off + n], delta=delta)
    dev.check()
    assert np.array_equal(dst[in_off:in_off + n].cpu().numpy().view(np.uint32), v)


@settings(max_examples=int(os.environ.get("FUZZ_EXAMPLES", "200")), deadline=None, suppress_health_check=list(HealthCheck))
@given(n=st.one_of(st.integers(1, 60_000), st.integers(60_000, 300_000)),
       kind=st.sampled_from(["classes", "sorted_small", "bytes"]),
       codec=st.sampled_from(["svb", "gb"]), delta=st.booleans(), seed=st.integers(0, 2**31),
       edit=st.sampled_from(["flip", "cut", "extend", "count_up", "count_down"]), where=st.floats(0, 1))
def test_fuzz_malformed(env, n, kind, codec, delta, seed, edit, where):
    """Corrupted streams: the GPU's status equals the oracle's (ok / truncated / trailing_bytes),
    and when both accept the stream they decode the same integers -- no read past the buffer
    changes either (the buffer is copied to an exact-size host array first)."""
    import paper_1709_08990_b200 as P
    v = _values(kind, n, seed)
    rng = np.random.default_rng(seed ^ 0x5A5A)
    enc = oracle.encode(v) if codec == "svb" else oracle.gb_encode(v)
    b = bytearray(enc)
    n2 = n
    if edit == "flip":
        i = min(int(where * len(b)), len(b) - 1)
        b[i] ^= 1 << int(rng.integers(0, 8))
    elif edit == "cut":
        b = b[: int(where * len(b))]
    elif edit == "extend":
        b += bytes(rng.integers(0, 256, 1 + int(where * 20)).astype(np.uint8))
    elif edit == "count_up":
        n2 = n + 1 + int(where * 7)
    else:
        n2 = max(0, n - 1 - int(where * 7))
    data = bytes(b)
    if codec == "svb":
        ost, ovals, _ = oracle.decode(data, n2, delta=delta)
    else:
        ost, ovals, _ = oracle.gb_decode(data, n2, delta=delta)
    out = np.zeros(max(n2, 1), np.uint32)
    if codec == "svb":
        gst = _status(P, (lambda: P.svb_decode_delta(data, n2, 0, out)) if delta else (lambda: P.svb_decode(data, n2, out)))
    else:
        gst = _status(P, (lambda: P.gb_decode_delta(data, n2, 0, out)) if delta else (lambda: P.gb_decode(data, n2, out)))
    assert gst == ost, (codec, edit, gst, ost)
    if ost == oracle.OK:
        assert np.array_equal(out[:n2], ovals[:n2])


@settings(max_examples=int(os.environ.get("FUZZ_EXAMPLES", "200")) // 2, deadline=None,
          suppress_health_check=list(HealthCheck))
@given(nseg=st.integers(1, 3000), long_frac=st.sampled_from([0.0, 0.01, 0.2, 1.0]),
       kind=st.sampled_from(["classes", "sorted_small", "sorted_wide", "constant", "bytes"]),
       delta=st.booleans(), seed=st.integers(0, 2**31), gap_in=st.booleans(), gap_out=st.booleans(),
       ring=st.sampled_from([0, 8, 11, 16]), occ=st.sampled_from([0, 1, 3]), hint=st.booleans())
def test_fuzz_batches(env, nseg, long_frac, kind, delta, seed, gap_in, gap_out, ring, occ, hint):
    """Segmented batches (segment-resident and tile-pipeline kernels) against the oracle: random
    segment lengths (short, the 1920 boundary, long), value shapes, stream / output gaps, ring
    sizes and CTA caps (many segments per warp, ring wrap-around)."""
    torch, lib, dev = env
    from paper_1709_08990_b200.device import DECODE_SEG_DTYPE, ENCODE_SEG_DTYPE, segments_to_tensor
    rng = np.random.default_rng(seed)
    if long_frac >= 1.0:
        nseg = min(nseg, 40)
    short = (rng.choice(np.array([0, 1, 2, 3, 4, 5, 127, 128, 129, 383, 384, 385, 1919, 1920]), nseg)
             if seed & 1 else rng.integers(0, 1921, nseg))
    sizes = np.where(rng.random(nseg) < long_frac, rng.integers(1921, 20_000, nseg), short).astype(np.int64)
    vals = [_values(kind, int(n), seed + i) for i, n in enumerate(sizes)]
    prevs = rng.integers(0, 2**32, nseg, dtype=np.uint64).astype(np.uint32) if delta else np.zeros(nseg, np.uint32)
    encs = [oracle.encode(v, delta=delta, prev=int(p)) for v, p in zip(vals, prevs)]
    gi = rng.integers(0, 5, nseg) if gap_in else np.zeros(nseg, np.int64)
    go = rng.integers(0, 17, nseg) if gap_out else np.zeros(nseg, np.int64)
    src = np.cumsum(gi + np.concatenate([[0], sizes[:-1]]))
    caps = (sizes + 3) // 4 + 4 * sizes
    dst = np.cumsum(go + np.concatenate([[0], caps[:-1]]))
    flat = np.zeros(int(src[-1] + sizes[-1]) + 4, np.uint32)
    for s_, v in zip(src, vals):
        flat[int(s_):int(s_) + v.size] = v
    es = np.zeros(nseg, ENCODE_SEG_DTYPE)
    es["src_offset"], es["dst_capacity"], es["dst_offset"], es["n"], es["prev"] = src, caps, dst, sizes, prevs
    d_out = torch.full((int(dst[-1] + caps[-1]) + 32,), 0x3C, dtype=torch.uint8, device="cuda")
    d_lens = torch.zeros(nseg, dtype=torch.int64, device="cuda")
    mx = int(sizes.max()) if hint else 0
    lib.bcgpu_debug_set_flags(dev._ctx, (ring << 24) | (ring << 16) | (occ << 12))
    try:
        dev.encode_batch(segments_to_tensor(es, "cuda"), nseg, torch.from_numpy(flat.view(np.int32)).cuda(), d_out,
                         d_lens, delta=delta, max_seg_n=mx)
        dev.check()
        got = d_out.cpu().numpy()
        assert np.array_equal(d_lens.cpu().numpy(), [len(e) for e in encs])
        for i, (e, d) in enumerate(zip(encs, dst)):
            assert got[int(d):int(d) + len(e)].tobytes() == e, f"encode segment {i} n={sizes[i]}"
        # decode the encoded streams where they lie (gaps between them), outputs at src offsets
        ds = np.zeros(nseg, DECODE_SEG_DTYPE)
        ds["src_offset"], ds["src_bytes"], ds["dst_offset"] = dst, [len(e) for e in encs], src
        ds["n"], ds["prev"] = sizes, prevs
        d_dec = torch.full((flat.size,), -5, dtype=torch.int32, device="cuda")
        dev.decode_batch(segments_to_tensor(ds, "cuda"), nseg, d_out, d_dec, delta=delta, max_seg_n=mx)
        dev.check()
        dec = d_dec.cpu().numpy().view(np.uint32)
        for i, (v, s_) in enumerate(zip(vals, src)):
            assert np.array_equal(dec[int(s_):int(s_) + v.size], v), f"decode segment {i} n={sizes[i]}"
    finally:
        lib.bcgpu_debug_set_flags(dev._ctx, 0)
