"""GPU parity: the sm_100a kernels, called through the C ABI, against the pinned
CPU oracle on identical seeded inputs.  Bit-exact for compressed bytes and
decoded integers (integer/byte work: no tolerance)."""
import json

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1709_08990_b200 as P
    return P


@pytest.fixture(scope="module")
def dev():
    from paper_1709_08990_b200.device import DeviceCodec
    return DeviceCodec(0)


def _mixed(rng, n, classes=(0, 1, 2, 3)):
    k = rng.choice(np.array(classes), n)
    lo = np.where(k == 0, 0, 1 << (8 * k)).astype(np.uint64)
    span = ((1 << (8 * (k + 1))) - lo).astype(np.uint64)
    return (lo + (rng.integers(0, 2**62, n, dtype=np.uint64) % span)).astype(np.uint32)


def _check_roundtrip(P, v, delta=False, prev=0):
    want = oracle.encode(v, delta=delta, prev=prev)
    got = P.svb_encode_delta(v, prev) if delta else P.svb_encode(v)
    assert got == want, f"encode mismatch n={v.size} delta={delta}"
    out = np.empty(v.size, np.uint32)
    if delta:
        last = P.svb_decode_delta(want, v.size, prev, out)
        assert last == (int(v[-1]) if v.size else prev)
    else:
        P.svb_decode(want, v.size, out)
    assert np.array_equal(out, v), f"decode mismatch n={v.size} delta={delta}"


# ---- SPEC golden vectors through the reference-shaped API -------------------
def test_spec_vectors(P, golden_dir):
    spec = json.loads((golden_dir / "spec_vectors.json").read_text())
    for case in spec["encode"]["cases"]:
        assert list(P.svb_encode(np.array(case["values"], np.uint32))) == case["bytes"]
    for case in spec["decode"]["cases"]:
        assert list(P.svb_decode(bytes(case["bytes"]), case["n"])) == case["values"]
    for src, want in spec["delta_encode"]["cases"]:
        # delta encode of src with base 0 == plain encode of the deltas
        assert P.svb_encode_delta(np.array(src, np.uint32), 0) == oracle.encode(np.array(want, np.uint32))
    for src, base, want in spec["prefix_sum"]["cases"]:
        out = np.empty(4, np.uint32)
        last = P.svb_decode_delta(oracle.encode(np.array(src, np.uint32)), 4, base, out)
        assert list(out) == want and last == want[-1]
    buf = P.encode(P.codec_id.stream_vbyte, np.array([3, 7, 19, 20], np.uint32), delta=True)
    assert buf.count == 4 and buf.delta and list(P.decode(buf)) == [3, 7, 19, 20]


def test_size_identity_10_bits(P):
    v = np.random.default_rng(3).integers(128, 256, 1000, dtype=np.uint32)
    assert len(P.svb_encode(v)) * 8 / 1000 == 10.0


# ---- random property round trips (acceptance 1) ----------------
def test_random_roundtrips(P):
    rng = np.random.default_rng(42)
    sizes = list(range(0, 70)) + [127, 128, 129, 1000, 4095, 4096, 4097, 8191, 8192, 8193, 10000, 16383,
                                  16384, 16385, 24577, 65536, 100003]
    for i, n in enumerate(sizes):
        v = _mixed(rng, n)
        _check_roundtrip(P, v, delta=False)
        _check_roundtrip(P, v, delta=True, prev=int(rng.integers(0, 2**32)) if i % 2 else 0)


@pytest.mark.parametrize("classes", [(0,), (1,), (2,), (3,), (0, 3), (0, 1)])
def test_adversarial_classes(P, classes):
    """all-0x00 / all-0xFF / alternating control streams, every length boundary."""
    rng = np.random.default_rng(sum(classes) + 17)
    for n in (1, 3, 4, 5, 8191, 8192, 8193, 40000):
        _check_roundtrip(P, _mixed(rng, n, classes))
        _check_roundtrip(P, np.sort(_mixed(rng, n, classes)), delta=True)


def test_length_boundaries(P):
    b = []
    for e in (8, 16, 24):
        b += [(1 << e) - 2, (1 << e) - 1, 1 << e, (1 << e) + 1]
    v = np.array(b * 300 + [0, 1, 2**32 - 1], np.uint32)
    _check_roundtrip(P, v)
    _check_roundtrip(P, v, delta=True, prev=2**32 - 1)  # prev > x_0: wraps


def test_malformed(P):
    v = np.arange(1, 100000, 7, dtype=np.uint32) * 977
    enc = P.svb_encode(v)
    out = np.empty(v.size, np.uint32)
    with pytest.raises(P.CodecError) as e:
        P.svb_decode(enc[:-1], v.size, out)
    assert e.value.code == P.errc.truncated
    with pytest.raises(P.CodecError) as e:
        P.svb_decode(enc + b"\x00\x01", v.size, out)
    assert e.value.code == P.errc.trailing_bytes
    with pytest.raises(P.CodecError) as e:
        P.svb_decode(enc[:10], v.size, out)
    assert e.value.code == P.errc.truncated
    with pytest.raises(P.CodecError) as e:
        P.encode(P.codec_id.vbyte, v)
    assert e.value.code == P.errc.unsupported
    # a truncated stream cut deep inside: guarded reads, error reported
    with pytest.raises(P.CodecError):
        P.svb_decode(enc[: len(enc) // 2], v.size, out)


def test_host_pipeline_pieces(P):
    """Arrays large enough for the pipelined host API (pieces of 4 Mi integers streamed
    over PCIe): round trips, odd tail, and malformed streams still reported."""
    rng = np.random.default_rng(13)
    n = 9 * (1 << 20) + 4 * 65536 + 777
    v = np.cumsum(rng.integers(0, 3000, n, dtype=np.uint64)).astype(np.uint32)
    _check_roundtrip(P, v, delta=True, prev=7)
    w = _mixed(rng, n, (0, 1, 3))
    _check_roundtrip(P, w)
    enc = oracle.encode(v, delta=True, prev=7)
    out = np.empty(n, np.uint32)
    with pytest.raises(P.CodecError) as e:
        P.svb_decode_delta(enc[:-3], n, 7, out)
    assert e.value.code == P.errc.truncated
    with pytest.raises(P.CodecError) as e:
        P.svb_decode_delta(enc + b"\x05", n, 7, out)
    assert e.value.code == P.errc.trailing_bytes


# ---- device API: misaligned buffers, offsets, blocks -------------------------
def test_device_misaligned_pointers(P, dev):
    import torch
    rng = np.random.default_rng(8)
    for n in (5, 1001, 20011):
        v = _mixed(rng, n)
        want = oracle.encode(v, delta=True, prev=99)
        for shift_in in (0, 1, 4, 7):
            for shift_out in (0, 1, 3):
                src = torch.zeros(n + 8, dtype=torch.int32, device="cuda")
                src[shift_out:shift_out + n] = torch.from_numpy(v.view(np.int32)).cuda()
                cap = (n + 3) // 4 + 4 * n
                outb = torch.zeros(cap + 16, dtype=torch.uint8, device="cuda")
                olen = torch.zeros(1, dtype=torch.int64, device="cuda")
                dev.encode(src[shift_out:shift_out + n], outb[shift_in:shift_in + cap], olen, delta=True, prev=99)
                m = int(olen.item())
                assert m == len(want)
                assert outb[shift_in:shift_in + m].cpu().numpy().tobytes() == want
                # decode from a misaligned input into a misaligned output
                dec = torch.zeros(n + 8, dtype=torch.int32, device="cuda")
                last = torch.zeros(1, dtype=torch.int32, device="cuda")
                dev.decode(outb[shift_in:shift_in + m], n, dec[shift_out:shift_out + n], delta=True, base=99,
                           last=last)
                dev.check()
                assert np.array_equal(dec[shift_out:shift_out + n].cpu().numpy().view(np.uint32), v)
                assert (int(last.item()) & 0xFFFFFFFF) == int(v[-1])


@pytest.mark.parametrize("flags", [0, 0x400000])
def test_dense_delta_streams(dev, flags):
    """Dense delta streams (every delta < 256: ceil(n/4) + n bytes) decode without a control
    scan, with implicit offsets (flag 0x400000 forces the scan): exact against the oracle at
    every tile/sub-tile boundary and tail, through the device API, and a stream of dense
    length whose control bytes are not all zero is reported as truncated."""
    import ctypes as C
    import torch
    from paper_1709_08990_b200._native import lib
    lib.bcgpu_debug_set_flags.argtypes = [C.c_void_p, C.c_uint32]
    rng = np.random.default_rng(11)
    lib.bcgpu_debug_set_flags(dev._ctx, flags)
    try:
        for n in (1, 3, 4, 5, 1023, 1024, 1025, 8191, 8192, 8193, 65536 * 3 + 5, 2_500_001):
            prev = int(rng.integers(0, 2**32))
            v = (prev + np.cumsum(rng.integers(0, 256, n, dtype=np.uint64))).astype(np.uint32)
            enc = oracle.encode(v, delta=True, prev=prev)
            assert len(enc) == (n + 3) // 4 + n
            d_in = torch.from_numpy(np.frombuffer(enc, np.uint8).copy()).cuda()
            d_o = torch.zeros(n, dtype=torch.int32, device="cuda")
            d_last = torch.zeros(1, dtype=torch.int32, device="cuda")
            dev.decode(d_in, n, d_o, delta=True, base=prev, last=d_last)
            dev.check()
            assert np.array_equal(d_o.cpu().numpy().view(np.uint32), v), (n, flags)
            assert int(d_last.item()) & 0xFFFFFFFF == int(v[-1])
        # dense length, one control field non-zero (one delta >= 256, its stream cut by a byte)
        for n, at in ((100_000, 77_777), (9000, 8999), (8192 * 5, 3)):
            g = rng.integers(0, 256, n, dtype=np.uint64)
            g[at] = 300
            v = np.cumsum(g).astype(np.uint32)
            enc = oracle.encode(v, delta=True, prev=0)
            bad = np.frombuffer(enc[:-1], np.uint8).copy()
            assert bad.size == (n + 3) // 4 + n
            d_o = torch.zeros(n, dtype=torch.int32, device="cuda")
            dev.decode(torch.from_numpy(bad).cuda(), n, d_o, delta=True, base=0)
            with pytest.raises(Exception) as e:
                dev.check()
            assert "truncated" in str(e.value), (n, at, str(e.value))
    finally:
        lib.bcgpu_debug_set_flags(dev._ctx, 0)


@pytest.mark.parametrize("flags", [16, 32, 4096])
def test_encode_both_paths(dev, flags):
    """Every single-array encode path, whichever the dispatch picks for the stream kind:
    16 = size scan + tile encode (two reads), 32 = slot encode + compaction (one read),
    4096 = one-pass encode with deferred look-back (for plain streams too)."""
    import ctypes as C
    import torch
    from paper_1709_08990_b200._native import lib
    lib.bcgpu_debug_set_flags.argtypes = [C.c_void_p, C.c_uint32]
    rng = np.random.default_rng(5 + flags)
    lib.bcgpu_debug_set_flags(dev._ctx, flags)
    try:
        for n in (1, 5, 1023, 1024, 8193, 65536 + 7, 600_001, 5_000_003):
            for delta, v in ((False, _mixed(rng, n)), (True, np.sort(_mixed(rng, n, (0, 1, 2))))):
                prev = int(rng.integers(0, 2**32)) if delta else 0
                want = oracle.encode(v, delta=delta, prev=prev)
                src = torch.from_numpy(v.view(np.int32)).cuda()
                outb = torch.zeros((n + 3) // 4 + 4 * n, dtype=torch.uint8, device="cuda")
                olen = torch.zeros(1, dtype=torch.int64, device="cuda")
                dev.encode(src, outb, olen, delta=delta, prev=prev)
                dev.check()
                m = int(olen.item())
                assert m == len(want) and outb[:m].cpu().numpy().tobytes() == want, (n, delta, flags)
    finally:
        lib.bcgpu_debug_set_flags(dev._ctx, 0)


def test_block_offsets_and_random_access(P):
    rng = np.random.default_rng(21)
    for n in (1, 3, 4, 7, 8192 * 3 + 5, 100001):
        v = _mixed(rng, n)
        enc = oracle.encode(v)
        want = oracle.block_data_offsets(enc, n)
        got = P.svb_block_data_offsets(enc, n)
        assert np.array_equal(got, want)
        ks = rng.integers(0, len(want), min(2000, len(want)))
        vals, cnts = P.svb_decode_blocks(enc, n, ks, want[ks])
        for j, k in enumerate(ks):
            ref = oracle.decode_block(enc, n, int(k), int(want[k]))
            assert cnts[j] == len(ref) and list(vals[j, :cnts[j]]) == list(ref)
    assert list(P.svb_decode_block(oracle.encode(np.array([1, 2, 300], np.uint32)), 3, 0, 0)) == [1, 2, 300]
    # svb_decode_block's contract on host data: a block past ceil(n/4) is out_of_range, a block
    # whose bytes lie past the end of the stream is truncated
    enc3 = oracle.encode(np.array([1, 2, 300, 70000, 5], np.uint32))
    with pytest.raises(P.CodecError) as e:
        P.svb_decode_block(enc3, 5, 2, 0)
    assert e.value.code == P.errc.out_of_range
    with pytest.raises(P.CodecError) as e:
        P.svb_decode_block(enc3[:-2], 5, 1, 7)
    assert e.value.code == P.errc.truncated


# ---- BASELINE.json configs (scaled where the oracle needs it) ---------------
def test_config1_full(P):
    from paper_1709_08990_b200 import gen
    v = gen.config_array(1)  # 2^20, the reference's CPU-runnable config
    _check_roundtrip(P, v)


def test_config2_scaled(P):
    from paper_1709_08990_b200 import gen
    v = gen.config_array(2, 1 << 22)
    _check_roundtrip(P, v, delta=True, prev=0)


def test_encode_sliced_pipeline(P):
    """> 2 L2 slices of the encode pipeline (8 Mi integers each), odd tail, prev-seeded delta."""
    rng = np.random.default_rng(31)
    n = 3 * (1 << 23) + 12345 + 3
    v = _mixed(rng, n, (0, 1))
    _check_roundtrip(P, v)
    s = np.cumsum(rng.integers(0, 300, n, dtype=np.uint64)).astype(np.uint32)
    _check_roundtrip(P, s, delta=True, prev=123456789)


def test_delta_sums_paths(P):
    """Delta decode's sums pass: all-zero-control sub-tiles (byte sums) next to general ones,
    at every 16-B phase of the data start, across many pipeline rounds."""
    rng = np.random.default_rng(77)
    for n in (4 * 1024 + 4, 4 * 1024 + 8, 4 * 1024 + 12, 9 * 1024 + 44, 200 * 1024 + 4 * 13 + 3, 3_000_001):
        g = rng.integers(0, 200, n, dtype=np.uint64)
        sub = np.arange(n) // 1024
        big = (sub % 3 == 1) & (rng.random(n) < 0.01)  # every third sub-tile gets some wide gaps
        g[big] += rng.integers(256, 1 << 20, int(big.sum()), dtype=np.uint64)
        v = np.cumsum(g).astype(np.uint32)
        _check_roundtrip(P, v, delta=True, prev=int(rng.integers(0, 2**32)))


def test_config3_scaled(P):
    from paper_1709_08990_b200 import gen
    v = gen.config_array(3, 1 << 23)
    _check_roundtrip(P, v)


def _batch_decode_check(dev, values_list, prevs, delta, max_hint):
    import torch
    from paper_1709_08990_b200.device import DECODE_SEG_DTYPE, ENCODE_SEG_DTYPE, segments_to_tensor
    encs = [oracle.encode(v, delta=delta, prev=p) for v, p in zip(values_list, prevs)]
    nseg = len(values_list)
    segs = np.zeros(nseg, DECODE_SEG_DTYPE)
    src_off = np.concatenate([[0], np.cumsum([len(e) for e in encs])])
    dst_off = np.concatenate([[0], np.cumsum([v.size for v in values_list])])
    segs["src_offset"], segs["src_bytes"] = src_off[:-1], np.diff(src_off)
    segs["dst_offset"], segs["n"], segs["prev"] = dst_off[:-1], [v.size for v in values_list], prevs
    blob = np.frombuffer(b"".join(encs), np.uint8)
    d_in = torch.from_numpy(blob.copy()).cuda()
    d_out = torch.zeros(int(dst_off[-1]) + 1, dtype=torch.int32, device="cuda")
    d_segs = segments_to_tensor(segs, "cuda")
    dev.decode_batch(d_segs, nseg, d_in, d_out, delta=delta, max_seg_n=max_hint)
    dev.check()
    got = d_out.cpu().numpy().view(np.uint32)
    assert np.array_equal(got[: dst_off[-1]], np.concatenate(values_list))
    # encode batch into worst-case slots, then compare every segment's bytes
    esegs = np.zeros(nseg, ENCODE_SEG_DTYPE)
    caps = np.array([(v.size + 3) // 4 + 4 * v.size for v in values_list], np.uint64)
    eoff = np.concatenate([[0], np.cumsum(caps)])
    esegs["src_offset"], esegs["dst_capacity"], esegs["dst_offset"] = dst_off[:-1], caps, eoff[:-1]
    esegs["n"], esegs["prev"] = [v.size for v in values_list], prevs
    d_vals = torch.from_numpy(np.concatenate(values_list).view(np.int32).copy()).cuda()
    d_enc = torch.zeros(int(eoff[-1]) + 16, dtype=torch.uint8, device="cuda")
    d_lens = torch.zeros(nseg, dtype=torch.int64, device="cuda")
    d_esegs = segments_to_tensor(esegs, "cuda")
    dev.encode_batch(d_esegs, nseg, d_vals, d_enc, d_lens, delta=delta, max_seg_n=max_hint)
    d_sizes = torch.zeros(nseg, dtype=torch.int64, device="cuda")
    dev.encoded_sizes_batch(d_esegs, nseg, d_vals, d_sizes, delta=delta)
    dev.check()
    lens = d_lens.cpu().numpy()
    assert np.array_equal(lens, [len(e) for e in encs])
    assert np.array_equal(d_sizes.cpu().numpy(), lens)
    enc_host = d_enc.cpu().numpy()
    for i, e in enumerate(encs):
        assert enc_host[int(eoff[i]): int(eoff[i]) + len(e)].tobytes() == e, i


def test_batch_config4_scaled(dev):
    from paper_1709_08990_b200 import gen
    lb = gen.posting_lists(3000, 4, cap_total=3000 * 1875)
    lists = [lb.values[int(lb.offsets[i]):int(lb.offsets[i + 1])] for i in range(3000)]
    _batch_decode_check(dev, lists, [0] * len(lists), True, int(lb.lengths.max()))


def test_batch_config5_scaled(dev):
    from paper_1709_08990_b200 import gen
    seq = gen.geometric_sorted(24 * 65536, 32.0, 5)
    chunks = [seq[i * 65536:(i + 1) * 65536] for i in range(24)]
    prevs = [0] + [int(c[-1]) for c in chunks[:-1]]
    _batch_decode_check(dev, chunks, prevs, True, 65536)


def test_batch_many_segments(dev):
    """Thousands of posting lists per warp pipeline (tile and segment hand-offs, every
    control-byte pattern of multi-byte gaps) through both batch kernels, bytes vs the oracle."""
    from paper_1709_08990_b200 import gen
    lb = gen.posting_lists(12000, 9, cap_total=12000 * 1500)
    lists = [lb.values[int(lb.offsets[i]):int(lb.offsets[i + 1])] for i in range(12000)]
    _batch_decode_check(dev, lists, [0] * len(lists), True, int(lb.lengths.max()))


def test_batch_mixed_sizes(dev):
    rng = np.random.default_rng(77)
    sizes = [0, 1, 2, 3, 4, 5, 31, 128, 129, 4095, 4096, 4097, 5000, 8192, 8193, 20000, 70001, 17, 3]
    lists = [_mixed(rng, int(n)) for n in sizes]
    prevs = [int(rng.integers(0, 2**32)) for _ in sizes]
    _batch_decode_check(dev, lists, prevs, True, 0)
    _batch_decode_check(dev, lists, [0] * len(sizes), False, max(sizes))


# ---- full BASELINE sizes: size-independent properties -----------------------
@pytest.mark.slow
def test_config2_full_roundtrip(dev):
    """64M delta: GPU encode == O1 encode bytes (digest), GPU decode round trip exact."""
    import hashlib

    import torch
    from paper_1709_08990_b200 import gen
    v = gen.config_array(2)
    want = oracle.encode(v, delta=True, prev=0)
    d_v = torch.from_numpy(v.view(np.int32)).cuda()
    cap = (v.size + 3) // 4 + 4 * v.size
    d_c = torch.empty(cap, dtype=torch.uint8, device="cuda")
    d_len = torch.zeros(1, dtype=torch.int64, device="cuda")
    dev.encode(d_v, d_c, d_len, delta=True, prev=0)
    m = int(d_len.item())
    assert m == len(want)
    assert hashlib.sha256(d_c[:m].cpu().numpy().tobytes()).hexdigest() == hashlib.sha256(want).hexdigest()
    d_o = torch.empty_like(d_v)
    dev.decode(d_c, v.size, d_o, in_len=m, delta=True, base=0)
    dev.check()
    assert torch.equal(d_o, d_v)


@pytest.mark.slow
def test_config3_full_roundtrip(dev):
    import hashlib

    import torch
    from paper_1709_08990_b200 import gen
    v = gen.config_array(3)
    want = oracle.encode(v)
    d_v = torch.from_numpy(v.view(np.int32)).cuda()
    cap = (v.size + 3) // 4 + 4 * v.size
    d_c = torch.empty(cap, dtype=torch.uint8, device="cuda")
    d_len = torch.zeros(1, dtype=torch.int64, device="cuda")
    dev.encode(d_v, d_c, d_len)
    m = int(d_len.item())
    assert m == len(want)
    assert hashlib.sha256(d_c[:m].cpu().numpy().tobytes()).hexdigest() == hashlib.sha256(want).hexdigest()
    d_o = torch.empty_like(d_v)
    dev.decode(d_c, v.size, d_o, in_len=m)
    dev.check()
    assert torch.equal(d_o, d_v)


def _slot_bytes(buf, eoff, lens, a, b):
    """Concatenated stream bytes of segments [a, b) of a worst-case-slot layout
    (segment s at eoff[s], lens[s] bytes)."""
    ln = lens[a:b].astype(np.int64)
    pk = np.zeros(b - a, np.int64)
    np.cumsum(ln[:-1], out=pk[1:])
    idx = np.arange(int(ln.sum()), dtype=np.int64) + np.repeat(eoff[a:b].astype(np.int64) - pk, ln)
    return buf[idx]


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [4, 5])
def test_batch_full_config(P, dev, cfg):
    """Full BASELINE.json sizes of the batch configs (cfg4: 1M posting lists, ~2^30 integers;
    cfg5: 2^31 integers in 64K-integer chunks with chained prev seeds), EVERY segment:
    - the device batch kernels (bench's timed path, worst-case slots): each segment's stream
      length and bytes equal oracle.encode_batch's, the total compressed size too, and the
      device decode round trip is exact;
    - the host batch C-ABI (packed streams): the same bytes back to back, offsets = the
      exclusive scan of the oracle's lengths, and its decode returns the input."""
    import torch

    import bench
    wl = bench.Batch(cfg, 0, 1, 1.0)
    wl.setup(dev, torch)
    wl.decode()
    torch.cuda.synchronize()
    wl.verify(torch)
    es, eoff = wl.host_segments()
    want = np.zeros(int(eoff[-1]) + 16, np.uint8)
    lens = np.zeros(wl.nseg, np.uint64)
    assert oracle.encode_batch(es, wl.values, want, lens, True) == oracle.OK
    assert np.array_equal(wl.enc_lens, lens), "a segment's stream length differs from the oracle's"
    assert wl.cmp == int(lens.sum())
    got = wl.d_c.cpu().numpy()
    wl.release()
    torch.cuda.empty_cache()
    step = 4096
    for a in range(0, wl.nseg, step):
        b = min(wl.nseg, a + step)
        assert np.array_equal(_slot_bytes(got, eoff, lens, a, b), _slot_bytes(want, eoff, lens, a, b)), (a, b)
    del got
    packed, offs = P.svb_encode_batch(wl.values, wl.lens, wl.prevs)
    assert offs[0] == 0 and np.array_equal(np.diff(offs), lens)
    for a in range(0, wl.nseg, step):
        b = min(wl.nseg, a + step)
        assert np.array_equal(packed[int(offs[a]):int(offs[b])], _slot_bytes(want, eoff, lens, a, b)), (a, b)
    del want
    dec = P.svb_decode_batch(packed, offs, wl.lens, wl.prevs)
    assert np.array_equal(dec, wl.values)
