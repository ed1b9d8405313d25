"""The host-buffer batch entry points (bcgpu_svb_{encode,decode}_batch_host): one
C-ABI call per batch, the chained-chunk contract of the reference (codec.hpp:87-90,
decode_payload_delta once per chunk) for every segment.  Bit-exact against the
oracle per segment, across piece boundaries of the host pipeline, with the
reference's error semantics (truncated / trailing_bytes)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1709_08990_b200 as P
    return P


def _lists(rng, sizes, delta):
    vals, prevs = [], []
    acc = 0
    for n in sizes:
        prevs.append(acc & 0xFFFFFFFF)
        if delta:
            g = rng.integers(0, 3000, n, dtype=np.uint64)
            big = rng.random(n) < 0.01  # some 3- and 4-byte gaps
            g[big] += rng.integers(1 << 16, 1 << 30, int(big.sum()), dtype=np.uint64)
            v = ((acc + np.cumsum(g)) & 0xFFFFFFFF).astype(np.uint32)
            acc = int(v[-1]) if n else acc
        else:
            v = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32) >> rng.integers(0, 32, n).astype(np.uint32)
        vals.append(v)
    return vals, prevs


def oracle_packed(allv, ns, prevs, delta):
    """The oracle's streams of every segment, packed back to back: (bytes, offsets)."""
    from paper_1709_08990_b200.device import ENCODE_SEG_DTYPE
    ns64 = ns.astype(np.uint64)
    src = np.zeros(ns.size + 1, np.uint64)
    np.cumsum(ns64, out=src[1:])
    caps = (ns64 + 3) // 4 + 4 * ns64
    es = np.zeros(ns.size, ENCODE_SEG_DTYPE)
    es["src_offset"], es["n"], es["prev"] = src[:-1], ns, prevs
    es["dst_capacity"] = caps
    es["dst_offset"] = np.concatenate([[0], np.cumsum(caps)[:-1]]).astype(np.uint64)
    tmp = np.zeros(int(caps.sum()) + 16, np.uint8)
    lens = np.zeros(ns.size, np.uint64)
    oracle.encode_batch(es, allv, tmp, lens, delta)
    offs = np.zeros(ns.size + 1, np.uint64)
    np.cumsum(lens, out=offs[1:])
    es["dst_offset"], es["dst_capacity"] = offs[:-1], lens
    packed = np.zeros(int(offs[-1]) + 16, np.uint8)
    oracle.encode_batch(es, allv, packed, lens, delta)
    return packed[: int(offs[-1])], offs


def _check(P, vals, prevs, delta):
    ns = np.array([v.size for v in vals], np.uint32)
    prevs = np.array(prevs, np.uint32)
    allv = np.concatenate(vals) if vals else np.zeros(0, np.uint32)
    got, offs = P.svb_encode_batch(allv, ns, prevs, delta=delta)
    want, woffs = oracle_packed(allv, ns, prevs, delta)
    assert np.array_equal(offs, woffs), "segment stream lengths differ from the oracle"
    assert np.array_equal(got, want), "packed streams differ from the oracle"
    dec, last = P.svb_decode_batch(got, offs, ns, prevs, delta=delta, want_last=True)
    assert np.array_equal(dec, allv)
    ends = np.cumsum(ns.astype(np.int64)) - 1
    want_last = np.where(ns > 0, allv[np.maximum(ends, 0)] if allv.size else 0, prevs)
    assert np.array_equal(last, want_last.astype(np.uint32))


def test_small_batches(P):
    rng = np.random.default_rng(1)
    for sizes in ([1], [0], [0, 0, 3], [5, 0, 17, 1920, 1921, 4096, 65536, 3], list(rng.integers(0, 300, 500))):
        for delta in (True, False):
            vals, prevs = _lists(rng, [int(x) for x in sizes], delta)
            _check(P, vals, prevs, delta)


def test_many_pieces(P):
    """> 4M integers and > 1M segments: several pieces of the host pipeline (cut by
    integers and by segment count), long and short segments mixed."""
    rng = np.random.default_rng(2)
    sizes = list(rng.integers(0, 12, 1_200_000)) + [70_000, 1_000_000, 3_000_001, 5] + list(rng.integers(0, 5000, 3000))
    vals, prevs = _lists(rng, [int(x) for x in sizes], True)
    _check(P, vals, prevs, True)


def test_errors(P):
    rng = np.random.default_rng(3)
    vals, prevs = _lists(rng, [10, 20, 30], True)
    ns = np.array([10, 20, 30], np.uint32)
    b, offs = P.svb_encode_batch(np.concatenate(vals), ns, prevs)
    with pytest.raises(P.CodecError) as e:  # the batch's bytes end early
        P.svb_decode_batch(b[:-1], offs, ns, prevs)
    assert e.value.code == P.errc.truncated
    bad = offs.copy()
    bad[2] -= 1  # segment 1 one byte short, segment 2 one byte long
    with pytest.raises(P.CodecError) as e:
        P.svb_decode_batch(b, bad, ns, prevs)
    assert e.value.code in (P.errc.truncated, P.errc.trailing_bytes)
    with pytest.raises(P.GpuError):  # offsets must not decrease
        P.svb_decode_batch(b, offs[::-1].copy(), ns, prevs)
    with pytest.raises(P.GpuError):  # output capacity too small
        P.svb_encode_batch(np.concatenate(vals), ns, prevs, out=np.empty(10, np.uint8))
