"""Batched seek / select on the GPU (svb_query.cu) against the decode-everything-then-scan
oracle (seek/select agree with it on every query; ties -> lowest index)."""
import numpy as np
import pytest

import oracle
import paper_1709_08990_b200 as P

pytestmark = pytest.mark.gpu


def _delta_buf(values):
    v = np.asarray(values, np.uint32)
    d = np.diff(v, prepend=np.uint32(0)).astype(np.uint32)
    return P.EncodedBuffer(P.codec_id.stream_vbyte, int(v.size), True, oracle.encode(d))


def test_spec_examples():
    b = _delta_buf([3, 7, 19, 20])
    assert P.seek(b, 8) == (2, 19)
    assert P.seek(b, 3) == (0, 3)
    assert P.seek(b, 21) is None
    assert P.select(b, 1) == 7 and P.select(b, 0) == 3 and P.select(b, 3) == 20


@pytest.mark.parametrize("n", [1, 5, 1023, 1024, 1025, 70_001, 3_000_003])
def test_seek_select_vs_oracle(n):
    rng = np.random.default_rng(n)
    gaps = rng.integers(0, 300, n, dtype=np.uint64)
    gaps[rng.random(n) < 0.2] = 0  # plateaus: duplicate values
    big = rng.random(n) < 0.002
    gaps[big] += rng.integers(1 << 10, 1 << 20, int(big.sum()), dtype=np.uint64)
    v = np.cumsum(gaps)
    v = (v * (2**31 // max(int(v[-1]), 1))).astype(np.uint32) if v[-1] >= 2**31 else v.astype(np.uint32)
    b = _delta_buf(v)
    t = np.concatenate([rng.integers(0, int(v[-1]) + 2, 4000, dtype=np.uint64).astype(np.uint32),
                        v[rng.integers(0, n, 500)], [0, v[0], v[-1], np.uint32(min(int(v[-1]) + 1, 2**32 - 1))]])
    idx, val = P.seek_batch(b, t)
    want = np.searchsorted(v, t, side="left")
    assert np.array_equal(idx, want.astype(np.uint64))
    hit = want < n
    assert np.array_equal(val[hit], v[want[hit]])
    q = rng.integers(0, n, 5000, dtype=np.uint64)
    q = np.concatenate([q, [0, n - 1]]).astype(np.uint64)
    assert np.array_equal(P.select_batch(b, q), v[q])


def test_query_errors():
    b = _delta_buf([5, 9, 9, 40])
    with pytest.raises(P.CodecError) as e:
        P.select(b, 4)
    assert e.value.code == P.errc.out_of_range
    plain = P.EncodedBuffer(P.codec_id.stream_vbyte, 4, False, oracle.encode(np.array([5, 9, 9, 40], np.uint32)))
    with pytest.raises(P.CodecError) as e:
        P.seek(plain, 3)
    assert e.value.code == P.errc.unsupported
    bad = P.EncodedBuffer(P.codec_id.stream_vbyte, 4, True, b.bytes[:-1])
    with pytest.raises(P.CodecError) as e:
        P.seek(bad, 3)
    assert e.value.code == P.errc.truncated
    empty = _delta_buf([])
    assert P.seek(empty, 0) is None
    with pytest.raises(P.CodecError):
        P.select(empty, 0)
