"""svb_append and the "SVB1" container (host-side format plumbing, svb_format.cpp), checked
against the pinned oracle's one-shot encoder and SPEC.md's examples.  CPU only: these
operations never touch the device."""
import numpy as np
import pytest

import oracle
import paper_1709_08990_b200 as P


def _buf(values, delta=False):
    v = np.asarray(values, np.uint32)
    return P.EncodedBuffer(P.codec_id.stream_vbyte, int(v.size), delta, oracle.encode(v))


def test_append_spec_examples():
    b = _buf([1, 2, 3])
    P.svb_append(b, 4)
    assert b.bytes == oracle.encode(np.array([1, 2, 3, 4], np.uint32)) and b.count == 4
    b = _buf([])
    P.svb_append(b, 7)
    assert b.bytes == oracle.encode(np.array([7], np.uint32)) and b.count == 1


def test_append_sequences_byte_identical():
    """1000 sequential appends from empty == one-shot encode, after every append;
    every byte length at every position mod 4."""
    rng = np.random.default_rng(4)
    k = rng.integers(0, 4, 1000)
    vals = (rng.integers(0, 2**32, 1000, dtype=np.uint64) >> (8 * (3 - k).astype(np.uint64))).astype(np.uint32)
    b = _buf([])
    for i, x in enumerate(vals):
        P.svb_append(b, int(x))
        assert b.bytes == oracle.encode(vals[: i + 1]), i
    for x in (0, 255, 256, 65535, 65536, 2**24 - 1, 2**24, 2**32 - 1):
        P.svb_append(b, x)
    assert b.bytes == oracle.encode(np.concatenate([vals, np.array([0, 255, 256, 65535, 65536, 2**24 - 1, 2**24,
                                                                      2**32 - 1], np.uint32)]))


def test_append_rejects_malformed():
    b = _buf([1, 2, 300, 4, 5])
    for bad in (b.bytes[:-1], b.bytes + b"\x00"):
        with pytest.raises(P.CodecError) as e:
            P.svb_append(P.EncodedBuffer(P.codec_id.stream_vbyte, 5, False, bad), 9)
        assert e.value.code in (P.errc.truncated, P.errc.trailing_bytes)
    with pytest.raises(P.CodecError) as e:
        P.svb_append(P.EncodedBuffer(P.codec_id.vbyte, 0, False, b""), 1)
    assert e.value.code == P.errc.unsupported


def test_container_spec_examples():
    empty = P.write_container(_buf([]))
    assert len(empty) == 14 and empty[:4] == b"SVB1" and empty[4] == 3
    z = P.write_container(_buf([0, 0, 0, 0]))
    assert len(z) == 19  # 14 + 1 + 4
    assert int.from_bytes(z[6:10], "little") == 4 and int.from_bytes(z[10:14], "little") == 5


def test_container_roundtrip_and_errors():
    rng = np.random.default_rng(9)
    v = np.cumsum(rng.integers(0, 5000, 10001, dtype=np.uint64)).astype(np.uint32)
    d = np.diff(v, prepend=np.uint32(0)).astype(np.uint32)
    b = P.EncodedBuffer(P.codec_id.stream_vbyte, int(v.size), True, oracle.encode(d))
    f = P.write_container(b)
    assert f[5] == 1 and P.read_container(f) == b  # SPEC.md:476 round trip, delta flag in bit 0
    cases = [
        (b"XVB1" + f[4:], P.errc.bad_magic),
        (f[:4] + b"\x07" + f[5:], P.errc.unknown_codec),
        (f[:5] + b"\x03" + f[6:], P.errc.reserved_flags),
        (f[:-1], P.errc.truncated),
        (f[:10], P.errc.truncated),
        (f + b"\x00", P.errc.trailing_bytes),
        # payload length inconsistent with count under the SVB size identity
        (f[:6] + (v.size + 4).to_bytes(4, "little") + f[10:], P.errc.length_mismatch),
        (f[:6] + (v.size - 1).to_bytes(4, "little") + f[10:], P.errc.length_mismatch),
    ]
    for data, code in cases:
        with pytest.raises(P.CodecError) as e:
            P.read_container(data)
        assert e.value.code == code, code
    with pytest.raises(P.CodecError) as e:  # other known codecs: outside this library
        P.read_container(f[:4] + b"\x00" + f[5:])
    assert e.value.code == P.errc.unsupported


def test_payload_length_identity():
    rng = np.random.default_rng(2)
    for n in (0, 1, 3, 4, 5, 1023, 4097):
        v = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
        e = oracle.encode(v)
        assert P.svb_payload_length(e, n) == len(e)


def test_container_varint_gb():
    # varint-GB payloads are verified by walking the group chain
    rng = np.random.default_rng(4)
    for n in (0, 1, 3, 4, 5, 999, 4096):
        v = (rng.integers(0, 2**32, n, dtype=np.uint64) >> rng.integers(0, 32, n).astype(np.uint64)).astype(np.uint32)
        b = P.EncodedBuffer(P.codec_id.varint_gb, n, False, oracle.gb_encode(v))
        f = P.write_container(b)
        assert f[4] == 1 and len(f) == 14 + len(b.bytes) and P.read_container(f) == b
        if n:
            for bad_count in (n + 1, n - 1 if n > 1 else n + 4):
                with pytest.raises(P.CodecError) as e:
                    P.read_container(f[:6] + bad_count.to_bytes(4, "little") + f[10:])
                assert e.value.code == P.errc.length_mismatch
    # a payload shorter than its chain (declared length cut with the count kept)
    v = np.arange(100, dtype=np.uint32) * 1000
    p = oracle.gb_encode(v)
    f = P.write_container(P.EncodedBuffer(P.codec_id.varint_gb, 100, False, p[:-3]))
    with pytest.raises(P.CodecError) as e:
        P.read_container(f)
    assert e.value.code == P.errc.length_mismatch
