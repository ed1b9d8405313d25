"""GPU parity for varint-GB (svb_gb.cu) through the C ABI, against the pinned oracle
(oracle/gb_oracle.c).  Bit-exact bytes and integers; the cases follow
the spec: its examples, every n mod 4, the all-small fast path vs mixed widths, delta,
truncated / trailing streams, device-pointer misalignment, and inputs large enough for
three levels of the decode's chunk-table tree."""
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


def _values(rng, n, kind):
    if kind == "small":
        return rng.integers(0, 256, n).astype(np.uint32)
    if kind == "wide":
        return rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    # mixed byte lengths, every class
    return (rng.integers(0, 2**32, n, dtype=np.uint64) >> (8 * rng.integers(0, 4, n)).astype(np.uint64)).astype(
        np.uint32)


def _roundtrip(P, v, delta=False, prev=0):
    payload = oracle.delta_encode(v, prev) if delta else v
    want = oracle.gb_encode(payload)
    got = P.gb_encode_delta(v, prev) if delta else P.gb_encode(v)
    assert got == want, f"encode mismatch n={v.size} delta={delta}"
    out = np.empty(v.size, np.uint32)
    if delta:
        last = P.gb_decode_delta(want, v.size, prev, out)
        assert last == (int(v[-1]) if v.size else prev)
    else:
        P.gb_decode(want, v.size, out)
    assert np.array_equal(out, v), f"decode mismatch n={v.size} delta={delta}"


def test_spec_vectors(P, golden_dir):
    gb = json.loads((golden_dir / "gb_spec_vectors.json").read_text())
    for c in gb["encode"]["cases"]:
        out = P.gb_encode(np.array(c["values"], np.uint32))
        if "bytes" in c:
            assert list(out) == c["bytes"], c.get("note")
        if "size" in c:
            assert len(out) == c["size"]
    for c in gb["decode"]["cases"]:
        assert list(P.gb_decode(bytes(c["bytes"]), c["n"])) == c["values"], c.get("note")
    codes = {"truncated": P.errc.truncated, "trailing_bytes": P.errc.trailing_bytes}
    for c in gb["errors"]["cases"]:
        with pytest.raises(P.CodecError) as e:
            P.gb_decode(bytes(c["bytes"]), c["n"])
        assert e.value.code == codes[c["status"]], c


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 7, 8, 31, 32, 33, 1023, 1024, 1025, 4095, 4096, 4097, 65537])
@pytest.mark.parametrize("kind", ["small", "mixed", "wide"])
def test_roundtrip_ragged(P, n, kind):
    rng = np.random.default_rng(n * 7 + len(kind))
    _roundtrip(P, _values(rng, n, kind))


@pytest.mark.parametrize("n", [1, 5, 1000, 4097, 300001])
def test_delta(P, n):
    rng = np.random.default_rng(n)
    v = np.cumsum(rng.integers(0, 3000, n, dtype=np.uint64)).astype(np.uint32) + np.uint32(12345)
    _roundtrip(P, v, delta=True, prev=12000)
    _roundtrip(P, rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32), delta=True, prev=7)  # wraps


def test_generic_codec_api(P):
    rng = np.random.default_rng(11)
    v = np.cumsum(rng.integers(0, 100, 5003)).astype(np.uint32)
    for delta in (False, True):
        b = P.encode(P.codec_id.varint_gb, v, delta)
        assert b.codec == P.codec_id.varint_gb and b.count == v.size
        assert np.array_equal(P.decode(b), v)
        f = P.write_container(b)
        assert P.read_container(f) == b


def test_errors_everywhere(P):
    rng = np.random.default_rng(5)
    v = _values(rng, 20001, "mixed")
    b = oracle.gb_encode(v)
    # cut anywhere: truncated; any suffix: trailing bytes (the oracle agrees on each)
    for cut in (1, 2, 17, 100, 4095, 4096, 4097, len(b) // 2, len(b) - 1):
        with pytest.raises(P.CodecError) as e:
            P.gb_decode(b[: len(b) - cut], v.size)
        assert oracle.gb_decode(b[: len(b) - cut], v.size)[0] == oracle.TRUNCATED
        assert e.value.code == P.errc.truncated, cut
    for extra in (b"\x00", b"\x01\x02\x03", bytes(5000)):
        with pytest.raises(P.CodecError) as e:
            P.gb_decode(b + extra, v.size)
        assert e.value.code == P.errc.trailing_bytes
    # the count disagrees with the stream
    for n2 in (v.size - 1, v.size - 4, v.size + 1):
        st = oracle.gb_decode(b, n2)[0]
        with pytest.raises(P.CodecError) as e:
            P.gb_decode(b, n2)
        assert int(e.value.code) + 1 == st
    with pytest.raises(P.CodecError) as e:
        P.gb_decode(b"\x00", 0)
    assert e.value.code == P.errc.trailing_bytes
    assert P.gb_decode(b"", 0).size == 0


def test_large_three_level_tree(P):
    # > 32 * 32 chunks of 4 KiB: the decode composes three levels of chunk tables
    rng = np.random.default_rng(21)
    n = 6_000_003
    v = _values(rng, n, "mixed")
    want = oracle.gb_encode(v)
    assert len(want) > 4096 * 32 * 32
    assert P.gb_encode(v) == want
    assert np.array_equal(P.gb_decode(want, n), v)
    d = np.cumsum(rng.integers(0, 40, n, dtype=np.uint64)).astype(np.uint32)
    _roundtrip(P, d, delta=True, prev=0)


def test_device_api_misaligned(P, dev):
    import torch
    rng = np.random.default_rng(8)
    for shift in (0, 1, 3, 7, 13):
        n = 70001
        v = _values(rng, n, "mixed")
        want = oracle.gb_encode(v)
        # input integers at a 4-B (not 16-B) offset, output bytes at any offset
        src = torch.from_numpy(np.concatenate([np.zeros(1, np.uint32), v]).view(np.int32)).cuda()[1:]
        dst = torch.zeros(P.svb_max_compressed_bytes(n) + 64, dtype=torch.uint8, device="cuda")
        out_len = torch.zeros(1, dtype=torch.int64, device="cuda")
        dev.gb_encode(src, dst[shift:], out_len, n=n)
        dev.check()
        assert int(out_len.item()) == len(want)
        assert bytes(dst[shift: shift + len(want)].cpu().numpy()) == want
        assert int(dst[:shift].sum().item()) == 0 and int(dst[shift + len(want):].sum().item()) == 0
        # decode from a misaligned device buffer into a misaligned output
        outb = torch.zeros(n + 1, dtype=torch.int32, device="cuda")
        dev.gb_decode(dst[shift: shift + len(want)], n, outb[1:])
        dev.check()
        assert np.array_equal(outb[1:].cpu().numpy().view(np.uint32), v)


@pytest.mark.slow
def test_gb_config2_full(P, dev):
    """BASELINE cfg2 size (64M sorted integers, delta): the GPU varint-GB stream equals the
    oracle's (digest) and decodes back exactly."""
    import hashlib

    import torch
    from paper_1709_08990_b200 import gen
    v = gen.config_array(2)
    want = oracle.gb_encode(oracle.delta_encode(v, 0))
    d_v = torch.from_numpy(v.view(np.int32)).cuda()
    d_c = torch.empty(P.svb_max_compressed_bytes(v.size), dtype=torch.uint8, device="cuda")
    d_len = torch.zeros(1, dtype=torch.int64, device="cuda")
    dev.gb_encode(d_v, d_c, d_len, delta=True)
    dev.check()
    m = int(d_len.item())
    assert m == len(want)
    assert hashlib.sha256(d_c[:m].cpu().numpy().tobytes()).hexdigest() == hashlib.sha256(want).hexdigest()
    d_o = torch.empty_like(d_v)
    dev.gb_decode(d_c, v.size, d_o, in_len=m, delta=True)
    dev.check()
    assert torch.equal(d_o, d_v)
