"""varint-GB oracle (oracle/gb_oracle.c) pinned to the reference's SPEC vectors -- CPU only.

Cases follow SPEC.md:164-214 (codec_varintgb): the examples, the incomplete final block,
the truncated / trailing errors, the size formula, and the fast-path vs general-path
differential the spec asks for."""
import json

import numpy as np
import pytest

import oracle

STATUS = {"ok": oracle.OK, "truncated": oracle.TRUNCATED, "trailing_bytes": oracle.TRAILING_BYTES}


@pytest.fixture(scope="module")
def gb(golden_dir):
    return json.loads((golden_dir / "gb_spec_vectors.json").read_text())


def test_spec_encode(gb):
    for c in gb["encode"]["cases"]:
        out = oracle.gb_encode(c["values"])
        if "bytes" in c:
            assert list(out) == c["bytes"], c.get("note")
        if "size" in c:
            assert len(out) == c["size"], c.get("note")
        assert oracle.gb_compressed_size(c["values"]) == len(out)


def test_spec_decode(gb):
    for fast in (True, False):
        for c in gb["decode"]["cases"]:
            st, v, _ = oracle.gb_decode(bytes(c["bytes"]), c["n"], fast=fast)
            assert st == oracle.OK and list(v) == c["values"], c.get("note")


def test_spec_errors(gb):
    for fast in (True, False):
        for c in gb["errors"]["cases"]:
            st, _, _ = oracle.gb_decode(bytes(c["bytes"]), c["n"], fast=fast)
            assert st == STATUS[c["status"]], c


def test_first_control_byte_layout():
    # integer 0 in the two least-significant bits
    assert oracle.gb_encode([1 << 8, 0, 0, 0])[0] == 0b01
    assert oracle.gb_encode([0, 0, 0, 1 << 24])[0] == 0b11 << 6


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 7, 8, 13, 255, 1000, 4097])
def test_roundtrip_ragged(n):
    rng = np.random.default_rng(n)
    v = (rng.integers(0, 2**32, n, dtype=np.uint64) >> rng.integers(0, 32, n).astype(np.uint64)).astype(np.uint32)
    b = oracle.gb_encode(v)
    assert len(b) == oracle.gb_compressed_size(v)
    for fast in (True, False):
        st, out, _ = oracle.gb_decode(b, n, fast=fast)
        assert st == oracle.OK and np.array_equal(out, v)
    # one byte short is truncated, one extra byte is trailing
    assert oracle.gb_decode(b[:-1], n)[0] == oracle.TRUNCATED
    assert oracle.gb_decode(b + b"\0", n)[0] == oracle.TRAILING_BYTES


def test_roundtrip_property_many():
    # roundtrip for all N mod 4 (a scaled-down sweep of the >= 1e5-case property)
    rng = np.random.default_rng(7)
    for _ in range(2000):
        n = int(rng.integers(0, 40))
        v = (rng.integers(0, 2**32, n, dtype=np.uint64) >> rng.integers(0, 32, n).astype(np.uint64)).astype(np.uint32)
        st, out, _ = oracle.gb_decode(oracle.gb_encode(v), n)
        assert st == oracle.OK and np.array_equal(out, v)


def test_size_formula_ten_bits():
    v = np.arange(4000, dtype=np.uint32) % 256
    assert len(oracle.gb_encode(v)) * 8 == 10 * v.size


def test_fast_vs_general_all_small():
    rng = np.random.default_rng(3)
    v = rng.integers(0, 256, 4096).astype(np.uint32)
    b = oracle.gb_encode(v)
    a, g = oracle.gb_decode(b, v.size, fast=True), oracle.gb_decode(b, v.size, fast=False)
    assert a[0] == g[0] == oracle.OK and np.array_equal(a[1], g[1])
    assert np.array_equal(oracle.gb_decode_group_general(0, bytes([1, 2, 3, 4]), 4), [1, 2, 3, 4])
    assert oracle.gb_decode_group_general(0xFF, bytes(15), 4) is None


def test_delta():
    rng = np.random.default_rng(5)
    vals = np.cumsum(rng.integers(0, 1000, 1001)).astype(np.uint32) + np.uint32(77)
    d = oracle.delta_encode(vals, 77)
    st, out, last = oracle.gb_decode(oracle.gb_encode(d), vals.size, delta=True, base=77)
    assert st == oracle.OK and np.array_equal(out, vals) and last == int(vals[-1])
    assert oracle.gb_decode(b"", 0, delta=True, base=9)[2] == 9
