"""Pin the CPU oracle (test infrastructure) before trusting it as the GPU checker.

Pins: SPEC.md golden vectors (tests/golden/spec_vectors.json) and outputs of the
reference headers' own inline code (tests/golden/ref_inline_pins.json, produced
by oracle/pin/make_ref_pins.sh).  Properties: SPEC.md:333-336 (round trip,
size identity, out-of-order block decode), SPEC.md:387-389 (delta), acceptance
criteria 1, 3, 4.  O1 (loop) and O2 (SSSE3 Fig. 4) are
cross-checked against each other everywhere.
"""
import json

import numpy as np
import pytest

import oracle


@pytest.fixture(scope="module")
def spec(golden_dir):
    return json.loads((golden_dir / "spec_vectors.json").read_text())


@pytest.fixture(scope="module")
def refpins(golden_dir):
    return json.loads((golden_dir / "ref_inline_pins.json").read_text())


def test_byte_length_spec(spec):
    for x, want in spec["byte_length"]["cases"]:
        assert oracle.byte_length(x) == want


def test_byte_length_matches_reference_inline_code(refpins):
    for x, want in refpins["byte_length"]:
        assert oracle.byte_length(x) == want, x
    for x, want in refpins["byte_length_random"]["values"]:
        assert oracle.byte_length(x) == want, x


def test_control_bytes_matches_reference_inline_code(refpins):
    for n, want in refpins["svb_control_bytes"]:
        assert oracle.control_bytes(n) == want


def test_byte_length_brute_force():
    # SPEC.md:79 invariant against a divide-by-256 loop
    rng = np.random.default_rng(1)
    xs = list(rng.integers(0, 2**32, 20000, dtype=np.uint64)) + [0, 255, 256, 65535, 65536, 2**24 - 1, 2**24,
                                                                  2**32 - 1]
    for x in xs:
        x = int(x)
        L, y = 1, x >> 8
        while y:
            L, y = L + 1, y >> 8
        assert oracle.byte_length(x) == L


def test_tables(spec, refpins):
    length, shuffle = oracle.tables()
    for c, want in spec["length_table"]["cases"]:
        assert length[c] == want
    for c in range(256):
        assert length[c] == sum(((c >> (2 * i)) & 3) + 1 for i in range(4))
    assert refpins["svb_shuffle_fill"] == 0xFF
    # table-driven block decode == scalar field extraction, all 256 x 100 fills
    rng = np.random.default_rng(7)
    for c in range(256):
        fills = rng.integers(0, 256, (100, 16), dtype=np.uint8)
        for data in fills:
            lanes = []
            for lane in range(4):
                v = 0
                for b in range(4):
                    idx = shuffle[c][4 * lane + b]
                    v |= (int(data[idx]) if idx < 16 else 0) << (8 * b)
                lanes.append(v)
            vals = oracle.decode_block(bytes([c]) + data.tobytes(), 4, 0, 0)
            assert lanes == list(vals)


def test_encode_spec(spec):
    for case in spec["encode"]["cases"]:
        assert list(oracle.encode(case["values"])) == case["bytes"]


@pytest.mark.parametrize("impl", ["o1", "o2"])
def test_decode_spec(spec, impl):
    for case in spec["decode"]["cases"]:
        st, vals, _ = oracle.decode(bytes(case["bytes"]), case["n"], impl=impl)
        assert st == oracle.OK
        assert list(vals) == case["values"]


def test_size_identity(spec):
    si = spec["size_identity"]
    rng = np.random.default_rng(3)
    v = rng.integers(si["range"][0], si["range"][1], si["n"], dtype=np.uint32)
    enc = oracle.encode(v)
    assert len(enc) == (si["n"] + 3) // 4 + si["n"]
    assert 8 * len(enc) / si["n"] == si["bits_per_int"]


def test_delta_spec(spec):
    for src, want in spec["delta_encode"]["cases"]:
        assert list(oracle.delta_encode(src)) == want
    for src, base, want in spec["prefix_sum"]["cases"]:
        assert list(oracle.prefix_sum(src, base)) == want
        assert list(oracle.prefix_sum4(src, base)) == want


def test_prefix_sum4_equals_scalar():
    rng = np.random.default_rng(11)
    blocks = rng.integers(0, 2**32, (20000, 4), dtype=np.uint64).astype(np.uint32)
    bases = rng.integers(0, 2**32, 20000, dtype=np.uint64)
    for blk, base in zip(blocks, bases):
        assert list(oracle.prefix_sum4(blk, int(base))) == list(oracle.prefix_sum(blk, int(base)))


def _mixed(rng, n):
    k = rng.integers(0, 4, n)
    lo = np.where(k == 0, 0, 1 << (8 * k)).astype(np.uint64)
    span = ((1 << (8 * (k + 1))) - lo).astype(np.uint64)
    return (lo + (rng.integers(0, 2**62, n, dtype=np.uint64) % span)).astype(np.uint32)


def test_roundtrip_property_o1_o2():
    """Acceptance criterion 1 (SVB part), scaled to the CPU suite: lengths 0..10^4,
    every n mod 4 residue, mixed classes, plain and delta (unsorted/wrapping)."""
    rng = np.random.default_rng(2024)
    for it in range(3000):
        n = int(rng.integers(0, 64)) if it % 3 else int(rng.integers(0, 10001))
        v = _mixed(rng, n)
        delta = bool(it & 1)
        prev = int(rng.integers(0, 2**32)) if delta and it % 5 == 0 else 0
        enc = oracle.encode(v, delta=delta, prev=prev)
        assert len(enc) == oracle.compressed_size(v, delta, prev)
        for impl in ("o1", "o2"):
            st, out, last = oracle.decode(enc, n, delta=delta, base=prev, impl=impl)
            assert st == oracle.OK
            assert np.array_equal(out, v)
            if delta:
                assert last == (int(v[-1]) if n else prev)


def test_delta_roundtrip_unsorted_wrapping():
    rng = np.random.default_rng(5)
    for _ in range(200):
        s = rng.integers(0, 2**32, int(rng.integers(0, 300)), dtype=np.uint64).astype(np.uint32)
        assert np.array_equal(oracle.prefix_sum(oracle.delta_encode(s), 0), s)


def test_out_of_order_block_decode():
    """blocks decoded in random order via the offset index == in-order decode."""
    rng = np.random.default_rng(9)
    for n in (1, 3, 4, 5, 257, 1000, 4099):
        v = _mixed(rng, n)
        enc = oracle.encode(v)
        offs = oracle.block_data_offsets(enc, n)
        out = np.zeros(n, np.uint32)
        for k in rng.permutation(len(offs)):
            blk = oracle.decode_block(enc, n, int(k), int(offs[k]))
            out[4 * k: 4 * k + len(blk)] = blk
        assert np.array_equal(out, v)


def test_malformed_inputs():
    v = np.array([1, 300, 70000, 2**31, 5], np.uint32)
    enc = oracle.encode(v)
    for impl in ("o1", "o2"):
        assert oracle.decode(enc[:-1], 5, impl=impl)[0] == oracle.TRUNCATED
        assert oracle.decode(enc + b"\0", 5, impl=impl)[0] == oracle.TRAILING_BYTES
        assert oracle.decode(enc[:1], 5, impl=impl)[0] == oracle.TRUNCATED  # shorter than the control stream
        assert oracle.decode(b"", 0, impl=impl)[0] == oracle.OK


def test_mt_reference_matches_o1():
    rng = np.random.default_rng(12)
    for n in (0, 1, 5, 1000, 100003):
        for delta in (False, True):
            v = np.sort(_mixed(rng, n)) if delta else _mixed(rng, n)
            ref = oracle.encode(v, delta=delta, prev=7)
            out = np.empty((n + 3) // 4 + 4 * n + 1, np.uint8)
            m = oracle.mt_encode(v, delta=delta, prev=7, threads=5, out=out)
            assert out[:m].tobytes() == ref
            dec = np.empty(max(n, 1), np.uint32)
            st, last = oracle.mt_decode(ref, n, dec, delta=delta, base=7, threads=5)
            assert st == oracle.OK and np.array_equal(dec[:n], v)
    # chunk seams with 1-byte ints (the <=3-byte store spill must stay inside its chunk)
    from paper_1709_08990_b200 import gen
    v = gen.config_array(2, 1 << 21)
    ref = oracle.encode(v, delta=True)
    for th in (2, 7, 16):
        out = np.empty((v.size + 3) // 4 + 4 * v.size + 1, np.uint8)
        m = oracle.mt_encode(v, delta=True, threads=th, out=out)
        assert out[:m].tobytes() == ref


def test_paper_mode_decode():
    """The paper's timing mode: O2 decode into a reused 4096-integer buffer,
    single segments and batches; the check value is the sum of each block's last integer."""
    rng = np.random.default_rng(21)
    buf = np.empty(4096, np.uint32)
    for n, delta in ((1, False), (4095, True), (4096, False), (4097, True), (100_003, True), (50_000, False)):
        v = np.cumsum(rng.integers(0, 1000, n)).astype(np.uint32) if delta else \
            rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32) >> rng.integers(0, 32, n).astype(np.uint32)
        enc = oracle.encode(v, delta=delta, prev=3)
        st, chk = oracle.paper_decode(enc, n, delta, 3, buf)
        idx = np.minimum(np.arange(0, n, 4096) + 4095, n - 1)
        assert st == oracle.OK and chk == int(v[idx].astype(np.uint64).sum()) % (1 << 64)
        assert oracle.paper_decode(enc[:-1], n, delta, 3, buf)[0] == oracle.TRUNCATED
    # batch form over the bcgpu_decode_segment layout
    segs_v = [np.cumsum(rng.integers(1, 300, k)).astype(np.uint32) for k in (5, 4096, 9000, 1)]
    encs = [oracle.encode(x, delta=True, prev=0) for x in segs_v]
    dt = np.dtype([("src_offset", "<u8"), ("src_bytes", "<u8"), ("dst_offset", "<u8"), ("n", "<u4"), ("prev", "<u4")])
    ds = np.zeros(len(encs), dt)
    ds["src_offset"] = np.concatenate([[0], np.cumsum([len(e) for e in encs])[:-1]])
    ds["src_bytes"] = [len(e) for e in encs]
    ds["n"] = [x.size for x in segs_v]
    st, chk = oracle.paper_decode_batch(ds, b"".join(encs), True, buf)
    want = sum(int(x[np.minimum(np.arange(0, x.size, 4096) + 4095, x.size - 1)].astype(np.uint64).sum()) for x in segs_v)
    assert st == oracle.OK and chk == want % (1 << 64)
