"""Context / launch-state hazards: workspace reallocation must not let
stale epoch-tagged look-back aggregates be taken as current, and launch attributes
must be applied per device."""
import ctypes as C
import threading

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def test_workspace_growth_keeps_epochs_fresh():
    """delta encode A (one-pass, tile aggregates tagged with epoch E); a call that grows
    the look-back workspace (varint-GB decode of a > 4 MiB stream); a filler call; then a
    delta encode of B with the same length: B must equal the oracle (stale aggregates
    of A must never pass for B's)."""
    import paper_1709_08990_b200 as P
    from paper_1709_08990_b200 import gen
    n = 3 << 20
    a = gen.geometric_sorted(n, 8.0, 101)
    b = gen.geometric_sorted(n, 40.0, 202)
    assert P.svb_encode_delta(a, 0) == oracle.encode(a, delta=True, prev=0)
    big = gen.config_array(3, 6 << 20)
    g = P.gb_encode(big)
    assert len(g) > 4 << 20
    assert np.array_equal(P.gb_decode(g, big.size), big)
    small = gen.config_array(1, 5000)
    assert np.array_equal(P.svb_decode(P.svb_encode(small), small.size), small)
    assert P.svb_encode_delta(b, 0) == oracle.encode(b, delta=True, prev=0)
    for _ in range(3):  # and again across several epochs
        assert P.svb_encode_delta(a, 7) == oracle.encode(a, delta=True, prev=7)
        assert P.svb_encode_delta(b, 9) == oracle.encode(b, delta=True, prev=9)


def test_threads_with_own_contexts():
    """concurrent calls from threads with their own contexts are safe
    (launch caches are per device and locked)."""
    import paper_1709_08990_b200 as P
    from paper_1709_08990_b200 import gen
    vals = [gen.config_array(3, 1 << 20 | k) for k in range(4)]
    errs = []

    def work(v):
        try:
            for _ in range(3):
                e = P.svb_encode(v)
                assert np.array_equal(P.svb_decode(e, v.size), v)
                s = np.sort(v)
                out = np.empty(s.size, np.uint32)
                P.svb_decode_delta(P.svb_encode_delta(s, 1), s.size, 1, out)
                assert np.array_equal(out, s)
        except Exception as ex:  # pragma: no cover
            errs.append(ex)
    ts = [threading.Thread(target=work, args=(v,)) for v in vals]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs


def test_two_devices_decode():
    """Pooled plain decode (> 48 KiB of dynamic shared memory) on device 0, then device 1
    in the same process: the attribute is applied per device."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("one GPU on this lease")
    from paper_1709_08990_b200 import gen
    from paper_1709_08990_b200.device import DeviceCodec
    v = gen.config_array(3, 1 << 22)
    enc = oracle.encode(v)
    for d in (0, 1):
        dev = DeviceCodec(d)
        with torch.cuda.device(d):
            d_in = torch.from_numpy(np.frombuffer(enc, np.uint8).copy()).cuda(d)
            d_o = torch.empty(v.size, dtype=torch.int32, device=f"cuda:{d}")
            dev.decode(d_in, v.size, d_o)
            dev.check()
            assert np.array_equal(d_o.cpu().numpy().view(np.uint32), v)
        dev.close()
