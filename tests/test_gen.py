"""Synthetic-input generators on CPU: the shard forms a rank uses
(bench.py generates only its own shard) equal the same part of the whole config,
and bench.Batch shards tile the whole workload exactly."""
import numpy as np
import pytest

import bench
from paper_1709_08990_b200 import gen


def test_geometric_range_equals_slice():
    full = gen.geometric_sorted(300_000, 32.0, 5)
    for i0, n in ((0, 1000), (1, 70_000), (123_457, 100_000), (299_999, 1), (65_536, 234_464), (5, 0)):
        assert np.array_equal(gen.geometric_sorted_range(i0, n, 32.0, 5), full[i0:i0 + n]), (i0, n)


def test_posting_lists_range_equals_slice():
    lb = gen.posting_lists(3000, 4, cap_total=3000 * 1875)
    for lo, hi in ((0, 3000), (1000, 2100), (2999, 3000), (5, 5)):
        r = gen.posting_lists_range(lb.lengths, lo, hi, 4)
        assert np.array_equal(r.values, lb.values[int(lb.offsets[lo]):int(lb.offsets[hi])])
        assert np.array_equal(r.lengths, lb.lengths[lo:hi])


def test_generator_loads_without_codec_library():
    """bench's reference arm loads gen.py standalone: it must not map libbytecodec_b200.so."""
    import subprocess
    import sys
    code = ("import bench, pathlib; bench._gen().config_array(3, 1000); "
            "m = pathlib.Path('/proc/self/maps').read_text(); "
            "assert 'libbytecodec_b200' not in m and 'libsvbgen' in m, 'codec library mapped'")
    subprocess.run([sys.executable, "-c", code], cwd=bench.ROOT, check=True)


@pytest.mark.parametrize("cfg,scale", [(4, 0.01), (5, 1 / 256)])
@pytest.mark.parametrize("world", [2, 3])
def test_batch_shards_tile_the_workload(cfg, scale, world):
    whole = bench.Batch(cfg, 0, 1, scale)
    parts = [bench.Batch(cfg, r, world, scale) for r in range(world)]
    assert sum(p.nseg for p in parts) == whole.nseg
    assert [p.seg_lo for p in parts] == [0] + [p.seg_hi for p in parts[:-1]]
    assert np.array_equal(np.concatenate([p.values for p in parts]), whole.values)
    assert np.array_equal(np.concatenate([p.lens for p in parts]), whole.lens)
    assert np.array_equal(np.concatenate([p.prevs for p in parts]), whole.prevs)
    if cfg == 5:  # chained chunks: prev of chunk k = last value of chunk k-1
        v = whole.values.reshape(-1, gen.CFG5_CHUNK)
        assert whole.prevs[0] == 0 and np.array_equal(whole.prevs[1:], v[:-1, -1])
