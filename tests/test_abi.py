"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/bcgpu/bcgpu.h declares, and its pure host functions agree with
the pinned oracle.  No compute call is made (no GPU here)."""
import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np

import oracle

ROOT = Path(__file__).resolve().parents[1]


def _declared_symbols():
    hdr = (ROOT / "include" / "bcgpu" / "bcgpu.h").read_text()
    return sorted(set(re.findall(r"\b(bcgpu_[a-z0-9_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    from paper_1709_08990_b200 import _native
    declared = _declared_symbols()
    assert len(declared) >= 20
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    # the ctypes signature table covers the whole header
    assert sorted(_native.SIGNATURES) == declared


def test_exports_are_dynamic_symbols():
    from paper_1709_08990_b200 import _native
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    for s in _declared_symbols():
        assert re.search(rf"\bT {s}$", out, re.M), s


def test_library_is_sm100a():
    from paper_1709_08990_b200 import _native
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_pure_host_functions_match_oracle():
    from paper_1709_08990_b200 import _native, codec
    lib = _native.lib
    rng = np.random.default_rng(0)
    for x in list(rng.integers(0, 2**32, 5000, dtype=np.uint64)) + [0, 255, 256, 2**16, 2**24, 2**32 - 1]:
        assert lib.bcgpu_byte_length(int(x)) == oracle.byte_length(int(x))
    for n in (0, 1, 3, 4, 5, 1 << 31):
        assert lib.bcgpu_svb_control_bytes(n) == oracle.control_bytes(n)
        assert lib.bcgpu_svb_max_compressed_bytes(n) == oracle.control_bytes(n) + 4 * n
    L, S = codec.svb_tables()
    OL, OS = oracle.tables()
    assert np.array_equal(L, OL) and np.array_equal(S, OS)
    assert lib.bcgpu_abi_version() == 1
    assert _native.status_string(1) == "truncated" and _native.status_string(2) == "trailing_bytes"


def test_errc_mapping_mirrors_reference_order():
    from paper_1709_08990_b200 import codec
    ref_order = ["truncated", "trailing_bytes", "run_too_long", "value_overflow", "oversized_integer",
                 "count_mismatch", "bad_stream_size", "bad_magic", "unknown_codec", "reserved_flags",
                 "length_mismatch", "unsupported", "out_of_range", "io_failure", "bad_config"]  # codec.hpp:28-47
    assert [e.name for e in codec.errc] == ref_order
    from paper_1709_08990_b200 import _native
    for i, name in enumerate(ref_order):
        assert _native.status_string(i + 1) == name
    assert [c.value for c in codec.codec_id] == [0, 1, 2, 3]  # codec.hpp:17-22


def test_no_cpu_fallback_without_device():
    """Without a GPU the product must fail loudly, never compute on the CPU."""
    import pytest
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1709_08990_b200 import codec
    with pytest.raises(codec.GpuError):
        codec.svb_encode(np.arange(10, dtype=np.uint32))


def test_cpp_headers_compile():
    """The C++ drop-in headers (bytecodec::) compile as C++20 and match the reference API surface."""
    src = ('#include "bytecodec/stream_vbyte.hpp"\n'
           "using namespace bytecodec;\n"
           "static_assert(std::is_same_v<decltype(&svb_control_bytes), size_t(*)(size_t)>);\n"
           "int main(){ return byte_length(1024) == 2 && svb_control_bytes(5) == 2 ? 0 : 1; }\n")
    out = ROOT / "build" / "hdrcheck"
    out.parent.mkdir(exist_ok=True)
    (out.parent / "hdrcheck.cpp").write_text("#include <type_traits>\n" + src)
    subprocess.run(["g++", "-std=c++20", "-I", str(ROOT / "include"), str(out.parent / "hdrcheck.cpp"), "-o",
                    str(out)], check=True)
    assert subprocess.run([str(out)]).returncode == 0


def test_generators_deterministic_and_in_range():
    from paper_1709_08990_b200 import gen
    a = gen.uniform_classes(100000, 1)
    b = gen.uniform_classes(100000, 1)
    assert np.array_equal(a, b)
    lens = np.array([oracle.byte_length(int(x)) for x in a[:20000]])
    counts = np.bincount(lens, minlength=5)[1:]
    assert all(abs(c / 20000 - 0.25) < 0.02 for c in counts)
    g = gen.geometric_sorted(200000, 8.0, 2)
    d = np.diff(g.astype(np.int64))
    assert g[0] == 0 and (d >= 1).all() and abs(d.mean() - 8.0) < 0.1
    g5 = gen.geometric_sorted(300000, 32.0, 5)
    d5 = np.diff(g5.astype(np.int64))
    assert (d5 >= 1).all() and abs(d5.mean() - 32.0) < 0.5
    lb = gen.posting_lists(2000, 4, cap_total=1 << 20)
    assert lb.lengths.sum() <= 1 << 20 and lb.lengths.min() >= 16
    for i in range(0, 2000, 97):
        s = lb.values[int(lb.offsets[i]):int(lb.offsets[i + 1])]
        assert (np.diff(s.astype(np.int64)) >= 1).all() and s.max() < (1 << 25)
