"""CPU oracle for the Stream VByte hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package, and only as the checker or
the timed CPU reference; the product (``paper_1709_08990_b200``) never does.

Wraps ``oracle/build/libsvb_oracle.so`` (built from ``svb_oracle.c`` by
``oracle/Makefile``): O1 = naive per-integer loop, O2 = the paper's SSSE3
table decoder.  Parity is pinned by ``tests/golden/``
(SPEC golden vectors + outputs of the reference headers' own inline code).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "libsvb_oracle.so"

OK, TRUNCATED, TRAILING_BYTES = 0, 1, 2


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def _load() -> C.CDLL:
    if not LIB.exists():
        build()
    lib = C.CDLL(str(LIB))
    vp, sz, u32, i = C.c_void_p, C.c_size_t, C.c_uint32, C.c_int
    sig = {
        "svbo_byte_length": (u32, [u32]),
        "svbo_control_bytes": (sz, [sz]),
        "svbo_tables": (None, [vp, vp]),
        "svbo_compressed_size": (sz, [vp, sz, i, u32]),
        "svbo_encode": (sz, [vp, sz, i, u32, vp]),
        "svbo_decode": (i, [vp, sz, sz, i, u32, vp, vp]),
        "svbo_ssse3_decode": (i, [vp, sz, sz, i, u32, vp, vp]),
        "svbo_ssse3_available": (i, []),
        "svbo_delta_encode": (None, [vp, sz, u32, vp]),
        "svbo_prefix_sum": (u32, [vp, sz, u32, vp]),
        "svbo_prefix_sum4": (None, [vp, u32, vp]),
        "svbo_block_data_offsets": (None, [vp, sz, vp]),
        "svbo_decode_block": (sz, [vp, sz, sz, sz, sz, vp]),
        "svbo_paper_decode": (i, [vp, sz, sz, i, u32, vp, vp]),
        "svbo_paper_decode_batch": (i, [vp, sz, vp, i, vp, vp]),
        "svbo_mt_encode": (sz, [vp, sz, i, u32, vp, i]),
        "svbo_mt_decode": (i, [vp, sz, sz, i, u32, vp, vp, i]),
        "svbo_decode_batch": (i, [vp, sz, vp, vp, i, i]),
        "svbo_encode_batch": (i, [vp, sz, vp, vp, vp, i, i]),
        "gbo_compressed_size": (sz, [vp, sz]),
        "gbo_encode": (sz, [vp, sz, vp]),
        "gbo_decode": (i, [vp, sz, sz, i, u32, vp, vp, i]),
        "gbo_decode_group_general": (vp, [C.c_uint8, vp, vp, sz, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


lib = _load()


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint32)


def _u8(b) -> np.ndarray:
    if isinstance(b, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytes(b), np.uint8)
    return np.ascontiguousarray(b, dtype=np.uint8)


def _ptr(a: np.ndarray):
    return a.ctypes.data if a.size else None


def byte_length(x: int) -> int:
    return int(lib.svbo_byte_length(x & 0xFFFFFFFF))


def control_bytes(n: int) -> int:
    return int(lib.svbo_control_bytes(n))


def tables() -> tuple[np.ndarray, np.ndarray]:
    length = np.zeros(256, np.uint8)
    shuffle = np.zeros((256, 16), np.uint8)
    lib.svbo_tables(length.ctypes.data, shuffle.ctypes.data)
    return length, shuffle


def compressed_size(values, delta: bool = False, prev: int = 0) -> int:
    v = _u32(values)
    return int(lib.svbo_compressed_size(_ptr(v), v.size, int(delta), prev & 0xFFFFFFFF))


def encode(values, delta: bool = False, prev: int = 0) -> bytes:
    """O1 encoder (stream_vbyte.hpp:36; delta: SPEC.md:366-374 with seed prev)."""
    v = _u32(values)
    out = np.empty(control_bytes(v.size) + 4 * v.size + 1, np.uint8)
    n = lib.svbo_encode(_ptr(v), v.size, int(delta), prev & 0xFFFFFFFF, out.ctypes.data)
    return out[:n].tobytes()


def decode(data, n: int, delta: bool = False, base: int = 0, impl: str = "o1") -> tuple[int, np.ndarray, int]:
    """O1 (naive loop) or O2 (SSSE3 Fig. 4) decode -> (status, values, last)."""
    b = _u8(data)
    out = np.zeros(max(n, 1), np.uint32)
    last = C.c_uint32(0)
    fn = lib.svbo_decode if impl == "o1" else lib.svbo_ssse3_decode
    st = fn(_ptr(b), b.size, n, int(delta), base & 0xFFFFFFFF, out.ctypes.data, C.byref(last))
    return int(st), out[:n], int(last.value)


def delta_encode(values, prev: int = 0) -> np.ndarray:
    v = _u32(values)
    out = np.empty(v.size, np.uint32)
    lib.svbo_delta_encode(_ptr(v), v.size, prev & 0xFFFFFFFF, _ptr(out))
    return out


def prefix_sum(values, base: int = 0) -> np.ndarray:
    v = _u32(values)
    out = np.empty(v.size, np.uint32)
    lib.svbo_prefix_sum(_ptr(v), v.size, base & 0xFFFFFFFF, _ptr(out))
    return out


def prefix_sum4(block, base: int = 0) -> np.ndarray:
    v = _u32(block)
    assert v.size == 4
    out = np.empty(4, np.uint32)
    lib.svbo_prefix_sum4(v.ctypes.data, base & 0xFFFFFFFF, out.ctypes.data)
    return out


def block_data_offsets(data, n: int) -> np.ndarray:
    b = _u8(data)
    out = np.zeros(max(1, control_bytes(n)), np.uint64)
    lib.svbo_block_data_offsets(_ptr(b), n, out.ctypes.data)
    return out[: control_bytes(n)]


def decode_block(data, n: int, block: int, data_offset: int) -> np.ndarray:
    b = _u8(data)
    out = np.zeros(4, np.uint32)
    k = lib.svbo_decode_block(_ptr(b), b.size, n, block, data_offset, out.ctypes.data)
    return out[:k]


def paper_decode(data, n: int, delta: bool = False, base: int = 0, buf: np.ndarray | None = None) -> tuple[int, int]:
    """The paper's timing mode: single-thread O2 decode into a reused
    4096-integer buffer.  Returns (status, sum of each 4096-block's last integer mod 2^64)."""
    b = _u8(data)
    if buf is None:
        buf = np.empty(4096, np.uint32)
    chk = C.c_uint64(0)
    st = lib.svbo_paper_decode(_ptr(b), b.size, n, int(delta), base & 0xFFFFFFFF, buf.ctypes.data, C.byref(chk))
    return int(st), int(chk.value)


def paper_decode_batch(segs: np.ndarray, data, delta: bool, buf: np.ndarray | None = None) -> tuple[int, int]:
    """paper_decode over every segment (bcgpu_decode_segment layout), one thread, one buffer."""
    b = _u8(data)
    s = np.ascontiguousarray(segs)
    if buf is None:
        buf = np.empty(4096, np.uint32)
    chk = C.c_uint64(0)
    st = lib.svbo_paper_decode_batch(s.ctypes.data, s.size, _ptr(b), int(delta), buf.ctypes.data, C.byref(chk))
    return int(st), int(chk.value)


def mt_encode(values, delta: bool = False, prev: int = 0, threads: int | None = None,
              out: np.ndarray | None = None) -> int:
    """Multi-threaded CPU reference encode into ``out`` (>= ceil(n/4)+4n bytes); returns the length."""
    v = _u32(values)
    if out is None:
        out = np.empty(control_bytes(v.size) + 4 * v.size + 1, np.uint8)
    return int(lib.svbo_mt_encode(_ptr(v), v.size, int(delta), prev & 0xFFFFFFFF, out.ctypes.data,
                                  threads or os.cpu_count() or 1))


def mt_decode(data, n: int, out: np.ndarray, delta: bool = False, base: int = 0,
              threads: int | None = None) -> tuple[int, int]:
    b = _u8(data)
    last = C.c_uint32(0)
    st = lib.svbo_mt_decode(_ptr(b), b.size, n, int(delta), base & 0xFFFFFFFF, out.ctypes.data, C.byref(last),
                            threads or os.cpu_count() or 1)
    return int(st), int(last.value)


def decode_batch(segs: np.ndarray, data, out: np.ndarray, delta: bool, threads: int | None = None) -> int:
    """segs: structured array with the bcgpu_decode_segment layout."""
    b = _u8(data)
    s = np.ascontiguousarray(segs)
    return int(lib.svbo_decode_batch(s.ctypes.data, s.size, _ptr(b), out.ctypes.data, int(delta),
                                     threads or os.cpu_count() or 1))


def encode_batch(segs: np.ndarray, values, out: np.ndarray, out_lens: np.ndarray, delta: bool,
                 threads: int | None = None) -> int:
    v = _u32(values)
    s = np.ascontiguousarray(segs)
    return int(lib.svbo_encode_batch(s.ctypes.data, s.size, _ptr(v), out.ctypes.data, out_lens.ctypes.data,
                                     int(delta), threads or os.cpu_count() or 1))


# ---- varint-GB (gb_oracle.h) ----
def gb_compressed_size(values) -> int:
    v = _u32(values)
    return int(lib.gbo_compressed_size(_ptr(v), v.size))


def gb_encode(values) -> bytes:
    v = _u32(values)
    out = np.empty((v.size + 3) // 4 + 4 * v.size + 1, dtype=np.uint8)
    m = lib.gbo_encode(_ptr(v), v.size, _ptr(out))
    return out[:m].tobytes()


def gb_decode(data, n: int, delta: bool = False, base: int = 0, fast: bool = True) -> tuple[int, np.ndarray, int]:
    """(status, values, last) -- varint_gb.hpp:21-25."""
    b = _u8(data)
    out = np.zeros(max(n, 1), dtype=np.uint32)
    last = C.c_uint32(0)
    st = lib.gbo_decode(_ptr(b), b.size, n, int(delta), base & 0xFFFFFFFF, _ptr(out), C.byref(last), int(fast))
    return st, out[:n], last.value


def gb_decode_group_general(control: int, data, k: int) -> np.ndarray | None:
    """varint_gb.hpp:30-31: one group decoded field by field; None when it runs past the data."""
    b = _u8(data)
    out = np.zeros(4, dtype=np.uint32)
    base = b.ctypes.data
    r = lib.gbo_decode_group_general(control, base, base + b.size, k, _ptr(out))
    return None if not r else out[:k]
