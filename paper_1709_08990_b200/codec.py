"""Python mirror of the reference's Stream VByte operator API.

Names, argument meaning and error behaviour follow
``proj/core/include/bytecodec/codec.hpp:17-96`` and ``stream_vbyte.hpp:24-54``
(namespace ``bytecodec``): the same ``codec_id`` tags, the same ``errc``
taxonomy raised as :class:`CodecError`, ``encode``/``decode`` over
:class:`EncodedBuffer`, and the ``svb_*`` functions.  Host arrays (numpy) go
through the C ABI's synchronous ``*_host`` entry points; CUDA tensors go
through :class:`DeviceCodec` (stream-ordered ``*_device`` entry points).
Every call runs on the GPU -- there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _native
from ._native import lib


class codec_id(enum.IntEnum):
    """Wire tags, reference codec.hpp:17-22."""
    vbyte = 0
    varint_gb = 1
    varint_g8iu = 2
    stream_vbyte = 3


class errc(enum.IntEnum):
    """reference codec.hpp:28-47 (same order)."""
    truncated = 0
    trailing_bytes = 1
    run_too_long = 2
    value_overflow = 3
    oversized_integer = 4
    count_mismatch = 5
    bad_stream_size = 6
    bad_magic = 7
    unknown_codec = 8
    reserved_flags = 9
    length_mismatch = 10
    unsupported = 11
    out_of_range = 12
    io_failure = 13
    bad_config = 14


class CodecError(RuntimeError):
    """codec_error (codec.hpp:49-58): carries an :class:`errc`."""

    def __init__(self, code: errc, what: str):
        super().__init__(what)
        self.code = code


class GpuError(RuntimeError):
    """A CUDA / argument failure the reference cannot produce."""


def _check(st: int, where: str) -> None:
    if st == 0:
        return
    if 1 <= st <= 15:
        raise CodecError(errc(st - 1), f"{where}: {_native.status_string(st)}")
    msg = f"{where}: {_native.status_string(st)}"
    if st == 101:
        msg += f" ({_native.last_cuda_error()})"
    raise GpuError(msg)


@dataclass
class EncodedBuffer:
    """encoded_buffer, codec.hpp:60-67."""
    codec: codec_id = codec_id.vbyte
    count: int = 0
    delta: bool = False
    bytes: bytes = field(default=b"")


def byte_length(x: int) -> int:
    """codec.hpp:70-72 (served by the library)."""
    return int(lib.bcgpu_byte_length(int(x) & 0xFFFFFFFF))


def svb_control_bytes(n: int) -> int:
    """stream_vbyte.hpp:34."""
    return int(lib.bcgpu_svb_control_bytes(n))


def svb_max_compressed_bytes(n: int) -> int:
    return int(lib.bcgpu_svb_max_compressed_bytes(n))


def svb_tables() -> tuple[np.ndarray, np.ndarray]:
    """decode_tables (stream_vbyte.hpp:24-32): (length[256], shuffle[256,16])."""
    length = np.zeros(256, np.uint8)
    shuffle = np.zeros((256, 16), np.uint8)
    lib.bcgpu_svb_tables(length.ctypes.data, shuffle.ctypes.data)
    return length, shuffle


# ---- per-thread context --------------------------------------------------
_tls = threading.local()


def _ctx(device: int = 0) -> int:
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        p = C.c_void_p()
        _check(lib.bcgpu_ctx_create(device, C.byref(p)), "bcgpu_ctx_create")
        ctxs[device] = p.value
    return ctxs[device]


def _u32_array(values) -> np.ndarray:
    a = np.ascontiguousarray(values, dtype=np.uint32)
    return a


def _byte_array(data) -> np.ndarray:
    if isinstance(data, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytes(data), dtype=np.uint8)
    return np.ascontiguousarray(data, dtype=np.uint8)


# ---- host-span API (reference signatures) --------------------------------
def _encode(values, delta: bool, prev: int) -> bytes:
    v = _u32_array(values)
    n = v.size
    out = np.empty(max(1, svb_max_compressed_bytes(n)), np.uint8)
    out_len = C.c_size_t(0)
    _check(lib.bcgpu_svb_encode_host(_ctx(), v.ctypes.data, n, int(delta), prev & 0xFFFFFFFF,
                                     out.ctypes.data, out.size, C.byref(out_len)), "svb_encode")
    return out[: out_len.value].tobytes()


def svb_encode(values) -> bytes:
    """stream_vbyte.hpp:36."""
    return _encode(values, False, 0)


def svb_encode_delta(values, prev: int = 0) -> bytes:
    """Extension E2: prev-seeded delta encode."""
    return _encode(values, True, prev)


def _decode(data, n: int, delta: bool, base: int, out) -> int:
    b = _byte_array(data)
    if out is None:
        raise ValueError("out must hold n integers")
    if out.dtype != np.uint32 or not out.flags.c_contiguous or out.size < n:
        raise ValueError("out must be a C-contiguous uint32 array of at least n elements")
    last = C.c_uint32(0)
    _check(lib.bcgpu_svb_decode_host(_ctx(), b.ctypes.data if b.size else None, b.size, n, int(delta),
                                     base & 0xFFFFFFFF, out.ctypes.data, C.byref(last)),
           "svb_decode_delta" if delta else "svb_decode")
    return int(last.value)


def svb_decode(data, n: int, out: np.ndarray | None = None) -> np.ndarray:
    """stream_vbyte.hpp:38-39 (both overloads: fills ``out`` or returns a new array)."""
    o = np.empty(n, np.uint32) if out is None else out
    _decode(data, n, False, 0, o)
    return o


def svb_decode_delta(data, n: int, base: int, out: np.ndarray) -> int:
    """stream_vbyte.hpp:41-42: fused decode + prefix sum; returns the last value."""
    return _decode(data, n, True, base, out)


def svb_block_data_offsets(data, n: int) -> np.ndarray:
    """stream_vbyte.hpp:48-49."""
    b = _byte_array(data)
    offs = np.empty(max(1, svb_control_bytes(n)), np.uint64)
    _check(lib.bcgpu_svb_block_offsets_host(_ctx(), b.ctypes.data if b.size else None, b.size, n,
                                            offs.ctypes.data), "svb_block_data_offsets")
    return offs[: svb_control_bytes(n)]


def svb_decode_block(data, n: int, block: int, data_offset: int) -> np.ndarray:
    """stream_vbyte.hpp:51-54: returns the block's integers (4, or fewer for the tail)."""
    vals, counts = svb_decode_blocks(data, n, np.array([block], np.uint64), np.array([data_offset], np.uint64))
    return vals[0, : counts[0]]


def svb_decode_blocks(data, n: int, blocks, offsets) -> tuple[np.ndarray, np.ndarray]:
    """Batched random-access block decode: (values[nblocks,4], counts[nblocks])."""
    b = _byte_array(data)
    blk = np.ascontiguousarray(blocks, np.uint64)
    off = np.ascontiguousarray(offsets, np.uint64)
    out = np.zeros((blk.size, 4), np.uint32)
    cnt = np.zeros(blk.size, np.uint32)
    _check(lib.bcgpu_svb_decode_blocks_host(_ctx(), b.ctypes.data if b.size else None, b.size, n,
                                            blk.ctypes.data, off.ctypes.data, blk.size, out.ctypes.data,
                                            cnt.ctypes.data), "svb_decode_block")
    return out, cnt


# ---- segmented batches through host memory (codec.hpp:87-90 once per segment) ----
def _np_ptr(a: np.ndarray | None):
    return a.ctypes.data if a is not None and a.size else None


def svb_encode_batch(values, seg_n, seg_prev=None, delta: bool = True, out: np.ndarray | None = None
                     ) -> tuple[np.ndarray, np.ndarray]:
    """Encode every segment (seg_n[s] integers of the concatenated ``values``, delta base
    seg_prev[s]) as its own stream; streams packed back to back.  Returns (bytes, offsets):
    segment s is bytes[offsets[s]:offsets[s+1]].  One C-ABI call, pipelined over pieces."""
    v = _u32_array(values)
    ns = np.ascontiguousarray(seg_n, dtype=np.uint32)
    if int(ns.sum(dtype=np.uint64)) != v.size:
        raise ValueError("sum(seg_n) must equal len(values)")
    pv = None if seg_prev is None else np.ascontiguousarray(seg_prev, dtype=np.uint32)
    cap = int(((ns.astype(np.uint64) + 3) // 4 + 4 * ns.astype(np.uint64)).sum())
    o = np.empty(max(1, cap), np.uint8) if out is None else out
    offs = np.zeros(ns.size + 1, np.uint64)
    _check(lib.bcgpu_svb_encode_batch_host(_ctx(), _np_ptr(v), _np_ptr(ns), _np_ptr(pv), ns.size, int(delta),
                                           o.ctypes.data, o.size, offs.ctypes.data), "svb_encode_batch")
    return o[: int(offs[-1])], offs


def svb_decode_batch(data, offsets, seg_n, seg_base=None, delta: bool = True, out: np.ndarray | None = None,
                     want_last: bool = False):
    """Decode the packed streams of :func:`svb_encode_batch` (segment s = data[offsets[s]:offsets[s+1]],
    seg_n[s] integers, delta base seg_base[s]) into one concatenated array; with want_last also
    every segment's last value (decode_payload_delta's return value)."""
    b = _byte_array(data)
    offs = np.ascontiguousarray(offsets, dtype=np.uint64)
    ns = np.ascontiguousarray(seg_n, dtype=np.uint32)
    if offs.size != ns.size + 1:
        raise ValueError("offsets must hold len(seg_n) + 1 entries")
    bs = None if seg_base is None else np.ascontiguousarray(seg_base, dtype=np.uint32)
    total = int(ns.sum(dtype=np.uint64))
    o = np.empty(max(1, total), np.uint32) if out is None else out
    last = np.zeros(max(1, ns.size), np.uint32) if want_last else None
    _check(lib.bcgpu_svb_decode_batch_host(_ctx(), _np_ptr(b), b.size, offs.ctypes.data, _np_ptr(ns), _np_ptr(bs),
                                           ns.size, int(delta), o.ctypes.data, _np_ptr(last)), "svb_decode_batch")
    res = o[:total]
    return (res, last[: ns.size]) if want_last else res


# ---- varint-GB (varint_gb.hpp:14-31) -----------------------
def _gb_encode(values, delta: bool, prev: int) -> bytes:
    v = _u32_array(values)
    n = v.size
    out = np.empty(max(1, svb_max_compressed_bytes(n)), np.uint8)
    out_len = C.c_size_t(0)
    _check(lib.bcgpu_gb_encode_host(_ctx(), v.ctypes.data, n, int(delta), prev & 0xFFFFFFFF, out.ctypes.data,
                                    out.size, C.byref(out_len)), "gb_encode")
    return out[: out_len.value].tobytes()


def gb_encode(values) -> bytes:
    """varint_gb.hpp:19."""
    return _gb_encode(values, False, 0)


def gb_encode_delta(values, prev: int = 0) -> bytes:
    """The delta transform (seeded with prev) then gb_encode -- encode(varint_gb, v, True)."""
    return _gb_encode(values, True, prev)


def _gb_decode(data, n: int, delta: bool, base: int, out) -> int:
    b = _byte_array(data)
    if out.dtype != np.uint32 or not out.flags.c_contiguous or out.size < n:
        raise ValueError("out must be a C-contiguous uint32 array of at least n elements")
    last = C.c_uint32(0)
    _check(lib.bcgpu_gb_decode_host(_ctx(), b.ctypes.data if b.size else None, b.size, n, int(delta),
                                    base & 0xFFFFFFFF, out.ctypes.data, C.byref(last)),
           "gb_decode_delta" if delta else "gb_decode")
    return int(last.value)


def gb_decode(data, n: int, out: np.ndarray | None = None) -> np.ndarray:
    """varint_gb.hpp:21-22 (both overloads: fills ``out`` or returns a new array)."""
    o = np.empty(n, np.uint32) if out is None else out
    _gb_decode(data, n, False, 0, o)
    return o


def gb_decode_delta(data, n: int, base: int, out: np.ndarray) -> int:
    """varint_gb.hpp:24-25: fused decode + prefix sum; returns the last value."""
    return _gb_decode(data, n, True, base, out)


_GPU_CODECS = (codec_id.stream_vbyte, codec_id.varint_gb)


def _require_gpu_codec(cid) -> codec_id:
    c = codec_id(cid)
    if c not in _GPU_CODECS:
        raise CodecError(errc.unsupported, "only stream_vbyte and varint_gb are implemented on the GPU path")
    return c


def encode_payload(cid, values) -> bytes:
    """codec.hpp:84."""
    return gb_encode(values) if _require_gpu_codec(cid) == codec_id.varint_gb else svb_encode(values)


def decode_payload(cid, data, n: int, out: np.ndarray) -> None:
    """codec.hpp:85."""
    if _require_gpu_codec(cid) == codec_id.varint_gb:
        gb_decode(data, n, out)
    else:
        svb_decode(data, n, out)


def decode_payload_delta(cid, data, n: int, base: int, out: np.ndarray) -> int:
    """codec.hpp:89-90."""
    if _require_gpu_codec(cid) == codec_id.varint_gb:
        return gb_decode_delta(data, n, base, out)
    return svb_decode_delta(data, n, base, out)


def encode(cid, values, delta: bool = False) -> EncodedBuffer:
    """codec.hpp:92-93 (delta base 0)."""
    c = _require_gpu_codec(cid)
    v = _u32_array(values)
    if v.size > 0xFFFFFFFF:
        raise CodecError(errc.out_of_range, "count exceeds uint32")
    if c == codec_id.varint_gb:
        data = gb_encode_delta(v, 0) if delta else gb_encode(v)
    else:
        data = svb_encode_delta(v, 0) if delta else svb_encode(v)
    return EncodedBuffer(c, int(v.size), bool(delta), data)


def decode(buf: EncodedBuffer) -> np.ndarray:
    """codec.hpp:95-96."""
    _require_gpu_codec(buf.codec)
    out = np.empty(buf.count, np.uint32)
    if buf.delta:
        decode_payload_delta(buf.codec, buf.bytes, buf.count, 0, out)
    else:
        decode_payload(buf.codec, buf.bytes, buf.count, out)
    return out


def _require_svb(cid) -> None:
    if codec_id(cid) != codec_id.stream_vbyte:
        raise CodecError(errc.unsupported, "this operation is defined for codec_id.stream_vbyte only")


# ---- format plumbing on the host (svb_format.cpp): no device, no context -------------
def svb_payload_length(data, n: int) -> int:
    """ceil(n/4) + the data bytes the control stream declares."""
    b = _byte_array(data)
    out = C.c_size_t(0)
    _check(lib.bcgpu_svb_payload_length(b.ctypes.data if b.size else None, b.size, n, C.byref(out)),
           "svb_payload_length")
    return int(out.value)


def svb_append(buf: EncodedBuffer, value: int) -> None:
    """svb_append, reference stream_vbyte.hpp:44-46: appends `value` as
    the next payload integer in place; the bytes stay identical to a one-shot encode."""
    _require_svb(buf.codec)
    b = np.frombuffer(bytes(buf.bytes) + b"\0" * 5, np.uint8).copy()
    n_old = len(buf.bytes)
    out = C.c_size_t(0)
    _check(lib.bcgpu_svb_append(b.ctypes.data, n_old, b.size, buf.count, int(value) & 0xFFFFFFFF, C.byref(out)),
           "svb_append")
    buf.bytes = b[: out.value].tobytes()
    buf.count += 1


def write_container(buf: EncodedBuffer) -> bytes:
    """The 14-byte "SVB1" container: header then payload."""
    p = _byte_array(buf.bytes)
    out = np.empty(14 + p.size, np.uint8)
    n = C.c_size_t(0)
    _check(lib.bcgpu_container_write(int(buf.codec), int(bool(buf.delta)), int(buf.count),
                                     p.ctypes.data if p.size else None, p.size, out.ctypes.data, out.size,
                                     C.byref(n)), "write_container")
    return out[: n.value].tobytes()


def read_container(data) -> EncodedBuffer:
    """Inverse of write_container; bad_magic / unknown_codec / reserved_flags / truncated /
    trailing_bytes / length_mismatch are distinct errors."""
    b = _byte_array(data)
    tag, delta, count = C.c_uint8(0), C.c_int(0), C.c_uint32(0)
    off, plen = C.c_size_t(0), C.c_size_t(0)
    _check(lib.bcgpu_container_read(b.ctypes.data if b.size else None, b.size, C.byref(tag), C.byref(delta),
                                    C.byref(count), C.byref(off), C.byref(plen)), "read_container")
    return EncodedBuffer(codec_id(tag.value), int(count.value), bool(delta.value),
                         b[off.value: off.value + plen.value].tobytes())


# ---- batched seek / select on the GPU (svb_query.cu) ---------------
def _require_delta(buf: EncodedBuffer) -> None:
    _require_svb(buf.codec)
    if not buf.delta:
        raise CodecError(errc.unsupported, "seek / select need a delta-coded buffer (SPEC.md:414)")


def seek_batch(buf: EncodedBuffer, targets) -> tuple[np.ndarray, np.ndarray]:
    """For every target the first (index, value) with value >= target over the buffer's
    non-decreasing logical sequence; index == buf.count means not found."""
    _require_delta(buf)
    b = _byte_array(buf.bytes)
    t = _u32_array(targets)
    idx = np.empty(t.size, np.uint64)
    val = np.empty(t.size, np.uint32)
    _check(lib.bcgpu_svb_seek_host(_ctx(), b.ctypes.data if b.size else None, b.size, buf.count, 0,
                                   t.ctypes.data if t.size else None, t.size, idx.ctypes.data if t.size else None,
                                   val.ctypes.data if t.size else None), "seek")
    return idx, val


def select_batch(buf: EncodedBuffer, indices) -> np.ndarray:
    """The logical value at every index (out_of_range if any index >= buf.count)."""
    _require_delta(buf)
    b = _byte_array(buf.bytes)
    i = np.ascontiguousarray(np.asarray(indices, dtype=np.uint64))
    val = np.empty(i.size, np.uint32)
    _check(lib.bcgpu_svb_select_host(_ctx(), b.ctypes.data if b.size else None, b.size, buf.count, 0,
                                     i.ctypes.data if i.size else None, i.size, val.ctypes.data if i.size else None),
           "select")
    return val


def seek(buf: EncodedBuffer, target: int):
    """(index, value) of the first value >= target, or None (not found)."""
    idx, val = seek_batch(buf, [target])
    return None if int(idx[0]) >= buf.count else (int(idx[0]), int(val[0]))


def select(buf: EncodedBuffer, i: int) -> int:
    """the i-th logical value."""
    if i < 0 or i >= buf.count:
        raise CodecError(errc.out_of_range, f"select: index {i} not below count {buf.count}")
    return int(select_batch(buf, [i])[0])
