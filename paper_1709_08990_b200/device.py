"""Stream-ordered device API over CUDA tensors (the C ABI's ``*_device`` calls).

Tensors are plain torch CUDA tensors used as device memory: uint32 values may
be held in ``torch.int32`` or ``torch.uint32`` storage (bit-identical), byte
streams in ``torch.uint8``.  Calls are asynchronous on the given stream
(default: torch's current stream); malformed input is reported by
:meth:`DeviceCodec.check` (``bcgpu_ctx_sync_status``).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native
from ._native import lib
from .codec import _check

DECODE_SEG_DTYPE = np.dtype([("src_offset", "<u8"), ("src_bytes", "<u8"), ("dst_offset", "<u8"),
                             ("n", "<u4"), ("prev", "<u4")])
ENCODE_SEG_DTYPE = np.dtype([("src_offset", "<u8"), ("dst_capacity", "<u8"), ("dst_offset", "<u8"),
                             ("n", "<u4"), ("prev", "<u4")])
assert DECODE_SEG_DTYPE.itemsize == C.sizeof(_native.DecodeSegment) == 32
assert ENCODE_SEG_DTYPE.itemsize == C.sizeof(_native.EncodeSegment) == 32


def _ptr(t) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("DeviceCodec expects CUDA tensors")
    return t.data_ptr()


def _stream(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def segments_to_tensor(segs: np.ndarray, device) -> torch.Tensor:
    """Structured segment array (DECODE/ENCODE_SEG_DTYPE) -> device uint8 tensor."""
    raw = np.ascontiguousarray(segs).view(np.uint8)
    return torch.from_numpy(raw.copy()).to(device)


class DeviceCodec:
    """One bcgpu_ctx (device workspace + look-back status) bound to a CUDA device."""

    def __init__(self, device: int | torch.device = 0):
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        p = C.c_void_p()
        _check(lib.bcgpu_ctx_create(self.device.index or 0, C.byref(p)), "bcgpu_ctx_create")
        self._ctx = p.value

    def close(self) -> None:
        if self._ctx:
            lib.bcgpu_ctx_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- single array ---------------------------------------------------
    def encode(self, values: torch.Tensor, out: torch.Tensor, out_len: torch.Tensor, *, n: int | None = None,
               delta: bool = False, prev: int = 0, stream=None) -> None:
        """svb_encode / prev-seeded delta encode into ``out`` (capacity >= ceil(n/4)+4n);
        the exact length lands in ``out_len`` (int64/uint64 CUDA scalar)."""
        n = values.numel() if n is None else n
        _check(lib.bcgpu_svb_encode_device(self._ctx, _ptr(values), n, int(delta), prev & 0xFFFFFFFF, _ptr(out),
                                           out.numel() * out.element_size(), _ptr(out_len), _stream(stream)),
               "svb_encode")

    def decode(self, data: torch.Tensor, n: int, out: torch.Tensor, *, in_len: int | None = None,
               delta: bool = False, base: int = 0, last: torch.Tensor | None = None, stream=None) -> None:
        """svb_decode / svb_decode_delta of ``data[:in_len]`` into ``out``."""
        in_len = data.numel() if in_len is None else in_len
        _check(lib.bcgpu_svb_decode_device(self._ctx, _ptr(data), in_len, n, int(delta), base & 0xFFFFFFFF,
                                           _ptr(out), _ptr(last), _stream(stream)), "svb_decode")

    def gb_encode(self, values: torch.Tensor, out: torch.Tensor, out_len: torch.Tensor, *, n: int | None = None,
                  delta: bool = False, prev: int = 0, stream=None) -> None:
        """varint-GB encode (varint_gb.hpp:19; delta: transform seeded with prev first) into ``out``
        (capacity >= ceil(n/4)+4n); the exact length lands in ``out_len``."""
        n = values.numel() if n is None else n
        _check(lib.bcgpu_gb_encode_device(self._ctx, _ptr(values), n, int(delta), prev & 0xFFFFFFFF, _ptr(out),
                                          out.numel() * out.element_size(), _ptr(out_len), _stream(stream)),
               "gb_encode")

    def gb_decode(self, data: torch.Tensor, n: int, out: torch.Tensor, *, in_len: int | None = None,
                  delta: bool = False, base: int = 0, last: torch.Tensor | None = None, stream=None) -> None:
        """gb_decode / gb_decode_delta (varint_gb.hpp:21-25) of ``data[:in_len]`` into ``out``."""
        in_len = data.numel() if in_len is None else in_len
        _check(lib.bcgpu_gb_decode_device(self._ctx, _ptr(data), in_len, n, int(delta), base & 0xFFFFFFFF,
                                          _ptr(out), _ptr(last), _stream(stream)), "gb_decode")

    def block_offsets(self, data: torch.Tensor, n: int, out: torch.Tensor, *, in_len: int | None = None,
                      stream=None) -> None:
        in_len = data.numel() if in_len is None else in_len
        _check(lib.bcgpu_svb_block_offsets_device(self._ctx, _ptr(data), in_len, n, _ptr(out), _stream(stream)),
               "svb_block_data_offsets")

    def decode_blocks(self, data: torch.Tensor, n: int, blocks: torch.Tensor, offsets: torch.Tensor,
                      out: torch.Tensor, counts: torch.Tensor, *, in_len: int | None = None, stream=None) -> None:
        in_len = data.numel() if in_len is None else in_len
        _check(lib.bcgpu_svb_decode_blocks_device(self._ctx, _ptr(data), in_len, n, _ptr(blocks), _ptr(offsets),
                                                  blocks.numel(), _ptr(out), _ptr(counts), _stream(stream)),
               "svb_decode_block")

    # ---- segmented batches ----------------------------------------------
    def decode_batch(self, segs: torch.Tensor, nseg: int, data: torch.Tensor, out: torch.Tensor, *,
                     delta: bool = False, max_seg_n: int = 0, stream=None) -> None:
        _check(lib.bcgpu_svb_decode_batch_device(self._ctx, _ptr(segs), nseg, _ptr(data), _ptr(out), int(delta),
                                                 max_seg_n, _stream(stream)), "svb_decode_batch")

    def encode_batch(self, segs: torch.Tensor, nseg: int, values: torch.Tensor, out: torch.Tensor,
                     out_lens: torch.Tensor, *, delta: bool = False, max_seg_n: int = 0, stream=None) -> None:
        _check(lib.bcgpu_svb_encode_batch_device(self._ctx, _ptr(segs), nseg, _ptr(values), _ptr(out),
                                                 _ptr(out_lens), int(delta), max_seg_n, _stream(stream)),
               "svb_encode_batch")

    def encoded_sizes_batch(self, segs: torch.Tensor, nseg: int, values: torch.Tensor, out_lens: torch.Tensor, *,
                            delta: bool = False, stream=None) -> None:
        _check(lib.bcgpu_svb_encoded_sizes_batch_device(self._ctx, _ptr(segs), nseg, _ptr(values), _ptr(out_lens),
                                                        int(delta), 0, _stream(stream)), "svb_encoded_sizes")

    def check(self, stream=None) -> None:
        """Synchronise and raise CodecError if the last call saw malformed input."""
        _check(lib.bcgpu_ctx_sync_status(self._ctx, _stream(stream)), "device status")
