"""ctypes binding of the C ABI (include/bcgpu/bcgpu.h) in lib/libbytecodec_b200.so.

The shared library is the product: CUDA kernels for sm_100a behind an
``extern "C"`` surface.  There is no CPU fallback -- if the library is missing
this module raises at import time, and every compute call needs a GPU.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_DIR = PKG_DIR / "lib"
LIB_PATH = LIB_DIR / "libbytecodec_b200.so"


class NativeLibraryMissing(ImportError):
    pass


def _load(path: Path) -> C.CDLL:
    if not path.exists():
        raise NativeLibraryMissing(
            f"{path} not found: build it with `make` at the repo root or "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    return C.CDLL(str(path), mode=os.RTLD_NOW | C.RTLD_GLOBAL)


class DecodeSegment(C.Structure):
    """bcgpu_decode_segment (bcgpu.h)."""
    _fields_ = [("src_offset", C.c_uint64), ("src_bytes", C.c_uint64), ("dst_offset", C.c_uint64),
                ("n", C.c_uint32), ("prev", C.c_uint32)]


class EncodeSegment(C.Structure):
    """bcgpu_encode_segment (bcgpu.h)."""
    _fields_ = [("src_offset", C.c_uint64), ("dst_capacity", C.c_uint64), ("dst_offset", C.c_uint64),
                ("n", C.c_uint32), ("prev", C.c_uint32)]


_vp, _sz, _u32, _u64, _int = C.c_void_p, C.c_size_t, C.c_uint32, C.c_uint64, C.c_int

# name -> (restype, argtypes); this table is also the export list the CPU tests check
SIGNATURES = {
    "bcgpu_abi_version": (_int, []),
    "bcgpu_ctx_create": (_int, [_int, C.POINTER(_vp)]),
    "bcgpu_ctx_destroy": (_int, [_vp]),
    "bcgpu_ctx_sync_status": (_int, [_vp, _vp]),
    "bcgpu_status_string": (C.c_char_p, [_int]),
    "bcgpu_last_cuda_error": (C.c_char_p, []),
    "bcgpu_kernel_launch_count": (_u64, []),
    "bcgpu_byte_length": (_u32, [_u32]),
    "bcgpu_svb_control_bytes": (_sz, [_sz]),
    "bcgpu_svb_max_compressed_bytes": (_sz, [_sz]),
    "bcgpu_svb_tables": (None, [_vp, _vp]),
    "bcgpu_svb_encode_device": (_int, [_vp, _vp, _sz, _int, _u32, _vp, _sz, _vp, _vp]),
    "bcgpu_svb_decode_device": (_int, [_vp, _vp, _sz, _sz, _int, _u32, _vp, _vp, _vp]),
    "bcgpu_svb_block_offsets_device": (_int, [_vp, _vp, _sz, _sz, _vp, _vp]),
    "bcgpu_svb_decode_blocks_device": (_int, [_vp, _vp, _sz, _sz, _vp, _vp, _sz, _vp, _vp, _vp]),
    "bcgpu_svb_decode_batch_device": (_int, [_vp, _vp, _sz, _vp, _vp, _int, _u32, _vp]),
    "bcgpu_svb_encode_batch_device": (_int, [_vp, _vp, _sz, _vp, _vp, _vp, _int, _u32, _vp]),
    "bcgpu_svb_encoded_sizes_batch_device": (_int, [_vp, _vp, _sz, _vp, _vp, _int, _u32, _vp]),
    "bcgpu_svb_encode_host": (_int, [_vp, _vp, _sz, _int, _u32, _vp, _sz, C.POINTER(_sz)]),
    "bcgpu_svb_decode_host": (_int, [_vp, _vp, _sz, _sz, _int, _u32, _vp, C.POINTER(_u32)]),
    "bcgpu_svb_decode_blocks_host": (_int, [_vp, _vp, _sz, _sz, _vp, _vp, _sz, _vp, _vp]),
    "bcgpu_svb_block_offsets_host": (_int, [_vp, _vp, _sz, _sz, _vp]),
    "bcgpu_svb_encode_batch_host": (_int, [_vp, _vp, _vp, _vp, _sz, _int, _vp, _sz, _vp]),
    "bcgpu_svb_decode_batch_host": (_int, [_vp, _vp, _sz, _vp, _vp, _vp, _sz, _int, _vp, _vp]),
    "bcgpu_svb_seek_batch_device": (_int, [_vp, _vp, _sz, _sz, _u32, _vp, _sz, _vp, _vp, _vp]),
    "bcgpu_svb_select_batch_device": (_int, [_vp, _vp, _sz, _sz, _u32, _vp, _sz, _vp, _vp]),
    "bcgpu_svb_seek_host": (_int, [_vp, _vp, _sz, _sz, _u32, _vp, _sz, _vp, _vp]),
    "bcgpu_svb_select_host": (_int, [_vp, _vp, _sz, _sz, _u32, _vp, _sz, _vp]),
    "bcgpu_gb_encode_device": (_int, [_vp, _vp, _sz, _int, _u32, _vp, _sz, _vp, _vp]),
    "bcgpu_gb_decode_device": (_int, [_vp, _vp, _sz, _sz, _int, _u32, _vp, _vp, _vp]),
    "bcgpu_gb_encode_host": (_int, [_vp, _vp, _sz, _int, _u32, _vp, _sz, C.POINTER(_sz)]),
    "bcgpu_gb_decode_host": (_int, [_vp, _vp, _sz, _sz, _int, _u32, _vp, C.POINTER(_u32)]),
    "bcgpu_svb_payload_length": (_int, [_vp, _sz, _sz, C.POINTER(_sz)]),
    "bcgpu_svb_append": (_int, [_vp, _sz, _sz, _sz, _u32, C.POINTER(_sz)]),
    "bcgpu_container_write": (_int, [C.c_uint8, _int, _sz, _vp, _sz, _vp, _sz, C.POINTER(_sz)]),
    "bcgpu_container_read": (_int, [_vp, _sz, C.POINTER(C.c_uint8), C.POINTER(_int), C.POINTER(_u32),
                                    C.POINTER(_sz), C.POINTER(_sz)]),
}

lib = _load(LIB_PATH)
for _name, (_res, _args) in SIGNATURES.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

ERRC_NAMES = ["truncated", "trailing_bytes", "run_too_long", "value_overflow", "oversized_integer",
              "count_mismatch", "bad_stream_size", "bad_magic", "unknown_codec", "reserved_flags",
              "length_mismatch", "unsupported", "out_of_range", "io_failure", "bad_config"]


def status_string(st: int) -> str:
    return lib.bcgpu_status_string(st).decode()


def last_cuda_error() -> str:
    return lib.bcgpu_last_cuda_error().decode()


def kernel_launch_count() -> int:
    return int(lib.bcgpu_kernel_launch_count())
