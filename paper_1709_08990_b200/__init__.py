"""B200-native Stream VByte (arXiv 1709.08990) behind the reference's bytecodec API.

- ``codec``  : the reference operator API (codec_id, errc, encode/decode, svb_*), host arrays
- ``device`` : stream-ordered device API over CUDA tensors (batches, offsets, blocks)
- ``gen``    : seeded synthetic inputs for the BASELINE.json configs

The compute lives in ``lib/libbytecodec_b200.so`` (sm_100a CUDA kernels behind
the C ABI of ``include/bcgpu/bcgpu.h``); importing this package fails loudly
when that library is missing.
"""
from . import _native  # noqa: F401  (loads the native library or raises)
from .codec import (CodecError, EncodedBuffer, GpuError, byte_length, codec_id, decode, decode_payload,
                    decode_payload_delta, encode, encode_payload, errc, svb_block_data_offsets, svb_control_bytes,
                    svb_decode, svb_decode_block, svb_decode_blocks, svb_decode_delta, svb_encode, svb_encode_delta,
                    svb_encode_batch, svb_decode_batch, svb_max_compressed_bytes, svb_tables, svb_append, svb_payload_length, write_container,
                    read_container, seek, seek_batch, select, select_batch, gb_encode, gb_encode_delta, gb_decode,
                    gb_decode_delta)

__all__ = [
    "CodecError", "EncodedBuffer", "GpuError", "byte_length", "codec_id", "decode", "decode_payload",
    "decode_payload_delta", "encode", "encode_payload", "errc", "svb_block_data_offsets", "svb_control_bytes",
    "svb_decode", "svb_decode_block", "svb_decode_blocks", "svb_decode_delta", "svb_encode", "svb_encode_delta",
    "svb_encode_batch", "svb_decode_batch", "svb_max_compressed_bytes", "svb_tables", "svb_append", "svb_payload_length", "write_container",
    "read_container", "seek", "seek_batch", "select", "select_batch", "gb_encode", "gb_encode_delta", "gb_decode",
    "gb_decode_delta",
]
