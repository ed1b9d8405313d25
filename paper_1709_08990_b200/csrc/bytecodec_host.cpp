// bytecodec_host.cpp -- the reference's C++ API (namespace bytecodec) on top of
// the C ABI.  Signatures: reference proj/core/include/bytecodec/codec.hpp:24-96
// stream_vbyte.hpp:32-54 and varint_gb.hpp:19-31; semantics: SPEC.md:164-214, 270-402.
//
// Each host thread owns one bcgpu_ctx per device (a ctx is single-stream).
// Errors from the GPU path surface as codec_error{errc} exactly where the
// reference would throw.
#include <map>
#include <memory>
#include <mutex>
#include <cstddef>
#include <stdexcept>
#include <string>

#include "bcgpu/bcgpu.h"
#include "bytecodec/codec.hpp"
#include "bytecodec/stream_vbyte.hpp"
#include "bytecodec/container.hpp"
#include "bytecodec/query.hpp"
#include "bytecodec/varint_gb.hpp"

namespace bytecodec {
namespace {

thread_local int t_device = 0;

struct CtxHolder {
    std::map<int, bcgpu_ctx*> by_dev;
    ~CtxHolder() {
        for (auto& kv : by_dev) bcgpu_ctx_destroy(kv.second);
    }
};
thread_local CtxHolder t_ctx;

[[noreturn]] void throw_status(int st, const char* where) {
    std::string msg = std::string(where) + ": " + bcgpu_status_string(st);
    if (st >= 1 && st <= 15) throw codec_error(static_cast<errc>(st - 1), msg);
    if (st == BCGPU_ERR_CUDA) msg += std::string(" (") + bcgpu_last_cuda_error() + ")";
    throw std::runtime_error(msg);
}

bcgpu_ctx* ctx() {
    auto it = t_ctx.by_dev.find(t_device);
    if (it != t_ctx.by_dev.end()) return it->second;
    bcgpu_ctx* c = nullptr;
    const int st = bcgpu_ctx_create(t_device, &c);
    if (st) throw_status(st, "bcgpu_ctx_create");
    t_ctx.by_dev[t_device] = c;
    return c;
}

void require_svb(codec_id id) {
    if (id != codec_id::stream_vbyte)
        throw codec_error(errc::unsupported, "this operation is defined for codec_id::stream_vbyte only");
}

// the codecs with a GPU path: Stream VByte and varint-GB
void require_gpu_codec(codec_id id) {
    if (id != codec_id::stream_vbyte && id != codec_id::varint_gb)
        throw codec_error(errc::unsupported, "only stream_vbyte and varint_gb are implemented on the GPU path");
}

std::vector<uint8_t> gb_encode_impl(std::span<const uint32_t> values, bool delta, uint32_t prev) {
    std::vector<uint8_t> out(bcgpu_svb_max_compressed_bytes(values.size()));
    size_t len = 0;
    const int st = bcgpu_gb_encode_host(ctx(), values.data(), values.size(), delta ? 1 : 0, prev, out.data(),
                                        out.size(), &len);
    if (st) throw_status(st, "gb_encode");
    out.resize(len);
    out.shrink_to_fit();
    return out;
}

std::vector<uint8_t> encode_impl(std::span<const uint32_t> values, bool delta, uint32_t prev) {
    std::vector<uint8_t> out(bcgpu_svb_max_compressed_bytes(values.size()));
    size_t len = 0;
    const int st = bcgpu_svb_encode_host(ctx(), values.data(), values.size(), delta ? 1 : 0, prev, out.data(),
                                         out.size(), &len);
    if (st) throw_status(st, "svb_encode");
    out.resize(len);
    out.shrink_to_fit();
    return out;
}

}  // namespace

void set_device(int device) { t_device = device; }

std::string_view codec_name(codec_id id) {
    switch (id) {
        case codec_id::vbyte: return "vbyte";
        case codec_id::varint_gb: return "varint-gb";
        case codec_id::varint_g8iu: return "varint-g8iu";
        case codec_id::stream_vbyte: return "stream-vbyte";
    }
    return "unknown";
}

std::optional<codec_id> codec_from_name(std::string_view name) {
    for (uint8_t t = 0; t < 4; ++t)
        if (codec_name(static_cast<codec_id>(t)) == name) return static_cast<codec_id>(t);
    return std::nullopt;
}

std::optional<codec_id> codec_from_tag(uint8_t tag) {
    if (tag < 4) return static_cast<codec_id>(tag);
    return std::nullopt;
}

const decode_tables& svb_tables() {
    static const decode_tables tables = [] {
        decode_tables t{};
        uint8_t len[256];
        uint8_t shuf[256][16];
        bcgpu_svb_tables(len, shuf);
        for (int c = 0; c < 256; ++c) {
            t.length[c] = len[c];
            for (int i = 0; i < 16; ++i) t.shuffle[c][i] = shuf[c][i];
        }
        return t;
    }();
    return tables;
}

std::vector<uint8_t> svb_encode(std::span<const uint32_t> values) { return encode_impl(values, false, 0); }

std::vector<uint8_t> svb_encode_delta(std::span<const uint32_t> values, uint32_t prev) {
    return encode_impl(values, true, prev);
}

void svb_decode(std::span<const uint8_t> bytes, size_t n, uint32_t* out) {
    const int st = bcgpu_svb_decode_host(ctx(), bytes.data(), bytes.size(), n, 0, 0, out, nullptr);
    if (st) throw_status(st, "svb_decode");
}

std::vector<uint32_t> svb_decode(std::span<const uint8_t> bytes, size_t n) {
    std::vector<uint32_t> out(n);
    svb_decode(bytes, n, out.data());
    return out;
}

uint32_t svb_decode_delta(std::span<const uint8_t> bytes, size_t n, uint32_t base, uint32_t* out) {
    uint32_t last = base;
    const int st = bcgpu_svb_decode_host(ctx(), bytes.data(), bytes.size(), n, 1, base, out, &last);
    if (st) throw_status(st, "svb_decode_delta");
    return last;
}

std::vector<size_t> svb_block_data_offsets(std::span<const uint8_t> bytes, size_t n) {
    std::vector<uint64_t> tmp(svb_control_bytes(n));
    const int st = bcgpu_svb_block_offsets_host(ctx(), bytes.data(), bytes.size(), n, tmp.data());
    if (st) throw_status(st, "svb_block_data_offsets");
    return std::vector<size_t>(tmp.begin(), tmp.end());
}

size_t svb_decode_block(std::span<const uint8_t> bytes, size_t n, size_t block, size_t data_offset,
                        uint32_t out[4]) {
    uint32_t cnt = 0;
    const int st = bcgpu_svb_decode_blocks_host(ctx(), bytes.data(), bytes.size(), n, &block, &data_offset, 1, out,
                                                &cnt);
    if (st) throw_status(st, "svb_decode_block");
    return cnt;
}

svb_batch svb_encode_batch(std::span<const uint32_t> values, std::span<const uint32_t> seg_n,
                           std::span<const uint32_t> seg_prev, bool delta) {
    if (!seg_prev.empty() && seg_prev.size() != seg_n.size())
        throw std::invalid_argument("svb_encode_batch: seg_prev must be empty or hold one base per segment");
    size_t total = 0, cap = 0;
    for (uint32_t n : seg_n) {
        total += n;
        cap += bcgpu_svb_max_compressed_bytes(n);
    }
    if (total != values.size()) throw std::invalid_argument("svb_encode_batch: sum(seg_n) != values.size()");
    svb_batch b;
    b.bytes.resize(cap);
    b.offsets.resize(seg_n.size() + 1);
    const int st = bcgpu_svb_encode_batch_host(ctx(), values.data(), seg_n.data(),
                                               seg_prev.empty() ? nullptr : seg_prev.data(), seg_n.size(),
                                               delta ? 1 : 0, b.bytes.data(), b.bytes.size(), b.offsets.data());
    if (st) throw_status(st, "svb_encode_batch");
    b.bytes.resize(b.offsets.back());
    return b;
}

std::vector<uint32_t> svb_decode_batch(std::span<const uint8_t> bytes, std::span<const uint64_t> offsets,
                                       std::span<const uint32_t> seg_n, std::span<const uint32_t> seg_base,
                                       uint32_t* out, bool delta) {
    if (offsets.size() != seg_n.size() + 1)
        throw std::invalid_argument("svb_decode_batch: offsets must hold seg_n.size() + 1 entries");
    if (!seg_base.empty() && seg_base.size() != seg_n.size())
        throw std::invalid_argument("svb_decode_batch: seg_base must be empty or hold one base per segment");
    std::vector<uint32_t> last(seg_n.size());
    const int st = bcgpu_svb_decode_batch_host(ctx(), bytes.data(), bytes.size(), offsets.data(), seg_n.data(),
                                               seg_base.empty() ? nullptr : seg_base.data(), seg_n.size(),
                                               delta ? 1 : 0, out, last.data());
    if (st) throw_status(st, "svb_decode_batch");
    return last;
}

void svb_append(encoded_buffer& buf, uint32_t value) {
    require_svb(buf.codec);
    const size_t len = buf.bytes.size();
    buf.bytes.resize(len + 5);  // worst case: a new control byte + 4 data bytes
    size_t new_len = 0;
    const int st = bcgpu_svb_append(buf.bytes.data(), len, buf.bytes.size(), buf.count, value, &new_len);
    if (st) {
        buf.bytes.resize(len);
        throw_status(st, "svb_append");
    }
    buf.bytes.resize(new_len);
    buf.count += 1;
}

std::vector<uint8_t> write_container(const encoded_buffer& buf) {
    std::vector<uint8_t> out(BCGPU_CONTAINER_HEADER + buf.bytes.size());
    size_t n = 0;
    const int st = bcgpu_container_write(static_cast<uint8_t>(buf.codec), buf.delta ? 1 : 0, buf.count,
                                         buf.bytes.data(), buf.bytes.size(), out.data(), out.size(), &n);
    if (st) throw_status(st, "write_container");
    out.resize(n);
    return out;
}

encoded_buffer read_container(std::span<const uint8_t> src) {
    uint8_t tag = 0;
    int delta = 0;
    uint32_t count = 0;
    size_t off = 0, plen = 0;
    const int st = bcgpu_container_read(src.data(), src.size(), &tag, &delta, &count, &off, &plen);
    if (st) throw_status(st, "read_container");
    encoded_buffer b;
    b.codec = static_cast<codec_id>(tag);
    b.count = count;
    b.delta = delta != 0;
    b.bytes.assign(src.begin() + (std::ptrdiff_t)off, src.begin() + (std::ptrdiff_t)(off + plen));
    return b;
}

static void require_delta(const encoded_buffer& buf) {
    require_svb(buf.codec);
    if (!buf.delta) throw codec_error(errc::unsupported, "seek / select need a delta-coded buffer");
}

std::vector<std::optional<seek_result>> seek(const encoded_buffer& buf, std::span<const uint32_t> targets) {
    require_delta(buf);
    std::vector<uint64_t> idx(targets.size());
    std::vector<uint32_t> val(targets.size());
    const int st = bcgpu_svb_seek_host(ctx(), buf.bytes.data(), buf.bytes.size(), buf.count, 0, targets.data(),
                                       targets.size(), idx.data(), val.data());
    if (st) throw_status(st, "seek");
    std::vector<std::optional<seek_result>> out(targets.size());
    for (size_t i = 0; i < targets.size(); ++i)
        if (idx[i] < buf.count) out[i] = seek_result{(size_t)idx[i], val[i]};
    return out;
}

std::optional<seek_result> seek(const encoded_buffer& buf, uint32_t target) {
    return seek(buf, std::span<const uint32_t>(&target, 1))[0];
}

std::vector<uint32_t> select(const encoded_buffer& buf, std::span<const size_t> indices) {
    require_delta(buf);
    std::vector<uint64_t> idx(indices.begin(), indices.end());
    std::vector<uint32_t> val(indices.size());
    const int st = bcgpu_svb_select_host(ctx(), buf.bytes.data(), buf.bytes.size(), buf.count, 0, idx.data(),
                                         idx.size(), val.data());
    if (st) throw_status(st, "select");
    return val;
}

uint32_t select(const encoded_buffer& buf, size_t i) { return select(buf, std::span<const size_t>(&i, 1))[0]; }

// ---- varint-GB (varint_gb.hpp) ----
std::vector<uint8_t> gb_encode(std::span<const uint32_t> values) { return gb_encode_impl(values, false, 0); }

std::vector<uint8_t> gb_encode_delta(std::span<const uint32_t> values, uint32_t prev) {
    return gb_encode_impl(values, true, prev);
}

void gb_decode(std::span<const uint8_t> bytes, size_t n, uint32_t* out) {
    const int st = bcgpu_gb_decode_host(ctx(), bytes.data(), bytes.size(), n, 0, 0, out, nullptr);
    if (st) throw_status(st, "gb_decode");
}

std::vector<uint32_t> gb_decode(std::span<const uint8_t> bytes, size_t n) {
    std::vector<uint32_t> out(n);
    gb_decode(bytes, n, out.data());
    return out;
}

uint32_t gb_decode_delta(std::span<const uint8_t> bytes, size_t n, uint32_t base, uint32_t* out) {
    uint32_t last = base;
    const int st = bcgpu_gb_decode_host(ctx(), bytes.data(), bytes.size(), n, 1, base, out, &last);
    if (st) throw_status(st, "gb_decode_delta");
    return last;
}

namespace detail {
const uint8_t* gb_decode_group_general(uint8_t control, const uint8_t* data, const uint8_t* end, size_t k,
                                       uint32_t* out) {
    for (size_t i = 0; i < k && i < 4; ++i) {
        const uint32_t l = ((control >> (2 * i)) & 3u) + 1u;
        if (end - data < static_cast<std::ptrdiff_t>(l)) return nullptr;
        uint32_t x = 0;
        for (uint32_t b = 0; b < l; ++b) x |= static_cast<uint32_t>(data[b]) << (8 * b);
        out[i] = x;
        data += l;
    }
    return data;
}
}  // namespace detail

// ---- codec-generic (codec.hpp:84-96): Stream VByte and varint-GB ----
std::vector<uint8_t> encode_payload(codec_id id, std::span<const uint32_t> values) {
    require_gpu_codec(id);
    return id == codec_id::varint_gb ? gb_encode(values) : svb_encode(values);
}

void decode_payload(codec_id id, std::span<const uint8_t> bytes, size_t n, uint32_t* out) {
    require_gpu_codec(id);
    if (id == codec_id::varint_gb)
        gb_decode(bytes, n, out);
    else
        svb_decode(bytes, n, out);
}

uint32_t decode_payload_delta(codec_id id, std::span<const uint8_t> bytes, size_t n, uint32_t base, uint32_t* out) {
    require_gpu_codec(id);
    return id == codec_id::varint_gb ? gb_decode_delta(bytes, n, base, out) : svb_decode_delta(bytes, n, base, out);
}

encoded_buffer encode(codec_id id, std::span<const uint32_t> values, bool delta) {
    require_gpu_codec(id);
    if (values.size() > 0xFFFFFFFFull) throw codec_error(errc::out_of_range, "count exceeds uint32");
    encoded_buffer b;
    b.codec = id;
    b.count = static_cast<uint32_t>(values.size());
    b.delta = delta;
    // base 0
    b.bytes = id == codec_id::varint_gb ? gb_encode_impl(values, delta, 0) : encode_impl(values, delta, 0);
    return b;
}

std::vector<uint32_t> decode(const encoded_buffer& buf) {
    require_gpu_codec(buf.codec);
    std::vector<uint32_t> out(buf.count);
    if (buf.delta)
        decode_payload_delta(buf.codec, buf.bytes, buf.count, 0, out.data());
    else
        decode_payload(buf.codec, buf.bytes, buf.count, out.data());
    return out;
}

}  // namespace bytecodec
