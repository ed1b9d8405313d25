// C++ drop-in test: a reference-style caller of namespace bytecodec (reference
// proj/core/include/bytecodec/{codec,stream_vbyte}.hpp signatures) linked
// against libbytecodec_b200.so.  Checks SPEC golden vectors (SPEC.md:308-320,
// 372-383, erratum E1), round trips, malformed input errors, the random-access
// API and varint-GB (varint_gb.hpp).  Exit code 0 = pass.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "bytecodec/codec.hpp"
#include "bytecodec/stream_vbyte.hpp"
#include "bytecodec/container.hpp"
#include "bytecodec/query.hpp"
#include "bytecodec/varint_gb.hpp"

using namespace bytecodec;

static int failures = 0;
#define CHECK(cond)                                                       \
    do {                                                                  \
        if (!(cond)) {                                                    \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                   \
        }                                                                 \
    } while (0)

int main() {
    // Fig. 3 values: control [0xC1, 0x40] + 13 data bytes (E1)
    const std::vector<uint32_t> fig3 = {1024, 12, 10, 1073741824, 1, 2, 3, 1024};
    const std::vector<uint8_t> fig3_bytes = {0xC1, 0x40, 0, 4, 12, 10, 0, 0, 0, 64, 1, 2, 3, 0, 4};
    CHECK(svb_encode(fig3) == fig3_bytes);
    CHECK(svb_decode(fig3_bytes, 8) == fig3);
    CHECK(svb_encode(std::vector<uint32_t>{0, 0, 0, 0}) == (std::vector<uint8_t>{0, 0, 0, 0, 0}));
    CHECK(svb_encode(std::vector<uint32_t>{}).empty());
    CHECK(svb_tables().length[0x00] == 4 && svb_tables().length[0xFF] == 16 && svb_tables().length[0xC1] == 8);
    CHECK(byte_length(0) == 1 && byte_length(1024) == 2 && byte_length(1073741824) == 4);

    // delta: prefix of (3,4,12,1) -> (3,7,19,20); base chaining
    {
        const std::vector<uint32_t> xs = {3, 7, 19, 20};
        encoded_buffer b = encode(codec_id::stream_vbyte, xs, true);
        CHECK(b.codec == codec_id::stream_vbyte && b.count == 4 && b.delta);
        CHECK(b.bytes == svb_encode(std::vector<uint32_t>{3, 4, 12, 1}));
        CHECK(decode(b) == xs);
        std::vector<uint32_t> out(4);
        const uint32_t last = decode_payload_delta(codec_id::stream_vbyte, svb_encode(std::vector<uint32_t>{0, 0, 0, 0}),
                                                   4, 42, out.data());
        CHECK(last == 42 && out == (std::vector<uint32_t>{42, 42, 42, 42}));
    }
    // random round trips incl. prev-seeded delta encode (extension E2) and wrap-around
    std::mt19937_64 rng(7);
    for (int it = 0; it < 40; ++it) {
        const size_t n = it < 20 ? (size_t)it : (size_t)(rng() % 200000);
        std::vector<uint32_t> v(n);
        for (auto& x : v) x = (uint32_t)(rng() >> (rng() % 33));
        const auto enc = svb_encode(v);
        CHECK(svb_decode(enc, n) == v);
        const uint32_t prev = (uint32_t)rng();
        const auto encd = svb_encode_delta(v, prev);
        std::vector<uint32_t> out(n);
        const uint32_t last = svb_decode_delta(encd, n, prev, out.data());
        CHECK(out == v);
        CHECK(last == (n ? v.back() : prev));
        // random access: every block through the offset index
        if (n) {
            const auto offs = svb_block_data_offsets(enc, n);
            CHECK(offs.size() == svb_control_bytes(n));
            const size_t k = (size_t)(rng() % offs.size());
            uint32_t blk[4];
            const size_t cnt = svb_decode_block(enc, n, k, offs[k], blk);
            CHECK(cnt == ((k + 1) * 4 <= n ? 4 : n - 4 * k));
            for (size_t i = 0; i < cnt; ++i) CHECK(blk[i] == v[4 * k + i]);
        }
    }
    // malformed input -> codec_error with the reference taxonomy (codec.hpp:28-58)
    {
        const std::vector<uint32_t> v = {1, 300, 70000, 1u << 31, 5};
        auto enc = svb_encode(v);
        std::vector<uint32_t> out(5);
        auto expect_errc = [&](std::vector<uint8_t> bytes, errc want) {
            try {
                svb_decode(bytes, 5, out.data());
                CHECK(false);
            } catch (const codec_error& e) {
                CHECK(e.code() == want);
            }
        };
        expect_errc(std::vector<uint8_t>(enc.begin(), enc.end() - 1), errc::truncated);
        auto longer = enc;
        longer.push_back(0);
        expect_errc(longer, errc::trailing_bytes);
        expect_errc(std::vector<uint8_t>(enc.begin(), enc.begin() + 1), errc::truncated);
        try {
            encode(codec_id::vbyte, v);
            CHECK(false);
        } catch (const codec_error& e) {
            CHECK(e.code() == errc::unsupported);
        }
    }
    // svb_append keeps the one-shot encoding; the SVB1 container round trip
    {
        std::mt19937 rng(11);
        encoded_buffer b = encode(codec_id::stream_vbyte, std::vector<uint32_t>{});
        std::vector<uint32_t> seq;
        for (int i = 0; i < 300; ++i) {
            const uint32_t x = rng() >> (rng() % 32);
            svb_append(b, x);
            seq.push_back(x);
        }
        CHECK(b.count == 300 && b.bytes == svb_encode(seq));
        const std::vector<uint8_t> f = write_container(b);
        CHECK(f.size() == 14 + b.bytes.size() && f[0] == 'S' && f[3] == '1');
        const encoded_buffer r = read_container(f);
        CHECK(r.count == b.count && r.delta == b.delta && r.bytes == b.bytes && r.codec == codec_id::stream_vbyte);
        auto bad = f;
        bad[0] = 'X';
        try {
            read_container(bad);
            CHECK(false);
        } catch (const codec_error& e) {
            CHECK(e.code() == errc::bad_magic);
        }
    }
    // seek / select on a compressed delta buffer
    {
        const encoded_buffer b = encode(codec_id::stream_vbyte, std::vector<uint32_t>{3, 7, 19, 20}, true);
        const auto r = seek(b, 8u);
        CHECK(r && r->index == 2 && r->value == 19);
        CHECK(seek(b, 3u) && seek(b, 3u)->index == 0);
        CHECK(!seek(b, 21u));
        CHECK(select(b, (size_t)1) == 7 && select(b, (size_t)3) == 20);
    }
    // varint-GB: Fig. 1a -> 0xC1 00 04 | 0C | 0A | 00 00 00 40; [5] -> 00 05
    {
        const std::vector<uint32_t> f1a = {1024, 12, 10, 1073741824};
        const std::vector<uint8_t> f1a_bytes = {0xC1, 0x00, 0x04, 0x0C, 0x0A, 0x00, 0x00, 0x00, 0x40};
        CHECK(gb_encode(f1a) == f1a_bytes);
        CHECK(gb_encode(std::vector<uint32_t>{1, 2, 3, 1024}).size() == 6);
        CHECK(gb_encode(std::vector<uint32_t>{5}) == (std::vector<uint8_t>{0x00, 0x05}));
        CHECK(gb_decode(f1a_bytes, 4) == f1a);
        CHECK(gb_decode(std::vector<uint8_t>{0, 1, 2, 3, 4}, 4) == (std::vector<uint32_t>{1, 2, 3, 4}));
        uint32_t g[4] = {};
        const uint8_t grp[] = {1, 2, 3, 4};
        CHECK(detail::gb_decode_group_general(0, grp, grp + 4, 4, g) == grp + 4 && g[3] == 4);
        CHECK(detail::gb_decode_group_general(0xFF, grp, grp + 4, 4, g) == nullptr);
        std::mt19937 rng(5);
        std::vector<uint32_t> v(10001);
        uint32_t acc = 0;
        for (auto& x : v) x = acc += rng() % 5000;
        const encoded_buffer b = encode(codec_id::varint_gb, v, true);
        CHECK(b.codec == codec_id::varint_gb && decode(b) == v);
        std::vector<uint32_t> out(v.size());
        CHECK(gb_decode_delta(gb_encode_delta(v, 0), v.size(), 0, out.data()) == v.back() && out == v);
        const encoded_buffer r = read_container(write_container(b));
        CHECK(r.codec == codec_id::varint_gb && r.bytes == b.bytes);
        auto cut = f1a_bytes;
        cut.pop_back();
        try {
            gb_decode(cut, 4);
            CHECK(false);
        } catch (const codec_error& e) {
            CHECK(e.code() == errc::truncated);
        }
    }
    {  // batch extension: one call == a loop of svb_encode_delta / svb_decode_delta per segment
        std::mt19937 rng(11);
        const std::vector<uint32_t> seg_n = {0, 1, 17, 4000, 3, 70000, 128, 0, 1921};
        std::vector<uint32_t> vals, prev;
        uint32_t acc = 0;
        for (uint32_t n : seg_n) {
            prev.push_back(acc);
            for (uint32_t i = 0; i < n; ++i) vals.push_back(acc += rng() % 3000);
        }
        const svb_batch b = svb_encode_batch(vals, seg_n, prev);
        size_t at = 0;
        for (size_t s = 0; s < seg_n.size(); ++s) {
            const std::vector<uint32_t> seg(vals.begin() + at, vals.begin() + at + seg_n[s]);
            const auto one = svb_encode_delta(seg, prev[s]);
            CHECK(std::vector<uint8_t>(b.bytes.begin() + b.offsets[s], b.bytes.begin() + b.offsets[s + 1]) == one);
            at += seg_n[s];
        }
        std::vector<uint32_t> out(vals.size());
        const auto last = svb_decode_batch(b.bytes, b.offsets, seg_n, prev, out.data());
        CHECK(out == vals && last.size() == seg_n.size() && last[0] == prev[0] && last[5] == vals[4000 + 1 + 17 + 3 + 70000 - 1]);
        auto cut = b.bytes;
        cut.resize(cut.size() - 1);
        try {
            svb_decode_batch(cut, b.offsets, seg_n, prev, out.data());
            CHECK(false);
        } catch (const codec_error& e) {
            CHECK(e.code() == errc::truncated);
        }
    }
    if (failures) {
        std::fprintf(stderr, "%d failures\n", failures);
        return 1;
    }
    std::printf("bytecodec C++ API: all checks passed\n");
    return 0;
}
