// ref_inline_pins.cpp -- emits golden values computed by the REFERENCE's own
// inline code: byte_length / vbyte_length (codec.hpp:69-81), svb_control_bytes
// (stream_vbyte.hpp:34) and svb_shuffle_fill (stream_vbyte.hpp:22).  These are
// the only executable definitions the headers-only reference contains
// (SURVEY.md §0, §8(c)); everything else in it is declaration-only.
// Built and run by oracle/pin/make_ref_pins.sh against /root/reference (this
// container only); the JSON it prints is committed as tests/golden/ref_inline_pins.json.
#include <cstdint>
#include <cstdio>

#include "bytecodec/codec.hpp"
#include "bytecodec/stream_vbyte.hpp"

static uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

int main() {
    using namespace bytecodec;
    std::printf("{\n  \"source\": \"reference headers proj/core/include/bytecodec/{codec,stream_vbyte}.hpp\",\n");
    std::printf("  \"svb_shuffle_fill\": %u,\n", (unsigned)svb_shuffle_fill);
    // boundary values and their neighbours
    const uint64_t bounds[] = {0, 1, 127, 128, 129, 255, 256, 257, 16383, 16384, 16385, 65535, 65536, 65537,
                               2097151, 2097152, 2097153, 16777215, 16777216, 16777217, 268435455, 268435456,
                               268435457, 1024, 1073741824, 4294967294ull, 4294967295ull};
    std::printf("  \"byte_length\": [");
    bool first = true;
    for (uint64_t b : bounds) {
        std::printf("%s[%llu, %u]", first ? "" : ", ", (unsigned long long)b, byte_length((uint32_t)b));
        first = false;
    }
    std::printf("],\n  \"vbyte_length\": [");
    first = true;
    for (uint64_t b : bounds) {
        std::printf("%s[%llu, %u]", first ? "" : ", ", (unsigned long long)b, vbyte_length((uint32_t)b));
        first = false;
    }
    // random values: x = mix(i) >> (mix(i) & 31) spans all byte-length classes
    std::printf("],\n  \"byte_length_random\": {\"count\": 4096, \"values\": [");
    for (int i = 0; i < 4096; ++i) {
        const uint64_t r = mix(0x9E3779B97F4A7C15ull * (i + 1));
        const uint32_t x = (uint32_t)(r >> 32) >> (r & 31);
        std::printf("%s[%u, %u]", i ? ", " : "", x, byte_length(x));
    }
    std::printf("]},\n  \"svb_control_bytes\": [");
    const uint64_t ns[] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 15, 16, 17, 1000, 1048576, 67108864, 268435456,
                           2147483648ull, 4294967295ull};
    first = true;
    for (uint64_t n : ns) {
        std::printf("%s[%llu, %zu]", first ? "" : ", ", (unsigned long long)n, svb_control_bytes((size_t)n));
        first = false;
    }
    std::printf("]\n}\n");
    return 0;
}
