"""The integer identities the encoders' group pack relies on (csrc/svb_pack.cuh), checked
exhaustively on the CPU: they replace shift / mask / select chains by multiplies on
byte-packed fields, so a wrong constant would corrupt bytes silently on the GPU.

Reference semantics: control byte field i = byte_length(x_i) - 1 in bits 2i..2i+1
(codec.hpp:70-72)."""
import itertools

M32 = 0xFFFFFFFF


def test_control_byte_from_packed_lengths():
    # group_ctrl: M holds byte_length - 1 of the four integers, one per byte;
    # (M * K) >> 24 gathers them into the control byte, dp4a(M, 1s) + 4 is the data size
    K = 0x01041040
    for m in itertools.product(range(4), repeat=4):
        M = m[0] | m[1] << 8 | m[2] << 16 | m[3] << 24
        c = ((M * K) & M32) >> 24
        assert c == m[0] | m[1] << 2 | m[2] << 4 | m[3] << 6
        assert sum((M >> (8 * i)) & 0xFF for i in range(4)) + 4 == sum(m) + 4


def test_packed_top_bit_indices_to_lengths():
    # group_ctrl: f = index of the top set bit of x | 0x80 (7..31), four packed one per byte;
    # one shift + mask turns them into byte_length - 1
    for f in itertools.product((7, 8, 15, 16, 23, 24, 31), repeat=4):
        F = f[0] + (f[1] << 8) + (f[2] << 16) + (f[3] << 24)
        M = (F >> 3) & 0x03030303
        assert [(M >> (8 * i)) & 0xFF for i in range(4)] == [x >> 3 for x in f]


def test_bit_offsets_from_control_byte():
    # group_bytes: fields spread one per byte by two multiplies, then one multiply gives the
    # running bit offsets 8 l0, 8 (l0 + l1), 8 (l0 + l1 + l2), 8 total
    for c in range(256):
        m = [(c >> (2 * i)) & 3 for i in range(4)]
        L = (((c & 0x33) * 0x1001 + (c & 0xCC) * 0x40040) & 0x03030303) & M32
        assert L == m[0] | m[1] << 8 | m[2] << 16 | m[3] << 24
        P8 = (L * 0x08080808 + 0x20181008) & M32
        ln = [x + 1 for x in m]
        assert [(P8 >> (8 * i)) & 0xFF for i in range(4)] == [8 * sum(ln[: i + 1]) for i in range(4)]


def test_group_concatenation_by_64_bit_shifts():
    # group_bytes: G = A | B << 8 (l0 + l1) with a 64-bit shift left for words 0-1 and a shift
    # right by 64 - 8 (l0 + l1) for words 2-3 (PTX shifts clamp at 64: a shift by 64 gives 0)
    def shl64(x, s):
        return 0 if s >= 64 else (x << s) & 0xFFFFFFFFFFFFFFFF

    def shr64(x, s):
        return 0 if s >= 64 else x >> s

    vals = {1: 0xAB, 2: 0xABCD, 3: 0xABCDEF, 4: 0xABCDEF12}
    for ln in itertools.product(range(1, 5), repeat=4):
        x = [vals[l] ^ (i * 0x11 & ((1 << (8 * l)) - 1) & 0x7F) for i, l in enumerate(ln)]
        A = x[0] + (x[1] << (8 * ln[0]))
        B = x[2] + (x[3] << (8 * ln[2]))
        la8 = 8 * (ln[0] + ln[1])
        lo = (A + shl64(B, la8)) & 0xFFFFFFFFFFFFFFFF  # the sum never carries: the bits are disjoint
        hi = shr64(B, 64 - la8)
        G = lo | hi << 64
        want = 0
        pos = 0
        for v, l in zip(x, ln):
            want |= v << pos
            pos += 8 * l
        assert G == want, (ln, hex(G), hex(want))
