"""Hand-derived pins for the oracle's bit-level helpers.

Every expected value below is worked out by hand from the IEEE-754 encodings
(binary32: 1 sign, 8 exponent, 23 fraction bits; bfloat16 = the top 16 bits of
binary32) or from the definitions of DESIGN.md readings R8 / R17 -- none of them
is computed by the function under test or by the CUDA path.

* f32_to_bf16_bits: round-to-nearest-even of binary32 to bfloat16 (the stored
  target rule of reading R17 / SURVEY O4).  The kept part is bits 31..16,
  the discarded half-ulp is 0x8000 of the low 16 bits.
* normalise_f32 / normalise_inputs: (v - 100)/400 and t/tau (reading R17 / Q13).
* unit_double: u = (r64 >> 11) * 2^-53 (reading R8), the draw behind init_params.
"""
import struct

import numpy as np
import pytest

from oracle import mlp, philox
from oracle import reservoir as ores


def f32(bits: int) -> np.float32:
    return np.frombuffer(struct.pack("<I", bits), dtype=np.float32)[0]


# (binary32 bits, expected bfloat16 bits, why)
BF16_CASES = [
    (0x3F800000, 0x3F80, "1.0 is exact"),
    (0x3F807FFF, 0x3F80, "just below the half-ulp: round down"),
    (0x3F808000, 0x3F80, "exact tie, kept lsb 0 (even): stays"),
    (0x3F808001, 0x3F81, "just above the half-ulp: round up"),
    (0x3F818000, 0x3F82, "exact tie, kept lsb 1 (odd): up to even"),
    (0x3F81FFFF, 0x3F82, "above the half-ulp: round up"),
    (0x3FFF8000, 0x4000, "tie at the largest mantissa, odd: carry into the exponent (2.0)"),
    (0x3FFFFFFF, 0x4000, "mantissa all ones: carry into the exponent (2.0)"),
    (0x3EAAAAAB, 0x3EAB, "1/3: remainder 0xAAAB > 0x8000 rounds up (0.333984375)"),
    (0x7F7F0000, 0x7F7F, "largest finite bfloat16 (3.3895e38), exact"),
    (0x7F7F7FFF, 0x7F7F, "below the tie under 2^128: largest finite stays"),
    (0x7F7F8000, 0x7F80, "tie, odd lsb 0x7F7F: rounds to +inf (RNE overflow)"),
    (0x7F7FFFFF, 0x7F80, "binary32 max rounds up past the largest finite bf16 to +inf"),
    (0x00000000, 0x0000, "+0"),
    (0x80000000, 0x8000, "-0 keeps its sign"),
    (0xBF800000, 0xBF80, "-1.0"),
    (0xBF808000, 0xBF80, "negative tie, even: magnitude stays"),
    (0xBF818000, 0xBF82, "negative tie, odd: magnitude rounds up (away from 0)"),
    (0xBFFFFFFF, 0xC000, "negative carry into the exponent (-2.0)"),
    (0x00008000, 0x0000, "subnormal tie, even: to +0"),
    (0x00018000, 0x0002, "subnormal tie, odd: up"),
    (0x007FFFFF, 0x0080, "largest subnormal rounds up to the smallest normal bf16"),
]


@pytest.mark.parametrize("bits,want,why", BF16_CASES)
def test_f32_to_bf16_bits_hand_cases(bits, want, why):
    got = int(ores.f32_to_bf16_bits(np.array([f32(bits)], dtype=np.float32))[0])
    assert got == want, "%08x -> %04x, want %04x (%s)" % (bits, got, want, why)


def test_bf16_bits_to_f64_hand_values():
    # 0x3EAB: exponent 0x7D = 125 -> 2^-2, fraction 0x2B = 43/128 -> 0.25 * 171/128
    assert ores.bf16_bits_to_f64(np.array([0x3EAB], np.uint16))[0] == 0.333984375
    # 0x7F7F: 2^127 * (1 + 127/128) = 2^127 * 255/128
    assert ores.bf16_bits_to_f64(np.array([0x7F7F], np.uint16))[0] == 2.0 ** 127 * 255 / 128
    assert ores.bf16_bits_to_f64(np.array([0xC000], np.uint16))[0] == -2.0


def test_stored_payload_bf16_rule_hand_value():
    # u = 300 K: (300 - 100)/400 = 0.5 = 0x3F000000 -> bf16 0x3F00 exactly;
    # u = 140 K: 40/400 = 0.1 -> binary32 RN(0.1) = 0x3DCCCCCD -> bf16: kept 0x3DCC,
    # remainder 0xCCCD > 0x8000 -> 0x3DCD
    got = ores.stored_payload(np.array([300.0, 140.0], np.float32), ores.STORE_BF16)
    assert [int(x) for x in got] == [0x3F00, 0x3DCD]


def test_normalise_f32_hand_values():
    got = ores.normalise_f32(np.array([300.0, 100.0, 500.0, 140.0, 0.0, 900.0], np.float32))
    assert got.dtype == np.float32
    bits = [int(x) for x in got.view(np.uint32)]
    # 0.5, +0, 1.0, RN32(0.1), -0.25, 2.0
    assert bits == [0x3F000000, 0x00000000, 0x3F800000, 0x3DCCCCCD, 0xBE800000, 0x40000000]


def test_normalise_f32_uses_fp32_ops():
    # u = 100.1f = 0x42C83333 = 100.09999847412109375 exactly.  u - 100 is exact
    # (Sterbenz): 0.09999847412109375 = 0x3DCCCC00.  The binary32 quotient by 400 is
    # the exact rational d/400 rounded to 24 significant bits, ties to even; it is
    # worked out below with integers (long division of the significand), independent
    # of numpy's float arithmetic.
    u = f32(0x42C83333)
    d = np.float32(u) - np.float32(100.0)
    assert int(np.array([d], np.float32).view(np.uint32)[0]) == 0x3DCCCC00
    got = int(ores.normalise_f32(np.array([u], np.float32)).view(np.uint32)[0])
    num = 0x3DCCCC00 & 0x7FFFFF | 0x800000          # 24-bit significand of d
    e = ((0x3DCCCC00 >> 23) & 0xFF) - 127 - 23       # d = num * 2^e
    # q = num * 2^e / 400; pick k so that num * 2^k // 400 has 24 significant bits
    k = 0
    while (num << k) // 400 < (1 << 23):
        k += 1
    qi, rem = divmod(num << k, 400)
    if 2 * rem > 400 or (2 * rem == 400 and qi & 1):
        qi += 1
    exp = e - k + 23 + 127                            # q = qi * 2^(e-k), qi in [2^23, 2^24)
    want = (exp << 23) | (qi & 0x7FFFFF)
    assert got == want


def test_normalise_inputs_hand_values():
    xn = mlp.normalise_inputs(np.array([[300.0, 100.0, 500.0, 140.0, 0.0]], np.float32), np.array([50]), 100)
    assert xn.shape == (1, 6)
    assert xn[0, 0] == 0.5 and xn[0, 1] == 0.0 and xn[0, 2] == 1.0 and xn[0, 4] == -0.25
    assert xn[0, 3] == 0.1                 # computed in fp64: (140 - 100)/400 = RN64(0.1)
    assert xn[0, 5] == 0.5                 # t / tau = 50 / 100
    xn = mlp.normalise_inputs(np.array([[100.0] * 5], np.float32), np.array([1]), 4)
    assert xn[0, 5] == 0.25 and not xn[0, :5].any()


@pytest.mark.parametrize("r,want", [
    (0, 0.0),
    (2 ** 63, 0.5),                         # (2^63 >> 11) 2^-53 = 2^52 2^-53
    (2 ** 64 - 1, 1.0 - 2.0 ** -53),        # (2^53 - 1) 2^-53: the largest value, < 1
    (2 ** 11, 2.0 ** -53),                  # the smallest non-zero value
    (2 ** 11 - 1, 0.0),                     # the 11 discarded bits never count
    (3 << 62, 0.75),
    ((1 << 64) - (1 << 11), 1.0 - 2.0 ** -53),
])
def test_unit_double_hand_values(r, want):
    got = float(philox.unit_double(np.array([r], dtype=np.uint64))[0])
    assert got == want
