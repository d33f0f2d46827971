"""Cached powers of ten for the Grisu2 digit generator in csrc/serialize.cu:
10^k = f * 2^e with f a 64-bit significand in [2^63, 2^64) rounded to nearest,
k = -300, -292, ..., 324 (exact rational arithmetic).  Prints the C++ rows."""
from fractions import Fraction


def cached(k):
    v = Fraction(10) ** k
    e = v.numerator.bit_length() - v.denominator.bit_length() - 64
    while True:
        q = v / Fraction(2) ** e if e >= 0 else v * Fraction(2) ** (-e)
        if q < 2 ** 63:
            e -= 1
        elif q >= 2 ** 64:
            e += 1
        else:
            break
    f = q.numerator // q.denominator
    if q - f >= Fraction(1, 2):
        f += 1
    if f == 2 ** 64:
        f, e = f // 2, e + 1
    return f, e


if __name__ == "__main__":
    for i in range(79):
        k = -300 + 8 * i
        f, e = cached(k)
        print(f"    {{0x{f:016X}ull, {e}, {k}}},")
