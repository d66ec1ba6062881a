"""Regenerates the cached-power table of include/roomray_b200_artifacts.hpp:
10^k for k = -300, -292, ..., 324 as a 64-bit significand f in [2^63, 2^64)
and binary exponent e (10^k ~= f * 2^e, rounded to nearest, ties to even),
the table Grisu2 (Loitsch 2010) indexes by binary exponent."""
from fractions import Fraction


def power(k):
    x = Fraction(10) ** k
    e = x.numerator.bit_length() - x.denominator.bit_length() - 64
    while True:
        q = x / Fraction(2) ** e
        if q >= 2 ** 64:
            e += 1
        elif q < 2 ** 63:
            e -= 1
        else:
            break
    f = int(q)
    rem = q - f
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and f % 2):
        f += 1
    if f == 2 ** 64:
        f, e = f // 2, e + 1
    return f, e


if __name__ == "__main__":
    rows = [power(k) + (k,) for k in range(-300, 325, 8)]
    for i in range(0, len(rows), 3):
        print("      " + " ".join(f"{{0x{f:016X}ull, {e}, {k}}}," for f, e, k in rows[i:i + 3]))
