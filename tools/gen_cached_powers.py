"""Generates the Grisu2 cached powers of ten used by the records writer (host/records.cpp) and
the oracle (oracle/records_ref.py): c_k = 10^k as a normalized 64-bit significand f and binary
exponent e (f * 2^e ~ 10^k, 2^63 <= f < 2^64, f rounded to nearest), k = -300, -292, ..., 324
(step 8), exact rational arithmetic (dev tool; prints the C++ table)."""
from fractions import Fraction


def cached_powers():
    out = []
    for k in range(-300, 325, 8):
        v = Fraction(10) ** k
        e = v.numerator.bit_length() - v.denominator.bit_length() - 64
        while v / Fraction(2) ** e >= 2 ** 64:
            e += 1
        while v / Fraction(2) ** e < 2 ** 63:
            e -= 1
        q = v / Fraction(2) ** e
        f = int(q)
        if q - f >= Fraction(1, 2):
            f += 1
        if f == 2 ** 64:
            f, e = 2 ** 63, e + 1
        out.append((f, e, k))
    return out


if __name__ == "__main__":
    rows = cached_powers()
    for i in range(0, len(rows), 3):
        print("    " + " ".join("{0x%016X, %d, %d}," % r for r in rows[i:i + 3]))
