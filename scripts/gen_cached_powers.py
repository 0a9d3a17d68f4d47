"""Generate the cached powers of ten for include/wgpf_grisu2.h: c_k = 10^k as
a normalised 64-bit significand f (bit 63 set, rounded to nearest) and a
binary exponent e with 10^k ~= f * 2^e, for k = -300, -292, ..., 324 (step 8
covers every binary exponent Grisu2 meets for doubles: Loitsch 2010, sec. 5)."""
from fractions import Fraction


def cached(k):
    v = Fraction(10) ** k
    e = 0
    # scale into [2^63, 2^64)
    while v >= 2 ** 64:
        v /= 2
        e += 1
    while v < 2 ** 63:
        v *= 2
        e -= 1
    f = int(v)
    rem = v - f
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and f % 2):
        f += 1
    if f == 2 ** 64:
        f //= 2
        e += 1
    return f, e


rows = []
for k in range(-300, 325, 8):
    f, e = cached(k)
    rows.append(f"    {{0x{f:016X}ull, {e}, {k}}},")
print("\n".join(rows))
print(len(rows))
