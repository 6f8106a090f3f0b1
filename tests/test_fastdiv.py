"""The kernels' reciprocal divider (csrc/sa_common.cuh FastDiv): q = mulhi(n, ceil(2^32/d)) with one
correction step, d = 1 special-cased.  Host model of the same integer arithmetic, checked against //
and % on edge and random values (the divisors the kernels use: ngroups, H, npairs, ring sizes)."""
import random


def fastdiv(n, d):
    if d == 1:
        return n, 0
    m = ((1 << 32) + d - 1) // d
    assert m < (1 << 32)
    q = (n * m) >> 32
    if n - q * d < 0:
        q -= 1
    r = n - ((n * m) >> 32) * d
    if r < 0:
        r += d
    return q, r


def test_fastdiv_matches_integer_division():
    rng = random.Random(0)
    divisors = list(range(1, 300)) + [1023, 1024, 2048, 4096, 16384, 65536, 131071, 1 << 20, (1 << 31) - 1]
    for d in divisors:
        for n in list(range(0, 600)) + [rng.randrange(0, 1 << 31) for _ in range(300)] + [(1 << 31) - 1]:
            assert fastdiv(n, d) == (n // d, n % d), (n, d)
