"""Shared seeded inputs for the parity tests (no reference files at run time)."""
from fractions import Fraction
import random


def random_pd_hankel(seed: int, n: int, f: int) -> list[int]:
    """Positive definite Hankel strip: moments of a discrete measure with n
    distinct positive dyadic nodes, truncated to f fractional bits -- the
    construction of the reference's tests (tests/test_ldlt.cpp:25-44),
    restated with a Python PRNG."""
    rng = random.Random(seed)
    nodes = [Fraction(1 + rng.randrange(64) + l * 64, 16) for l in range(n)]
    weights = [Fraction(1 + rng.randrange(255), 256) for _ in range(n)]
    strip = []
    for s in range(2 * n - 1):
        mu = sum(wt * nd ** s for wt, nd in zip(weights, nodes))
        num = mu.numerator << f
        q = abs(num) // mu.denominator
        strip.append(q if num >= 0 else -q)
    return strip


def strip_from_ints(vals: list[int], f: int) -> list[int]:
    """strip_matrix (tests/test_ldlt.cpp:16-21): integers at f frac bits."""
    return [v << f for v in vals]
