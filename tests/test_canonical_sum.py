"""The canonical SSE sum's specification (oracle/canon.py) on CPU: it is the
correctly rounded exact sum whenever no partial falls 63+ binades below the
row's largest, it never depends on order or grouping, and it keeps the
IEEE special-value behaviour of a plain sum of non-negative terms.  The
device primitive is checked against it bit for bit in test_gpu_canonical.py."""

from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

from oracle.canon import canonical_rows, canonical_sum


def _exact(v) -> float:
    return float(sum((Fraction(float(x)) for x in v), Fraction(0)))


def test_equals_correctly_rounded_exact_sum():
    rng = np.random.default_rng(0)
    for trial in range(300):
        n = int(rng.integers(1, 400))
        v = rng.lognormal(0.0, 4.0, n) * 10.0 ** rng.integers(-30, 30)   # < 60 binades per row
        assert canonical_sum(v) == _exact(v), trial


def test_order_and_grouping_free():
    rng = np.random.default_rng(1)
    v = rng.lognormal(0.0, 12.0, 5000)
    s = canonical_sum(v)
    for _ in range(5):
        assert canonical_sum(rng.permutation(v)) == s


def test_rounding_ties_and_sticky_bits():
    assert canonical_sum([2.0 ** 53, 1.0]) == 2.0 ** 53                  # tie -> even
    assert canonical_sum([2.0 ** 53, 3.0]) == 2.0 ** 53 + 4.0            # tie -> even (up)
    assert canonical_sum([2.0 ** 53, 1.0, 2.0 ** -60]) == 2.0 ** 53 + 2  # sticky breaks the tie
    assert canonical_sum([1.0, 2.0 ** -53]) == 1.0
    assert canonical_sum([1.0, 2.0 ** -53, 2.0 ** -100]) == 1.0 + 2.0 ** -52


def test_special_values():
    assert canonical_sum([0.0, 0.0]) == 0.0
    assert math.isnan(canonical_sum([1.0, math.nan, math.inf]))
    assert canonical_sum([1.0, math.inf]) == math.inf
    assert canonical_sum([1.7e308, 1.7e308]) == math.inf                 # overflow of the sum
    tiny = 5e-324
    assert canonical_sum([tiny] * 7) == 7 * tiny                         # subnormals are exact
    assert canonical_sum([2.0 ** -1022, tiny]) == 2.0 ** -1022 + tiny
    assert list(canonical_rows([[1.0, 2.0], [0.0, 0.0]])) == [3.0, 0.0]


def test_truncation_bound():
    """Partials more than 116 binades below the largest are dropped; the
    error stays far below one ulp of the sum."""
    v = [1.0] + [2.0 ** -120] * 1000
    assert canonical_sum(v) == 1.0
    assert abs(canonical_sum(v) - _exact(v)) <= 2.0 ** -100
