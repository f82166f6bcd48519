"""Python restatement of the engine's canonical SSE sum (TEST INFRASTRUCTURE ONLY).

The reference sums a row's squared errors left to right (R:fitness.py:23,
`np.cumsum(d * d)[-1]`); the device engine sums them per case tile in a fixed
order and then combines the tile partials with the order-free canonical sum
of `paper_2106_04034_b200/csrc/common.cuh` (canon_exp / canon_add /
canon_finish), so the result is the same for any split of the tiles over
shards and GPUs.  There is no reference counterpart for this step: the
function below is the specification the device primitive is checked against
bit for bit (tests/test_canonical_sum.py, tests/test_gpu_canonical.py), with
Python integers standing in for the u64 digit limbs.

Definition, for non-negative partials v_j of one row:
  * any NaN -> NaN; else any +inf -> +inf; all zero -> 0.0;
  * A = max_j ilogb(v_j) (exact exponent, subnormals included);
  * X_j = floor(v_j * 2^(116 - A)) (an integer < 2^117);
  * result = round_to_nearest_even(sum_j X_j * 2^(A - 116)), rounded to 53
    bits first and then scaled (the device's ldexp; a second rounding only
    happens for subnormal results).
"""

from __future__ import annotations

import math

import numpy as np

ANCHOR = 116


def canon_exp(v: float) -> int:
    """ilogb(v) for finite v > 0 (common.cuh canon_exp)."""
    m, e = math.frexp(v)          # v = m * 2^e, 0.5 <= m < 1
    return e - 1


def _fixed(v: float, A: int) -> int:
    """floor(v * 2^(ANCHOR - A)) (common.cuh canon_add)."""
    m, e = math.frexp(v)
    M = int(m * (1 << 53))        # exact: v = M * 2^(e - 53)
    sh = e - 53 + ANCHOR - A
    return M << sh if sh >= 0 else M >> (-sh)


def _round_scaled(S: int, scale: int) -> float:
    """S * 2^scale rounded like common.cuh canon_finish."""
    if S == 0:
        return 0.0
    h = S.bit_length() - 1
    if h <= 52:
        mant, e = S, 0
    else:
        drop = h - 52
        mant = S >> drop
        rem = S & ((1 << drop) - 1)
        half = 1 << (drop - 1)
        if rem > half or (rem == half and (mant & 1)):
            mant += 1
            if mant == 1 << 53:
                mant >>= 1
                drop += 1
        e = drop
    try:
        return math.ldexp(float(mant), e + scale)
    except OverflowError:
        return math.inf


def canonical_sum(values) -> float:
    """Order-free sum of one row of non-negative fp64 partials."""
    v = np.asarray(values, dtype=np.float64).ravel()
    if np.isnan(v).any():
        return math.nan
    if np.isinf(v).any():
        return math.inf
    nz = [float(x) for x in v if x > 0.0]
    if not nz:
        return 0.0
    A = max(canon_exp(x) for x in nz)
    S = sum(_fixed(x, A) for x in nz)
    return _round_scaled(S, A - ANCHOR)


def canonical_rows(M) -> np.ndarray:
    """canonical_sum of every row of a 2-D array."""
    M = np.atleast_2d(np.asarray(M, dtype=np.float64))
    return np.array([canonical_sum(r) for r in M])
