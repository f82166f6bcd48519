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


LIMBS = 4
EXP_ZERO = -0x7F7F7F80        # common.cuh kExpZero / kExpInf / kExpNaN
EXP_INF = 0x7FFFFFF0
EXP_NAN = 0x7FFFFFFF


def anchor(values) -> int:
    """The row's anchor key: max canon_exp over the partials, with the
    special keys for NaN / +inf / all-zero (common.cuh canon_exp)."""
    v = np.asarray(values, dtype=np.float64).ravel()
    if np.isnan(v).any():
        return EXP_NAN
    if np.isinf(v).any():
        return EXP_INF
    nz = v[v > 0.0]
    return max(canon_exp(float(x)) for x in nz) if nz.size else EXP_ZERO


def digits(values, A: int) -> list[int]:
    """Digit-limb sums of floor(v * 2^(116 - A)) (common.cuh canon_add):
    limb d = sum of the 32-bit digits d of every X.  Limb sums are plain
    integer additions, so they can be split over ranks in any grouping."""
    out = [0] * LIMBS
    if A >= EXP_INF or A == EXP_ZERO:
        return out
    for x in np.asarray(values, dtype=np.float64).ravel():
        if x > 0.0:
            X = _fixed(float(x), A)
            for d in range(LIMBS):
                out[d] += (X >> (32 * d)) & 0xFFFFFFFF
    return out


def finish(limbs, A: int) -> float:
    """Round sum(limbs[d] * 2^(32 d)) * 2^(A - 116) once (common.cuh canon_finish)."""
    if A == EXP_NAN:
        return math.nan
    if A == EXP_INF:
        return math.inf
    if A < -1100:
        return 0.0
    return _round_scaled(sum(int(l) << (32 * d) for d, l in enumerate(limbs)), A - ANCHOR)


def canonical_sum(values) -> float:
    """Order-free sum of one row of non-negative fp64 partials."""
    A = anchor(values)
    return finish(digits(values, A), A)


def canonical_rows(M) -> np.ndarray:
    """canonical_sum of every row of a 2-D array."""
    M = np.atleast_2d(np.asarray(M, dtype=np.float64))
    return np.array([canonical_sum(r) for r in M])
