"""ORACLE — TEST INFRASTRUCTURE ONLY.

The paper's algorithms written out literally, one statement per line of the
paper's pseudo-code, in Python fp64 (small inputs only), plus exact rational
arithmetic for extended-exponent pairs.  These follow the paper's order and
notation; they are pinned against the plain definition (oracle.softmax) and
against mpmath in tests/test_oracle_pins.py.

  three_pass_recompute  Alg. 1, PAPER.md:88-104 (§3)
  three_pass_reload     Alg. 2, PAPER.md:108-128 (§3)
  two_pass              Alg. 3, PAPER.md:151-174 (§4)
  ext_exp               ExtExp: PAPER.md:143 (range reduction), 149 (pair)
  pair_value / pair_merge_exact
                        (m, n) represents m * 2^n; the Alg. 3
                        update m_sum <- m_i 2^{n_i-n_max} + m_sum 2^{n_sum-n_max}
                         evaluated exactly.
"""
from __future__ import annotations

import math
from fractions import Fraction

LOG2E = 1.0 / math.log(2.0)
LN2 = math.log(2.0)
NEG_INF = float("-inf")


def ext_exp(x: float) -> tuple[float, float]:
    """(m, n) with n = round(x log2 e) and m = e^{x - n ln 2}; no reconstruction."""
    n = float(round(x * LOG2E))
    m = math.exp(x - n * LN2)
    return m, n


def _scale(m: float, k: float) -> float:
    """m * 2^k for integer-valued k <= 0 or k = -inf (identity element)."""
    if k == NEG_INF:
        return 0.0
    return math.ldexp(m, int(k))


def two_pass(X: list[float]) -> list[float]:
    """Alg. 3 SoftmaxTwoPass, literally."""
    N = len(X)
    m_sum = 0.0
    n_sum = NEG_INF
    for i in range(N):                               # Pass 1: read X
        m_i, n_i = ext_exp(X[i])
        n_max = max(n_i, n_sum)
        m_sum = _scale(m_i, n_i - n_max) + _scale(m_sum, n_sum - n_max)
        n_sum = n_max
    lambda_sum = 1.0 / m_sum
    Y = [0.0] * N
    for i in range(N):                               # Pass 2: read X, write Y
        m_i, n_i = ext_exp(X[i])
        Y[i] = _scale(m_i * lambda_sum, n_i - n_sum)
    return Y


def _exp(x: float) -> float:
    return math.exp(x)


def three_pass_recompute(X: list[float]) -> list[float]:
    """Alg. 1 SoftmaxThreePassRecompute, literally."""
    N = len(X)
    mu = max(X)                                      # Pass 1: read X
    sigma = sum(_exp(X[i] - mu) for i in range(N))   # Pass 2: read X
    lam = 1.0 / sigma
    return [lam * _exp(X[i] - mu) for i in range(N)]  # Pass 3: read X, write Y


def three_pass_reload(X: list[float]) -> list[float]:
    """Alg. 2 SoftmaxThreePassReload, literally."""
    N = len(X)
    mu = max(X)                                      # Pass 1: read X
    sigma = 0.0
    Y = [0.0] * N
    for i in range(N):
        Y[i] = _exp(X[i] - mu)                       # Pass 2: read X, write Y
        sigma = sigma + Y[i]
    lam = 1.0 / sigma
    for i in range(N):
        Y[i] = lam * Y[i]                            # Pass 3: read Y, write Y
    return Y


# ---------------------------------------------------------------- exact pairs

def pair_value(m: float, n: float) -> Fraction:
    """Exact value m * 2^n of a pair; (m, -inf) is 0."""
    if n == NEG_INF:
        return Fraction(0)
    assert float(n).is_integer()
    n = int(n)
    return Fraction(m) * (Fraction(2) ** n)


def pair_merge_exact(a: tuple[float, float], b: tuple[float, float]) -> tuple[Fraction, float]:
    """Exact sum of two pairs and the max exponent (Alg. 3 update)."""
    n_max = max(a[1], b[1])
    return pair_value(*a) + pair_value(*b), n_max


def mantissa_exact(value: Fraction, n: float) -> Fraction:
    """m such that m * 2^n = value (the exact mantissa at exponent n)."""
    if n == NEG_INF:
        return Fraction(0)
    return value / (Fraction(2) ** int(n))
