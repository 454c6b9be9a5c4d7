"""Pins for the oracle (-m "not gpu").

The oracle is checked against things other than itself: closed forms of the
softmax definition, its invariants, mpmath brute force at 50 digits, a second
independent formula, the paper's literal algorithms, and values the paper
states (tests/golden/paper_facts.json).  Each test names the passage it pins.
"""
import json
import math
import os
from fractions import Fraction

import mpmath
import numpy as np
import pytest

import oracle
import workloads
from oracle import algorithms as alg

mpmath.mp.dps = 50
LD = np.longdouble


def mp_softmax(x):
    """Brute-force softmax at 50 digits (PAPER.md:31 definition, no shift)."""
    xs = [mpmath.mpf(float(v)) for v in x]
    e = [mpmath.e ** v for v in xs]
    s = mpmath.fsum(e)
    return [v / s for v in e]


def f32(a):
    return np.asarray(a, np.float32)


# ------------------------------------------------------------------ closed forms

def test_single_element_is_one():
    for v in [0.0, 1.0, -1e4, 1e4, 88.7, -103.9, 3.4e38, -3.4e38]:
        o = oracle.softmax(f32([v]))
        assert o[0] == LD(1), v


@pytest.mark.parametrize("n", [1, 2, 3, 7, 1000, 4097])
@pytest.mark.parametrize("c", [0.0, 88.0, -1e4, 1e4, 123.456])
def test_constant_row_is_exactly_one_over_n(n, c):
    o = oracle.softmax(np.full(n, c, np.float32))
    assert np.all(o == LD(1) / LD(n))


@pytest.mark.parametrize("a,b", [(0.0, 1.0), (1.0, 0.0), (-3.5, 2.25), (100.0, -100.0),
                                 (1e4, 1e4 - 20.0), (-1e4, -1e4 + 0.5), (88.0, 89.0)])
def test_two_elements_logistic(a, b):
    o = oracle.softmax(f32([a, b]))
    av, bv = float(np.float32(a)), float(np.float32(b))
    want0 = 1 / (1 + mpmath.e ** (mpmath.mpf(bv) - mpmath.mpf(av)))
    assert abs(float(o[0]) - float(want0)) <= 1e-15 * float(want0) + 1e-300
    want1 = 1 / (1 + mpmath.e ** (mpmath.mpf(av) - mpmath.mpf(bv)))
    assert abs(float(o[1]) - float(want1)) <= 1e-15 * float(want1) + 1e-300


def test_one_two_three():
    # [1,2,3] -> 0.0900305731703805, 0.244728471054798, 0.665240955774822 (SPEC.md:211-213 decimals,
    # corrected to full precision by the closed form e^i / (e + e^2 + e^3))
    o = oracle.softmax(f32([1, 2, 3])).astype(np.float64)
    e = math.e
    s = e + e * e + e ** 3
    np.testing.assert_allclose(o, [e / s, e * e / s, e ** 3 / s], rtol=1e-15)
    np.testing.assert_allclose(o, [0.0900305731703805, 0.244728471054798, 0.665240955774822],
                               rtol=1e-14)


@pytest.mark.parametrize("n,d", [(2, 5.0), (10, -30.0), (1000, 80.0), (1000, 1e4)])
def test_zeros_then_d(n, d):
    x = np.zeros(n, np.float32)
    x[-1] = d
    o = oracle.softmax(x)
    ed = mpmath.e ** mpmath.mpf(d)
    want_last = ed / (n - 1 + ed)
    want_zero = 1 / (n - 1 + ed)
    assert abs(mpmath.mpf(float(o[-1])) - want_last) <= 1e-15 * want_last
    assert abs(mpmath.mpf(float(o[0])) - want_zero) <= 1e-15 * want_zero + mpmath.mpf(1e-300)


def test_huge_spread_row():
    o = oracle.softmax(f32([10000, 0, -10000]))
    assert o[0] == LD(1)
    assert float(o[1]) == 0.0 and float(o[2]) == 0.0  # e^{-1e4} underflows fp64 exp: true value 1.1e-4343


def test_equal_values_at_fp32_overflow_edge():
    o = oracle.softmax(f32([88, 88, 88, 88]))
    assert np.all(o == LD(0.25))


# ------------------------------------------------------------------ invariants

def _rows():
    yield workloads.generate("c1")[0]
    for lo, hi, n in [(-1e4, 1e4, 5000), (-5, 5, 333), (-200, 300, 4096)]:
        yield workloads.uniform(n, lo, hi, seed=1, stream=n)


def test_sum_is_one():
    for x in _rows():
        o = oracle.softmax(x)
        assert abs(float(np.sum(o, dtype=np.longdouble)) - 1.0) <= x.size * 2.0 ** -60


def test_shift_invariance_exact_on_integer_grid():
    # integer x and integer c with |x + c| < 2^24 are exact in fp32, so x - mu is identical:
    # the oracle must be bitwise shift-invariant (PAPER.md:80 holds for any c).
    rng = np.random.default_rng(5)
    x = rng.integers(-3000, 3000, size=2000).astype(np.float32)
    base = oracle.softmax(x)
    for c in [1.0, -777.0, 12345.0, 1 << 20]:
        assert np.array_equal(oracle.softmax((x + np.float32(c)).astype(np.float32)), base)


def test_monotone_and_permutation_equivariant():
    x = workloads.uniform(3000, -100, 100, seed=3, stream=9)
    o = oracle.softmax(x)
    order = np.argsort(x, kind="stable")
    assert np.all(np.diff(o[order].astype(np.float64)) >= 0)
    perm = np.random.default_rng(1).permutation(x.size)
    # S is summed in a different order, so equal up to long-double rounding of the sum
    p = oracle.softmax(np.ascontiguousarray(x[perm]))
    assert np.all(np.abs(p - o[perm]) <= LD(1e-17) * o[perm])


def test_shifted_and_unshifted_formulas_agree():
    # P3: max-subtracted fp64/long-double vs unshifted long-double expl, |x| <= 1e4 < ln(LDBL_MAX)
    for x in _rows():
        a = oracle.softmax(x)
        b = oracle.softmax_unshifted(x)
        big = a > LD(1e-300)
        rel = np.abs((a[big] - b[big]) / a[big]).astype(np.float64)
        assert rel.max() <= 1e-13
        assert np.all(np.abs(a[~big] - b[~big]) <= LD(1e-300))


ADVERSARIAL = [
    [1e4, -1e4, 0.0, 1e4],
    [88.7228, 88.7228, -103.972, 0.0],
    [-103.97208, -103.97208, -103.97208],
    [89.0, 90.0, 91.0, -104.0, -105.0],
    [0.5, 0.5, 0.5, 0.5, 0.5, 0.5, 0.5, 0.5, -0.5, -0.5, -0.5, -0.5, -0.5, -0.5, -0.5, -0.5],
    [-1e4 + 0.25, -1e4, -1e4 - 0.25],
    [3.0, -7.0, 11.5, 0.0, -0.0, 1e-30, -1e-30, 42.0],
    [700.0, 720.0, 740.0, 745.0],
]


@pytest.mark.parametrize("x", ADVERSARIAL)
def test_mpmath_brute_force(x):
    # P4: 50-digit brute force on N <= 16 adversarial vectors
    x32 = f32(x)
    o = oracle.softmax(x32)
    want = mp_softmax(x32)
    for oi, wi in zip(o, want):
        if wi > mpmath.mpf(1e-300):
            assert abs(mpmath.mpf(float(oi)) - wi) <= mpmath.mpf(2e-16) * wi
        else:
            assert float(oi) <= 1e-300


# ------------------------------------------------------------------ literal algorithms (Alg. 1-3)

@pytest.mark.parametrize("fn", [alg.two_pass, alg.three_pass_recompute, alg.three_pass_reload])
def test_literal_algorithms_match_definition(fn):
    for x in list(_rows())[:3] + [f32(v) for v in ADVERSARIAL]:
        xs = [float(v) for v in x[:2000]]
        got = np.array(fn(xs), np.float64)
        want = oracle.softmax(f32(xs)).astype(np.float64)
        big = want > 1e-290
        np.testing.assert_allclose(got[big], want[big], rtol=5e-12)
        assert np.all(np.abs(got[~big]) <= 1e-290)


def test_two_pass_literal_never_overflows():
    # "m values are never scaled up" -- Alg. 3 stays finite where e^x overflows fp64
    xs = [800.0, 1000.0, 5000.0, 1e4, 1e4]
    y = alg.two_pass(xs)
    assert all(math.isfinite(v) for v in y)
    assert abs(sum(y) - 1.0) < 1e-12
    with pytest.raises(OverflowError):
        math.exp(xs[1])  # the naive e^x of the same inputs overflows fp64


# ------------------------------------------------------------------ ExtExp definition

EXTEXP_TABLE = [0.0, 1.0, -1.0, 10.0, 100.0, -100.0, 200.0, -200.0, 1000.0, -1000.0, 1e4, -1e4,
                88.72283935546875, -103.97207641601562, 0.6931471824645996]


def test_extexp_definition_against_mpmath():
    x = f32(EXTEXP_TABLE + list(workloads.uniform(500, -1e4, 1e4, seed=2, stream=3)))
    m, n = oracle.extexp(x)
    for xi, mi, ni in zip(x, m, n):
        xm = mpmath.mpf(float(xi))
        nn = mpmath.nint(xm / mpmath.log(2))
        assert ni == float(nn)
        want = mpmath.e ** (xm - nn * mpmath.log(2))
        assert abs(mpmath.mpf(float(mi)) - want) <= mpmath.mpf(1e-15) * want  # float() of long double
        assert math.sqrt(2) / 2 * (1 - 1e-12) <= float(mi) <= math.sqrt(2) * (1 + 1e-12)


def test_extexp_known_values():
    # x = 0 -> (1, 0); x = 10 -> n = 14, t = 0.2959394722 (SPEC.md:115's 0.29449 is wrong)
    m, n = oracle.extexp(f32([0.0, 10.0, 200.0]))
    assert n[0] == 0 and m[0] == LD(1)
    assert n[1] == 14 and abs(float(m[1]) - math.exp(10 - 14 * math.log(2))) < 1e-15
    assert abs(10 - 14 * math.log(2) - 0.2959394722) < 1e-10
    assert n[2] == 289 and abs(float(m[2]) - 0.7264866428) < 1e-9


# ------------------------------------------------------------------ exact pair arithmetic

def test_pair_merge_examples():
    ninf = float("-inf")
    v, n = alg.pair_merge_exact((0.0, ninf), (1.0, 5.0))
    assert (v, n) == (Fraction(32), 5.0) and alg.mantissa_exact(v, n) == 1
    v, n = alg.pair_merge_exact((1.0, 3.0), (1.0, 3.0))
    assert alg.mantissa_exact(v, n) == 2 and n == 3.0
    v, n = alg.pair_merge_exact((1.5, 10.0), (1.0, 0.0))
    assert alg.mantissa_exact(v, n) == Fraction(3, 2) + Fraction(1, 1024) and n == 10.0
    v, n = alg.pair_merge_exact((1.0, 128.0), (1.0, -128.0))
    assert alg.mantissa_exact(v, n) == 1 + Fraction(1, 2 ** 256)
    assert float(alg.mantissa_exact(v, n)) == 1.0  # rounds to 1.0 in binary32/64
    v, n = alg.pair_merge_exact((0.0, ninf), (0.0, ninf))
    assert v == 0 and n == ninf


# ------------------------------------------------------------------ paper facts (golden)

def test_paper_overflow_underflow_thresholds(golden_dir):
    facts = json.load(open(os.path.join(golden_dir, "paper_facts.json")))
    hi = facts["exp_overflow_threshold"]["value"]
    lo = facts["exp_underflow_threshold"]["value"]
    with np.errstate(over="ignore", under="ignore"):
        assert np.isinf(np.exp(np.float32(hi)))           # overflows above 89 (exact edge 88.7228)
        assert np.isfinite(np.exp(np.float32(88.72)))
        assert np.exp(np.float32(lo)) == 0.0               # underflows below -104 (edge -103.972)
        assert np.exp(np.float32(-103.0)) > 0.0
    # m range of the reduced exponential
    m, _ = oracle.extexp(workloads.uniform(20000, -1e4, 1e4, seed=4, stream=4))
    assert float(m.min()) >= math.sqrt(2) / 2 - 1e-12 and float(m.max()) <= math.sqrt(2) + 1e-12


def test_naive_fp32_softmax_fails_on_c1_but_oracle_is_finite():
    # PAPER.md:76 / SPEC.md:407: naive fp32 e^x overflows on config 1, the oracle does not
    x = workloads.generate("c1")[0]
    assert int(np.sum(x > 88.7228)) > 0
    with np.errstate(over="ignore", invalid="ignore"):
        e = np.exp(x)
        naive = e / e.sum()
    assert not np.all(np.isfinite(naive))
    o = oracle.softmax(x)
    assert np.all(np.isfinite(o.astype(np.float64)))
    assert abs(float(o.sum()) - 1) < 1e-15


def test_cost_model_fixture(golden_dir):
    c = json.load(open(os.path.join(golden_dir, "paper_facts.json")))["cost_model"]
    for k in ("three_pass_recompute", "three_pass_reload", "two_pass"):
        assert c[k]["reads"] + c[k]["writes"] == c[k]["total"]
    tp = c["two_pass"]["total"]
    # Table 2: Recompute moves 4N, Reload 5N, Two-Pass 3N element transfers, i.e. 4/3 and 5/3
    assert Fraction(c["three_pass_recompute"]["total"], tp) == Fraction(4, 3)
    assert Fraction(c["three_pass_reload"]["total"], tp) == Fraction(5, 3)
    assert abs(c["three_pass_recompute"]["total"] / tp - 1 - c["advantage_vs_recompute"]) < 0.01
    assert abs(c["three_pass_reload"]["total"] / tp - 1 - c["advantage_vs_reload"]) < 0.01


# ------------------------------------------------------------------ the checker itself

def test_checker_accepts_rounded_oracle_and_rejects_perturbations():
    x = workloads.generate("c1")[0]
    o = oracle.softmax(x)
    y = o.astype(np.float32)
    r = oracle.check(x, y)
    assert r.ok and r.n_rel + r.n_abs == x.size and r.n_rel > 0 and r.n_abs > 0
    i = int(np.argmax(o))
    y2 = y.copy()
    y2[i] *= np.float32(1 + 3e-5)
    assert oracle.check(x, y2).n_bad == 1 and oracle.check(x, y2).first_bad == i
    small = np.nonzero((o < LD(oracle.FLT_MIN)) & (o > 0))[0]
    y3 = y.copy()
    y3[small[0]] = np.float32(float(o[small[0]]) + 2e-37)
    assert oracle.check(x, y3).n_bad == 1
    y4 = y.copy()
    y4[3] = np.nan
    assert oracle.check(x, y4).n_bad == 1


def test_bf16_oracle_equals_f32_oracle_on_converted_values():
    x = workloads.generate("c4b", 0, 1, 0, 5000)[0]
    xf = workloads.bf16_to_f32(x)
    assert np.array_equal(oracle.softmax(x), oracle.softmax(xf))
    mu_b, S_b = oracle.row_stats(x)
    mu_f, S_f = oracle.row_stats(xf)
    assert mu_b == mu_f and S_b == S_f


# ------------------------------------------------------------------ exp_scaled, ext_exp's n, ulp32
# (the checkers of the GPU ExtExp / Exp unit tests and of the accuracy sweep, §4)

def _mp_ld(v):
    """Exact mpmath value of a numpy long double (64-bit significand = two doubles)."""
    fr, ex = np.frexp(np.longdouble(v))  # fr in [0.5, 1): no double overflow / underflow
    hi = float(fr)
    return mpmath.ldexp(mpmath.mpf(hi) + mpmath.mpf(float(fr - np.longdouble(hi))), int(ex))


def _mp_nint_log2e(x):
    """Nearest integer to the EXACT product x log2 e (x a binary32 value), at 50 digits."""
    return int(mpmath.nint(mpmath.mpf(float(x)) / mpmath.log(2)))


def _near_half_integer_x(count, lim, seed):
    """binary32 x whose exact x log2 e lies as close as binary32 allows to a half-integer
    k + 1/2 (both binary32 neighbours of (k + 1/2) ln 2), |x| <= lim."""
    rng = np.random.default_rng(seed)
    kmax = int(lim / math.log(2)) - 1
    ks = rng.integers(-kmax, kmax, count)
    xs = []
    for k in ks:
        t = float((mpmath.mpf(int(k)) + mpmath.mpf(0.5)) * mpmath.log(2))
        c = np.float32(t)
        xs += [c, np.nextafter(c, np.float32(np.inf)), np.nextafter(c, np.float32(-np.inf))]
    return np.array(xs, np.float32)


def test_exp_scaled_against_mpmath():
    # oracle.exp_scaled(x, k) = e^{x - k ln 2} (the value a pair (m, k) must carry)
    # graded at 50 digits for k = nint(x log2 e), that k +- 1, and k = 0, over |x| <= 2^21 (the
    # accuracy domain, reading G11) including x log2 e next to half-integers
    lim = float(2 ** 21)
    x = np.concatenate([f32(EXTEXP_TABLE), workloads.uniform(150, -lim, lim, seed=7, stream=1),
                        workloads.uniform(150, -100.0, 100.0, seed=7, stream=2),
                        _near_half_integer_x(60, lim, seed=3)])
    ln2 = mpmath.log(2)
    for dk in (0, 1, -1, None):
        if dk is None:  # k = 0: plain e^x, inside long double's range only (|x| < 11356)
            sel = x[np.abs(x) < 11000]
            k = np.zeros(sel.size)
        else:
            sel = x
            k = np.array([_mp_nint_log2e(v) + dk for v in sel], np.float64)
        got = oracle.exp_scaled(sel, k)
        for xi, ki, gi in zip(sel, k, got):
            want = mpmath.e ** (mpmath.mpf(float(xi)) - int(ki) * ln2)
            # long double: the argument x - k ln2 carries |k| * 2^-64-ish absolute error
            tol = mpmath.mpf(2e-18) * (1 + abs(int(ki)))
            assert abs(_mp_ld(gi) - want) <= tol * want + mpmath.mpf(1e-300), (xi, ki, gi)
    # the scaling is by 2^-k exactly: k and k+1 differ by a factor of 2 (a sign or scale slip fails)
    a = oracle.exp_scaled(f32([3.0, -7.5, 1000.0]), np.array([1.0, -2.0, 1443.0]))
    b = oracle.exp_scaled(f32([3.0, -7.5, 1000.0]), np.array([2.0, -1.0, 1444.0]))
    assert np.all(np.abs(a / (2 * b) - 1) < LD(1e-15))
    assert oracle.exp_scaled(f32([0.0]), np.array([0.0]))[0] == LD(1)
    assert oracle.exp_scaled(f32([0.0]), np.array([-3.0]))[0] == LD(8)


def test_ext_exp_exponent_is_nearest_integer_of_exact_product():
    # n = round(x log2 e); both oracle ExtExps (C long double, Python fp64 literal
    # Alg. 3) against the nearest integer of the EXACT product at 50 digits, including x whose
    # product lies next to a half-integer, where a floor / ceil / truncation would differ
    lim = float(2 ** 21)
    x = np.concatenate([f32(EXTEXP_TABLE), workloads.uniform(200, -lim, lim, seed=8, stream=1),
                        _near_half_integer_x(300, lim, seed=5),
                        _near_half_integer_x(100, 200.0, seed=6)])
    want = np.array([_mp_nint_log2e(v) for v in x], np.float64)
    _, n_c = oracle.extexp(x)
    assert np.array_equal(n_c, want)
    n_py = np.array([alg.ext_exp(float(v))[1] for v in x])
    assert np.array_equal(n_py, want)
    # fractional parts both sides of 1/2 occur (so rounding direction is really exercised)
    frac = np.array([float(mpmath.mpf(float(v)) / mpmath.log(2) - mpmath.floor(mpmath.mpf(float(v)) / mpmath.log(2)))
                     for v in x])
    assert np.any((frac > 0.5) & (frac < 0.5 + 1e-6)) and np.any((frac < 0.5) & (frac > 0.5 - 1e-6))
    # m = e^{x - n ln2} inside [sqrt(2)/2, sqrt(2)] for the literal version too
    for v in x[:200]:
        m, n = alg.ext_exp(float(v))
        assert math.sqrt(2) / 2 * (1 - 1e-9) <= m <= math.sqrt(2) * (1 + 1e-9)


def test_ulp32_at_binade_edges():
    # binary32 spacing (IEEE 754: 24-bit significand): ulp(1) = 2^-23, constant across a binade,
    # doubling at each power of two; equal to nextafter(v) - v for positive normal v
    from ulp import ulp32
    assert ulp32(1.0) == 2.0 ** -23
    assert ulp32(np.nextafter(np.float32(2.0), np.float32(0))) == 2.0 ** -23
    assert ulp32(2.0) == 2.0 ** -22
    assert ulp32(0.5) == 2.0 ** -24
    assert ulp32(np.float32(np.finfo(np.float32).tiny)) == 2.0 ** -149
    assert ulp32(-3.0) == 2.0 ** -22
    rng = np.random.default_rng(0)
    e = rng.integers(-125, 127, 2000)
    v = np.concatenate([np.exp2(e.astype(np.float64)),
                        (np.exp2(e.astype(np.float64)) * rng.uniform(1, 2, e.size)).astype(np.float32),
                        np.nextafter(np.exp2(e.astype(np.float32)), np.float32(0))]).astype(np.float32)
    nxt = np.nextafter(v, np.float32(np.inf)).astype(np.float64) - v.astype(np.float64)
    assert np.array_equal(ulp32(v), nxt)
