"""GPU unit parity of the device building blocks (tp_debug_op through the C ABI).

ExtExp and Exp against their plain definitions (oracle, long double); pow2_flush
exhaustively; the pair merge against exact rational arithmetic.
"""
import math
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle
import workloads
from oracle import algorithms as alg

pytestmark = pytest.mark.gpu

tp = pytest.importorskip("paper_2001_04438_b200")


def _extexp(x):
    m, n = tp.debug_op(0, torch.from_numpy(np.asarray(x, np.float32)).cuda())
    torch.cuda.synchronize()
    return m.cpu().numpy(), n.cpu().numpy()


def _sweep():
    table = [0.0, 1.0, -1.0, 10.0, 100.0, -100.0, 200.0, -200.0, 1000.0, -1000.0, 1e4, -1e4,
             88.72283935546875, -103.97207641601562, 0.6931471824645996, 1e-30, -1e-30]
    # near-ties of x*log2e = k + 1/2
    ties = [(k + 0.5) * math.log(2) for k in range(-200, 200)]
    rnd = [workloads.uniform(200000, -1e4, 1e4, seed=11, stream=1),
           workloads.uniform(200000, -100, 100, seed=11, stream=2),
           workloads.uniform(50000, -1, 1, seed=11, stream=3)]
    return np.concatenate([np.asarray(table + ties, np.float32)] + rnd).astype(np.float32)


def test_extexp_pair_represents_exp():
    # (m, n) with m * 2^n = e^x; m within the polynomial's accuracy
    x = _sweep()
    m, n = _extexp(x)
    assert np.all(n == np.rint(n))
    want = oracle.exp_scaled(x, n.astype(np.float64))      # e^x 2^-n in long double
    rel = np.abs((m.astype(np.longdouble) - want) / want).astype(np.float64)
    assert rel.max() <= 3.0e-7, rel.max()
    # n is the nearest integer to x log2 e up to the fp32 rounding of log2 e (reading G1)
    dev = np.abs(n.astype(np.float64) - x.astype(np.float64) / math.log(2))
    # |x log2e| * 2^-24 bounds the error of the fp32 product x * RN32(log2 e)
    assert np.all(dev <= 0.5 + 1.4427 * 2.0 ** -24 * np.abs(x) + 1e-12)
    assert m.min() >= 0.70 and m.max() <= 1.42


def test_extexp_exact_points():
    m, n = _extexp([0.0, 1e4, -1e4, 200.0])
    assert m[0] == 1.0 and n[0] == 0.0            # fma(p, 0, 1) = 1 exactly
    ref_m, ref_n = oracle.extexp(np.float32([1e4, -1e4, 200.0]))
    assert np.array_equal(n[1:], ref_n.astype(np.float32))
    np.testing.assert_allclose(m[1:], ref_m.astype(np.float64), rtol=3e-7)


def test_extexp_clamped_domain():
    # |x| up to 2^21 stays accurate to 2e-5 (reading G11); beyond it outputs stay finite
    x = np.concatenate([workloads.uniform(100000, -2.0 ** 21, 2.0 ** 21, seed=3, stream=8),
                        np.float32([3.4e38, -3.4e38, 1e30, -1e30])]).astype(np.float32)
    m, n = _extexp(x)
    assert np.all(np.isfinite(m)) and np.all(np.isfinite(n)) and m.min() > 0
    inside = np.abs(x) <= 2.0 ** 21
    want = oracle.exp_scaled(x[inside], n[inside].astype(np.float64))
    rel = np.abs((m[inside].astype(np.longdouble) - want) / want).astype(np.float64)
    assert rel.max() <= 2e-5


def test_pow2_flush_exhaustive():
    k = np.concatenate([np.arange(-300, 2, dtype=np.float32), np.float32([-np.inf, np.nan])])
    s, _ = tp.debug_op(1, torch.from_numpy(k).cuda())
    s = s.cpu().numpy()
    for ki, si in zip(k[:-2], s[:-2]):
        want = 0.0 if ki < -126 else math.ldexp(1.0, int(ki))   # PAPER.md:252-258 (reading G5)
        assert si == np.float32(want), (ki, si)
    assert s[-2] == 0.0 and s[-1] == 0.0                         # identity and NaN (reading G6)


def test_mufu_ex2_is_exact_on_integers():
    # the kernels build 2^(n_i - n_max) with ex2.approx.ftz on integer arguments: it must be the
    # exact power of two for k >= -126, 0 below (flush, reading G5) and for -inf
    k = np.concatenate([np.arange(-400, 2, dtype=np.float32), np.float32([-np.inf, -1e30, -3e6])])
    s, _ = tp.debug_op(4, torch.from_numpy(k).cuda())
    s = s.cpu().numpy()
    for ki, si in zip(k, s):
        want = 0.0 if ki < -126 else math.ldexp(1.0, int(ki))
        assert si == np.float32(want), (ki, si)


def _merge(a, b):
    a = torch.from_numpy(np.asarray(a, np.float32).reshape(-1)).cuda()
    b = torch.from_numpy(np.asarray(b, np.float32).reshape(-1)).cuda()
    m, n = tp.debug_op(2, a, b)
    return m.cpu().numpy(), n.cpu().numpy()


def test_pair_merge_examples():
    # SPEC.md:48-59 examples, exact
    inf = np.inf
    A = [[0, -inf], [1, 3], [1.5, 10], [1, 128], [0, -inf], [1, 0]]
    B = [[1, 5], [1, 3], [1, 0], [1, -128], [0, -inf], [1, 0]]
    m, n = _merge(A, B)
    assert (m[0], n[0]) == (1.0, 5.0)
    assert (m[1], n[1]) == (2.0, 3.0)
    assert m[2] == np.float32(1.5 + 2.0 ** -10) and n[2] == 10.0
    assert (m[3], n[3]) == (1.0, 128.0)
    assert m[4] == 0.0 and n[4] == -np.inf                      # identity + identity (no NaN)
    assert (m[5], n[5]) == (2.0, 0.0)


def test_pair_merge_random_vs_exact():
    rng = np.random.default_rng(7)
    K = 20000
    ma = rng.uniform(0.7, 3000, K).astype(np.float32)
    mb = rng.uniform(0.7, 3000, K).astype(np.float32)
    na = rng.integers(-200, 200, K).astype(np.float32)
    nb = (na + rng.integers(-40, 40, K)).astype(np.float32)
    m, n = _merge(np.stack([ma, na], 1), np.stack([mb, nb], 1))
    assert np.array_equal(n, np.maximum(na, nb))
    for i in range(0, K, 7):
        v, nm = alg.pair_merge_exact((float(ma[i]), float(na[i])), (float(mb[i]), float(nb[i])))
        exact = alg.mantissa_exact(v, nm)
        ulp = Fraction(math.ulp(float(np.float32(float(exact)))) ) * Fraction(2 ** 29)  # fp64 ulp -> fp32 ulp
        err = abs(Fraction(float(m[i])) - exact)
        assert err <= ulp / 2 + Fraction(1, 2 ** 60), (i, float(err), float(ulp))


def test_exp_with_reconstruction_ulp():
    # Alg. 4 on d <= 0: within 3 ulp of e^d where the result is normal,
    # flushed to 0 when n < -126
    d = np.concatenate([workloads.uniform(300000, -87.3, 0.0, seed=5, stream=5),
                        np.float32([0.0, -1.0, -50.0, -87.33, -103.9, -104.0, -200.0, -1e4])]).astype(np.float32)
    e, _ = tp.debug_op(3, torch.from_numpy(d).cuda())
    e = e.cpu().numpy()
    true = oracle.exp_scaled(d, np.zeros(d.size))              # plain e^d, long double
    normal = true >= np.longdouble(np.finfo(np.float32).tiny)
    ulp = np.array([math.ulp(float(np.float32(t))) * 2 ** 29 for t in true[normal].astype(np.float64)])
    err = np.abs(e[normal].astype(np.longdouble) - true[normal]).astype(np.float64) / ulp
    assert err.max() <= 3.0, err.max()
    assert np.all(e[~normal] <= np.float32(np.finfo(np.float32).tiny))
    assert e[-1] == 0.0 and e[-2] == 0.0


# ------------------------------------------------------------------ exhaustive-lite ULP metrology (NEXT-2)

from ulp import ulp32 as _ulp32  # noqa: E402  (pinned at binade edges in test_oracle_pins.py)


@pytest.mark.parametrize("what", ["exp", "extexp"])
def test_exp_within_2_ulp_on_strided_fp32_sweep(what):
    # "maximum error under 2 ULP, validated through exhaustive evaluation".  The
    # exhaustive run is tools/exp_accuracy.py (profiles/r01b_exp_accuracy.json: 1.95 / 1.96 ulp);
    # here every 1021st fp32 of the domain, graded against the oracle's long-double definitions.
    import struct
    L = tp.lib()
    st = torch.cuda.current_stream().cuda_stream
    f2b = lambda v: struct.unpack("<I", struct.pack("<f", v))[0]  # noqa: E731
    if what == "exp":   # Alg. 4 on x in [ln FLT_MIN, 0] (normal outputs)
        spans = [(f2b(-0.0), f2b(-87.33654))]
    else:               # ExtExp on |x| <= 1e4 (the configurations' domain)
        spans = [(f2b(0.0), f2b(1e4)), (f2b(-0.0), f2b(-1e4))]
    worst = 0.0
    for b0, b1 in spans:
        bits = np.arange(b0, b1 + 1, 1021, dtype=np.uint64).astype(np.uint32)
        x = bits.view(np.float32)
        xd = torch.from_numpy(x.copy()).cuda()
        if what == "exp":
            y = tp.debug_op(3, xd)
            y = (y[0] if isinstance(y, tuple) else y).cpu().numpy()
            ref = oracle.exp_scaled(x, np.zeros(x.size))          # e^x in long double
            got = y
        else:
            m, n = tp.debug_op(0, xd)
            got, n = m.cpu().numpy(), n.cpu().numpy()
            ref = oracle.exp_scaled(x, n.astype(np.float64))      # e^x 2^-n: the m the pair must carry
        err = np.abs(got.astype(np.longdouble) - ref).astype(np.float64) / _ulp32(ref.astype(np.float64))
        worst = max(worst, float(err.max()))
    assert worst < 2.0, worst


# ------------------------------------------------------------------ the hot path's own forms (tp_debug_op 6, 7)

def test_hot_path_extexp_matches_definition_and_the_scalar_form():
    # op 6 = ext_exp2v<false>, exactly what pass 1 / pass 2 evaluate (FFMA2, n recovered from the
    # rounding sum): (m, n) represents e^x, and inside the accuracy domain it
    # is bit-identical to the clamped scalar ExtExp (op 0) the other unit tests grade
    lim = float(2 ** 21)
    x = np.concatenate([_sweep(), workloads.uniform(100000, -lim, lim, seed=12, stream=1)]).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    m6, n6 = (t.cpu().numpy() for t in tp.debug_op(6, xd))
    m0, n0 = (t.cpu().numpy() for t in tp.debug_op(0, xd))
    assert np.array_equal(m6.view(np.uint32), m0.view(np.uint32)) and np.array_equal(n6, n0)
    want = oracle.exp_scaled(x, n6.astype(np.float64))
    rel = np.abs((m6.astype(np.longdouble) - want) / want).astype(np.float64)
    small = np.abs(x) <= 1e4
    assert rel[small].max() <= 3.0e-7 and rel.max() <= 1e-5, (rel[small].max(), rel.max())
    # n: nearest integer of the exact product x * RN32(log2 e) (reading G1)
    n_exact = np.rint(x.astype(np.float64) * np.float64(np.float32(1.4426950408889634)))
    assert np.all(np.abs(n6 - n_exact) <= 0.0)


def test_hot_path_pow2_bits_exhaustive():
    # op 7 = pow2_bits(d): 2^(d - 127) built in the exponent field (Alg. 3's rescaling factors,
    # PAPER.md:161, 168), +0 for d <= 0 (flush below 2^-126); every d
    d = np.arange(-2000, 255, dtype=np.float32)
    got = tp.debug_op(7, torch.from_numpy(d).cuda())[0].cpu().numpy()
    want = np.array([np.float32(2.0 ** (int(k) - 127)) if k >= 1 else np.float32(0.0) for k in d], np.float32)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


# ------------------------------------------------------------------ warp value (tp_debug_op 8)

def _warp_cases(nwarps, seed):
    """Thread pairs like pass 1's accumulators: m in [sqrt(2)/2, 32 sqrt(2)], integer n around a
    per-warp base with spreads from a few to thousands (the flush band at 126-127 included),
    empty threads (0, -FLT_MAX), a few all-empty warps, and short mantissas (ties in the sums)."""
    rng = np.random.default_rng(seed)
    m = rng.uniform(0.70710678, 45.254834, size=(nwarps, 32)).astype(np.float32)
    short = rng.random((nwarps, 32)) < 0.2
    m[short] = (np.round(m[short] * 8) / 8).astype(np.float32)  # few significant bits
    base = rng.integers(-3_000_000, 3_000_000, size=(nwarps, 1))
    spread = rng.choice([3, 30, 120, 126, 127, 128, 140, 300, 3000], size=(nwarps, 1))
    n = (base - rng.integers(0, spread + 1, size=(nwarps, 32))).astype(np.float32)
    n[:, 0:1] = base  # one thread at the warp maximum
    band = rng.random((nwarps, 32)) < 0.1  # exactly at the flush boundary of the warp maximum
    n[band] = (base - rng.choice([125, 126, 127], size=(nwarps, 32)))[band]
    empty = rng.random((nwarps, 32)) < 0.05
    m[empty], n[empty] = 0.0, -np.float32(3.4028234663852886e38)
    m[:4], n[:4] = 0.0, -np.float32(3.4028234663852886e38)  # all-empty warps
    return m, n


def test_warp_value_is_the_pair_merge_tree():
    # reading G8: the kernels' warp value (maximum first, then a sum tree of the exactly rescaled
    # mantissas) is the perfect tree of pair merges (Alg. 3's update) over the
    # same 32 thread pairs in lane order, bit for bit, including spreads across the 2^-126 flush
    m, n = _warp_cases(20000, 21)
    a = torch.from_numpy(np.stack([m, n], -1).reshape(-1)).cuda()
    o = tp.debug_op(8, a)[0].cpu().numpy().reshape(-1, 32)[:, :4]
    assert np.array_equal(o[:, 0].view(np.uint32), o[:, 2].view(np.uint32)), "M differs"
    assert np.array_equal(o[:, 1], o[:, 3]), "N differs"
    # and against exact rationals: M 2^N within half an ulp per level of the 5-level tree
    for w in range(4, 400):
        nmax = int(n[w][m[w] > 0].max())
        exact = sum(Fraction(float(mi)) * Fraction(2) ** (int(ni) - nmax) for mi, ni in zip(m[w], n[w])
                    if mi > 0 and int(ni) - nmax >= -126)
        assert o[w, 1] == nmax
        rel = abs(Fraction(float(o[w, 0])) - exact) / exact
        assert rel <= Fraction(5, 2 ** 24), (w, float(rel))
    assert np.all(o[:4, 0] == 0.0) and np.all(o[:4, 1] == -np.float32(3.4028234663852886e38))
