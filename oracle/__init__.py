"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU implementations used to check the CUDA path
of the Two-Pass softmax build (arXiv 2001.04438, PAPER.md).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
import this package.  It imports nothing from paper_2001_04438_b200/ and the
CUDA path imports nothing from here.

Contents
  oracle.c (-> liboracle.so), wrapped below:
    row_stats, softmax, softmax_unshifted, check, extexp, exp_scaled
      plain definition of softmax (§1; shift identity
      PAPER.md:78-86 §3), fp64 exp + long-double accumulation; the unshifted
      long-double formula as an independent cross-check; ExtExp's plain
      definition (§4).
  algorithms.py:
      Alg. 1-3 of the paper written out literally in fp64 (small inputs),
      and exact rational arithmetic of (m, n) pairs.

Every function is pinned in tests/test_oracle_pins.py (closed forms,
invariants, mpmath brute force, two-formula agreement); exp_scaled and the
rounding of ExtExp's n (both oracle versions) against mpmath at 50 digits over
|x| <= 2^21, next to half-integer products included.  No parity is
unpinned in this package; the one unpinned item of the build (the paper's
exact polynomial coefficients) is not computed here at all.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

FLT_MIN = float(np.finfo(np.float32).tiny)
RTOL = 2e-5   # BASELINE.json:north_star, outputs >= FLT_MIN
ATOL = 1e-37  # BASELINE.json:north_star, outputs <  FLT_MIN


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain C, no -ffast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-ffp-contract=off",
                               "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        vp, i64, dbl, ld = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_longdouble
        for nm in ("oracle_row_stats_f32", "oracle_row_stats_bf16"):
            getattr(L, nm).argtypes = [vp, i64, ctypes.POINTER(dbl), ctypes.POINTER(ld)]
        for nm in ("oracle_softmax_f32", "oracle_softmax_bf16", "oracle_softmax_unshifted_f32"):
            getattr(L, nm).argtypes = [vp, i64, vp]
        for nm in ("oracle_check_f32", "oracle_check_bf16"):
            f = getattr(L, nm)
            f.argtypes = [vp, vp, i64, dbl, ld, dbl, dbl, vp, ctypes.POINTER(i64)]
            f.restype = i64
        L.oracle_extexp.argtypes = [vp, i64, vp, vp]
        L.oracle_exp_scaled.argtypes = [vp, vp, i64, vp]
        L.oracle_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"], "oracle needs C-contiguous arrays"
    return a.ctypes.data


def _kind(x: np.ndarray) -> str:
    if x.dtype == np.float32:
        return "f32"
    if x.dtype == np.uint16:
        return "bf16"  # bf16 bit patterns
    raise TypeError(f"oracle takes float32 or bf16-as-uint16, got {x.dtype}")


def threads() -> int:
    """OpenMP threads the oracle runs on."""
    return int(lib().oracle_threads())


def row_stats(x: np.ndarray) -> tuple[float, np.longdouble]:
    """mu = max_i x_i and S = sum_i exp(x_i - mu) of one row."""
    x = np.ascontiguousarray(x).reshape(-1)
    mu, S = ctypes.c_double(), ctypes.c_longdouble()
    getattr(lib(), f"oracle_row_stats_{_kind(x)}")(_p(x), x.size, ctypes.byref(mu), ctypes.byref(S))
    return mu.value, np.longdouble(S.value)


def softmax(x: np.ndarray) -> np.ndarray:
    """Row-wise softmax in long double: o_i = exp(x_i - mu) / S."""
    x = np.ascontiguousarray(x)
    x2 = x.reshape(-1, x.shape[-1]) if x.ndim else x.reshape(1, 1)
    out = np.empty(x2.shape, np.longdouble)
    f = getattr(lib(), f"oracle_softmax_{_kind(x)}")
    for r in range(x2.shape[0]):
        row = np.ascontiguousarray(x2[r])
        o = np.empty(row.size, np.longdouble)
        f(_p(row), row.size, _p(o))
        out[r] = o
    return out.reshape(x.shape)


def softmax_unshifted(x: np.ndarray) -> np.ndarray:
    """Independent formula: expl(x_i) / sum_k expl(x_k), |x| <= 11356."""
    x = np.ascontiguousarray(x, np.float32)
    x2 = x.reshape(-1, x.shape[-1])
    out = np.empty(x2.shape, np.longdouble)
    for r in range(x2.shape[0]):
        row = np.ascontiguousarray(x2[r])
        o = np.empty(row.size, np.longdouble)
        lib().oracle_softmax_unshifted_f32(_p(row), row.size, _p(o))
        out[r] = o
    return out.reshape(x.shape)


@dataclass
class CheckResult:
    n_bad: int
    first_bad: int
    max_rel: float
    max_abs: float
    n_rel: int
    n_abs: int
    y_sum: float

    @property
    def ok(self) -> bool:
        return self.n_bad == 0

    def merge(self, o: "CheckResult", offset: int = 0) -> "CheckResult":
        fb = self.first_bad
        if fb < 0 and o.first_bad >= 0:
            fb = o.first_bad + offset
        return CheckResult(self.n_bad + o.n_bad, fb, max(self.max_rel, o.max_rel),
                           max(self.max_abs, o.max_abs), self.n_rel + o.n_rel,
                           self.n_abs + o.n_abs, self.y_sum + o.y_sum)


def check(x: np.ndarray, y: np.ndarray, stats: tuple[float, np.longdouble] | None = None,
          rtol: float = RTOL, atol: float = ATOL) -> CheckResult:
    """Grade y against the oracle element by element (BASELINE.json:north_star).

    x, y: one row (or a gathered sample of one row, then `stats` = that row's
    full (mu, S) is required).  Relative branch for o_i >= FLT_MIN, absolute
    branch below (the branch is chosen on the ORACLE value).
    """
    x = np.ascontiguousarray(x).reshape(-1)
    y = np.ascontiguousarray(y, np.float32).reshape(-1)
    assert x.size == y.size
    mu, S = row_stats(x) if stats is None else stats
    st = np.zeros(5, np.float64)
    fb = ctypes.c_int64()
    nbad = getattr(lib(), f"oracle_check_{_kind(x)}")(_p(x), _p(y), x.size, mu,
                                                       ctypes.c_longdouble(S), rtol, atol,
                                                       _p(st), ctypes.byref(fb))
    return CheckResult(int(nbad), int(fb.value), float(st[0]), float(st[1]), int(st[2]),
                       int(st[3]), float(st[4]))


def check_rows(x: np.ndarray, y: np.ndarray, rtol: float = RTOL, atol: float = ATOL) -> CheckResult:
    """check() row by row of a [rows, cols] matrix."""
    x2 = x.reshape(-1, x.shape[-1])
    y2 = y.reshape(-1, y.shape[-1])
    res = CheckResult(0, -1, 0.0, 0.0, 0, 0, 0.0)
    for r in range(x2.shape[0]):
        res = res.merge(check(x2[r], y2[r], None, rtol, atol), offset=r * x2.shape[1])
    return res


def extexp(x: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """ExtExp plain definition: n = round(x log2 e), m = e^{x - n ln2}."""
    x = np.ascontiguousarray(x, np.float32).reshape(-1)
    m = np.empty(x.size, np.longdouble)
    n = np.empty(x.size, np.float64)
    lib().oracle_extexp(_p(x), x.size, _p(m), _p(n))
    return m, n


def exp_scaled(x: np.ndarray, k: np.ndarray) -> np.ndarray:
    """e^{x} * 2^{-k} in long double (the value a pair (m, k) must represent)."""
    x = np.ascontiguousarray(x, np.float32).reshape(-1)
    k = np.ascontiguousarray(k, np.float64).reshape(-1)
    out = np.empty(x.size, np.longdouble)
    lib().oracle_exp_scaled(_p(x), _p(k), x.size, _p(out))
    return out
