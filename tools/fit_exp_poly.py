"""Derive the degree-5 polynomial of ExtExp / Exp.

The paper's coefficients (Sollya, Brisebarre-Chevillard) are not printed
(SURVEY.md gap G3), so the CUDA path uses coefficients derived here:

  1. minimax of the RELATIVE error of p(t) = 1 + t(c1 + t(c2 + t(c3 + t(c4 + t c5))))
     against e^t on |t| <= A (A covers the reduced range [-ln2/2, ln2/2] plus the
     rounding slack of the fp32 range reduction), solved as a linear program;
  2. round to binary32, then a greedy search over neighbouring binary32 values
     minimising the max ULP error of the fp32 Horner evaluation with FMA
     (emulated here in long double) on a dense grid of fp32 t values.

Output: the coefficients as C hex-float literals, pasted into
paper_2001_04438_b200/csrc/extexp.cuh.  This script is a constant generator for
the CUDA path only; the oracle never uses these coefficients.

Run:  python tools/fit_exp_poly.py
"""
import numpy as np
from scipy.optimize import linprog

A = 0.3476  # > ln2/2 = 0.34657; covers |t| for |x| <= 2^21
LD = np.longdouble


def lp_minimax(npts=4000):
    t = np.cos(np.linspace(0, np.pi, npts)) * A
    # variables c1..c5, e ; minimize e  s.t. |(1 + sum c_k t^k) e^-t - 1| <= e
    et = np.exp(-t)
    V = np.stack([t ** k * et for k in range(1, 6)], axis=1)
    r = 1 - et
    Aub = np.vstack([np.hstack([V, -np.ones((npts, 1))]), np.hstack([-V, -np.ones((npts, 1))])])
    bub = np.concatenate([r, -r])
    res = linprog(np.r_[np.zeros(5), 1.0], A_ub=Aub, b_ub=bub, bounds=[(None, None)] * 6,
                  method="highs")
    return res.x[:5], res.x[5]


def f32(v):
    return np.float32(v)


def fma32(a, b, c):
    """RN32(a*b + c) via long double (a*b exact in 64-bit mantissa)."""
    return (LD(a) * LD(b) + LD(c)).astype(np.float32)


def horner(c, t):
    p = np.full(t.shape, c[4], np.float32)
    for k in (3, 2, 1, 0):
        p = fma32(p, t, np.full(t.shape, c[k], np.float32))
    return fma32(p, t, np.ones(t.shape, np.float32))


T = np.unique(np.concatenate([
    np.linspace(-A, A, 400001).astype(np.float32),
    (np.random.default_rng(0).uniform(-A, A, 400000)).astype(np.float32)]))
TRUE = np.exp(T.astype(LD))


def ulp_err(c):
    p = horner(c, T).astype(LD)
    ulp = np.where(TRUE >= 1, LD(2.0 ** -23), LD(2.0 ** -24))
    return float(np.max(np.abs(p - TRUE) / ulp))


def search(c):
    c = [f32(v) for v in c]
    best = ulp_err(c)
    improved = True
    while improved:
        improved = False
        for k in range(5):
            for d in (-3, -2, -1, 1, 2, 3):
                cand = list(c)
                v = np.float32(c[k])
                for _ in range(abs(d)):
                    v = np.nextafter(v, np.float32(np.inf if d > 0 else -np.inf))
                cand[k] = v
                e = ulp_err(cand)
                if e < best - 1e-9:
                    best, c, improved = e, cand, True
    return c, best


def main():
    c, e = lp_minimax()
    print(f"LP minimax relative error (real coefficients): {e:.3e}")
    c32, err = search(c)
    print(f"max ULP error of fp32 Horner p(t) on |t|<={A}: {err:.3f}")
    for k, v in enumerate(c32, 1):
        print(f"#define TP_C{k} {float(v).hex()}f  /* {float(v):.9g} */")


if __name__ == "__main__":
    main()
