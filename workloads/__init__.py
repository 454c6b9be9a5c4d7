"""Seeded synthetic workloads for the Two-Pass softmax build (BASELINE.json:configs).

This module is the ONLY code shared by the oracle side (tests, oracle/) and the
CUDA side (bench.py, GPU tests).  It draws numbers and holds no softmax
arithmetic.  Generation is counter-based (workloads/gen.c), so any row range
or column chunk of a config can be produced on its own: a rank generates only
its shard and the values equal the corresponding slice of the full input.

Input recipe (gap ledger G15-G18):
  C1  1 x 1,000 fp32,     U[-100, 100]                                  configs[0]
  C2  64 x 32,768 fp32,   N(0, sd=4) + per-row offset U[-50, 50]         configs[1]
  C3  1 x 2^26 fp32,      U[-1000, 1000]                                 configs[2]
  C4  256 x 800,000 fp32, N(0, sd=10) + per-row offset U[-500, 500]      configs[3]
  C4b C4 rounded to bf16 (RNE)                                           configs[3]
  C5  1 x 2^31 fp32,      U[-1e4, 1e4]; Bernoulli(0.01) positions set to
      M = max of the drawn uniforms                                      configs[4]
All seeds are 0 (G17).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libworkloads.so")
_SRC = os.path.join(_HERE, "gen.c")


def build(force: bool = False) -> str:
    """Compile gen.c -> libworkloads.so (host C, OpenMP)."""
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
        i64, u64, dbl, vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
        L.wl_uniform_f32.argtypes = [vp, i64, u64, u64, i64, dbl, dbl]
        L.wl_normal_f32.argtypes = [vp, i64, u64, u64, i64, dbl, dbl]
        L.wl_rows_normal_offset_f32.argtypes = [vp, i64, i64, i64, i64, i64, u64, u64, u64, dbl, dbl]
        L.wl_uniform_max_f32.argtypes = [i64, u64, u64, dbl, dbl]
        L.wl_uniform_max_f32.restype = ctypes.c_float
        L.wl_bernoulli_set_f32.argtypes = [vp, i64, u64, u64, i64, dbl, ctypes.c_float]
        L.wl_bernoulli_set_f32.restype = i64
        L.wl_f32_to_bf16.argtypes = [vp, vp, i64]
        L.wl_bf16_to_f32.argtypes = [vp, vp, i64]
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


# ---------------------------------------------------------------- primitives

def uniform(n: int, lo: float, hi: float, seed: int = 0, stream: int = 0, offset: int = 0,
            out: np.ndarray | None = None) -> np.ndarray:
    out = np.empty(n, np.float32) if out is None else out
    lib().wl_uniform_f32(_ptr(out), n, seed, stream, offset, lo, hi)
    return out


def normal(n: int, mean: float, sd: float, seed: int = 0, stream: int = 0, offset: int = 0) -> np.ndarray:
    out = np.empty(n, np.float32)
    lib().wl_normal_f32(_ptr(out), n, seed, stream, offset, mean, sd)
    return out


def to_bf16(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bits (uint16), round to nearest even."""
    x = np.ascontiguousarray(x, np.float32)
    out = np.empty(x.shape, np.uint16)
    lib().wl_f32_to_bf16(_ptr(x), _ptr(out), x.size)
    return out


def bf16_to_f32(b: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(b, np.uint16)
    out = np.empty(b.shape, np.float32)
    lib().wl_bf16_to_f32(_ptr(b), _ptr(out), b.size)
    return out


# ---------------------------------------------------------------- configs

@dataclass(frozen=True)
class Config:
    key: str
    rows: int
    cols: int
    dtype: str  # "f32" or "bf16" (input dtype; output is always fp32)
    desc: str
    cite: str

    @property
    def elements(self) -> int:
        return self.rows * self.cols


CONFIGS = {
    "c1": Config("c1", 1, 1000, "f32", "single row, U[-100,100]", "BASELINE.json:configs[0]"),
    "c2": Config("c2", 64, 32768, "f32", "N(0,4)+U[-50,50] row offset", "BASELINE.json:configs[1]"),
    "c3": Config("c3", 1, 1 << 26, "f32", "single row, U[-1000,1000]", "BASELINE.json:configs[2]"),
    "c4": Config("c4", 256, 800000, "f32", "N(0,10)+U[-500,500] row offset", "BASELINE.json:configs[3]"),
    "c4b": Config("c4b", 256, 800000, "bf16", "C4 rounded to bf16", "BASELINE.json:configs[3]"),
    "c5": Config("c5", 1, 1 << 31, "f32", "U[-1e4,1e4], 1% ties at the max", "BASELINE.json:configs[4]"),
}

_STREAM = {"c1": 16, "c2": 32, "c3": 48, "c4": 64, "c4b": 64, "c5": 80}
_c5_tie_cache: dict = {}


def c5_tie_value(seed: int = 0) -> float:
    """M of config 5: the max of the drawn uniforms over the full 2^31 row (G16)."""
    if seed not in _c5_tie_cache:
        _c5_tie_cache[seed] = float(lib().wl_uniform_max_f32(1 << 31, seed, _STREAM["c5"], -1e4, 1e4))
    return _c5_tie_cache[seed]


def set_c5_tie_value(v: float, seed: int = 0) -> None:
    """Seed the cache with M computed elsewhere (multi-rank runs: rank 0 scans, broadcasts)."""
    _c5_tie_cache[seed] = float(v)


def generate(key: str, row0: int = 0, nrows: int | None = None, col0: int = 0,
             ncols: int | None = None, seed: int = 0, out: np.ndarray | None = None) -> np.ndarray:
    """Generate rows [row0, row0+nrows) x cols [col0, col0+ncols) of config `key`.

    Returns float32 [nrows, ncols] (uint16 bf16 bits for dtype bf16).  `out`, if
    given, must be a C-contiguous float32 array of that shape (for f32 configs),
    e.g. a pinned host buffer viewed through numpy.
    """
    cfg = CONFIGS[key]
    nrows = cfg.rows - row0 if nrows is None else nrows
    ncols = cfg.cols - col0 if ncols is None else ncols
    assert 0 <= row0 and row0 + nrows <= cfg.rows and 0 <= col0 and col0 + ncols <= cfg.cols
    st = _STREAM[key]
    if out is None or cfg.dtype == "bf16":
        buf = np.empty((nrows, ncols), np.float32)
    else:
        buf = out
        assert buf.dtype == np.float32 and buf.shape == (nrows, ncols) and buf.flags["C_CONTIGUOUS"]
    L = lib()
    if key in ("c1", "c3", "c5"):
        lo, hi = {"c1": (-100.0, 100.0), "c3": (-1000.0, 1000.0), "c5": (-1e4, 1e4)}[key]
        assert nrows == 1 or cfg.rows == 1
        L.wl_uniform_f32(_ptr(buf), nrows * ncols, seed, st, col0, lo, hi)
        if key == "c5":
            L.wl_bernoulli_set_f32(_ptr(buf), nrows * ncols, seed, st + 1, col0, 0.01,
                                   ctypes.c_float(c5_tie_value(seed)))
    else:
        sd, off = {"c2": (4.0, 50.0), "c4": (10.0, 500.0), "c4b": (10.0, 500.0)}[key]
        L.wl_rows_normal_offset_f32(_ptr(buf), nrows, ncols, row0, col0, cfg.cols, seed,
                                    st, st + 1, sd, off)
    if cfg.dtype == "bf16":
        b = to_bf16(buf)
        if out is not None:
            out[...] = b
            return out
        return b
    return buf


def ragged_case(rows: int, cols: int, lo: float = -50.0, hi: float = 50.0, seed: int = 0,
                stream: int = 7) -> np.ndarray:
    """Generic uniform test matrix (for ragged/edge-case shapes)."""
    return uniform(rows * cols, lo, hi, seed, stream).reshape(rows, cols)
