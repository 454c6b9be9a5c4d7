"""The staging-ring index arithmetic of the resident-row kernels (csrc/tp_rowres.cuh, ResDiv):
k / d and k % d by one 32-bit multiply-high with magic = floor((2^32 - 1) / d) + 1, claimed exact
for d = 2..8 (rows staged per CTA) and k < 2^29 (kResMaxRowsPerGroup, enforced by the launchers).
Host-side check of that claim: the error term e = magic * d - 2^32 must satisfy k * e < 2^32."""
import random
import re
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KMAX = 1 << 29


def _quot(k, d):
    magic = (0xFFFFFFFF // d + 1) & 0xFFFFFFFF
    return (k * magic) >> 32


def test_limit_matches_the_header():
    src = open(os.path.join(ROOT, "paper_2001_04438_b200", "csrc", "tp_rowres.cuh")).read()
    assert re.search(r"kResMaxRowsPerGroup = \(int64_t\)1 << 29;", src)
    assert "0xffffffffu / (unsigned)d_ + 1u" in src
    assert re.search(r"constexpr int kResSlots = 8;", src)  # d never exceeds the staged slots


def test_multiply_high_division_is_exact_below_the_limit():
    rng = random.Random(0)
    for d in range(2, 9):
        magic = 0xFFFFFFFF // d + 1
        e = magic * d - (1 << 32)
        assert 0 <= e <= d and (KMAX - 1) * e < (1 << 32)  # the exactness condition
        ks = [0, 1, d - 1, d, d + 1, KMAX - 1, KMAX - d, KMAX - d - 1]
        ks += [m * d + r for m in (1, 1000, (KMAX // d) - 1) for r in (0, d - 1)]
        ks += [rng.randrange(KMAX) for _ in range(20000)]
        for k in ks:
            if 0 <= k < KMAX:
                q = _quot(k, d)
                assert q == k // d and k - q * d == k % d, (k, d)
