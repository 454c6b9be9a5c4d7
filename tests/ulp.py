"""ULP of binary32 (test helper; pinned in tests/test_oracle_pins.py).

ulp32(v) = 2^(floor(log2 |v|) - 23) for normal binary32 magnitudes: the spacing of binary32
numbers in the binade [2^e, 2^(e+1)) that contains v (IEEE 754 binary32, 24-bit significand).
The grading of the exponential's accuracy ("maximum error under 2 ULP") divides
by it.
"""
import numpy as np


def ulp32(v):
    v = np.abs(np.asarray(v, np.float64))
    return np.exp2(np.floor(np.log2(v)) - 23)
