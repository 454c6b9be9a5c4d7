"""The oracle and the CUDA path share no code (static checks, -m "not gpu").

Only the seeded input generators (workloads/) serve both.  The product
package must never import, load or execute anything under oracle/.
"""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _files(d, exts):
    for dp, _, fns in os.walk(os.path.join(ROOT, d)):
        for fn in fns:
            if fn.endswith(exts):
                yield os.path.join(dp, fn)


def test_oracle_does_not_reference_product():
    for f in _files("oracle", (".py", ".c", ".h")):
        src = open(f).read()
        assert "paper_2001_04438_b200" not in src, f
        assert "csrc" not in src and "twopass.h" not in src, f


def test_product_does_not_reference_oracle():
    pat = re.compile(r"\boracle\b")
    for f in list(_files("paper_2001_04438_b200", (".py", ".cu", ".cuh", ".h", ".cpp"))) + \
            list(_files("include", (".h",))):
        src = open(f).read()
        assert not pat.search(src), f"{f} mentions the oracle"


def test_workloads_is_independent_of_both():
    for f in _files("workloads", (".py", ".c")):
        src = open(f).read()
        assert "paper_2001_04438_b200" not in src and "import oracle" not in src, f
