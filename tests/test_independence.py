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


IMPORT_PRODUCT = re.compile(r"^\s*(import|from)\s+paper_2001_04438_b200|#include\s*[<\"].*(csrc|twopass)"
                            r"|libtwopass", re.M)
IMPORT_ORACLE = re.compile(r"^\s*(import|from)\s+oracle\b|#include\s*[<\"].*oracle|liboracle", re.M)


def test_oracle_does_not_reference_product():
    for f in _files("oracle", (".py", ".c", ".h")):
        src = open(f).read()
        assert not IMPORT_PRODUCT.search(src), f


def test_product_does_not_reference_oracle():
    for f in list(_files("paper_2001_04438_b200", (".py", ".cu", ".cuh", ".h", ".cpp"))) + \
            list(_files("include", (".h",))):
        src = open(f).read()
        assert not IMPORT_ORACLE.search(src), f"{f} imports/loads the oracle"


def test_workloads_is_independent_of_both():
    for f in _files("workloads", (".py", ".c")):
        src = open(f).read()
        assert not IMPORT_PRODUCT.search(src) and not IMPORT_ORACLE.search(src), f
