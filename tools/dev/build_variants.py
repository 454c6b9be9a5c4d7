"""Build variant libraries exp_libs/<name>.so with extra -D defines (development A/B tool).

    python tools/dev/build_variants.py name=DEF1,DEF2 name2=DEF3 ...   (name=- : no defines)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2001_04438_b200 import build as b  # noqa: E402

for spec in sys.argv[1:]:
    name, defs = spec.split("=", 1)
    d = tuple(x for x in defs.split(",") if x and x != "-")
    out = os.path.join(ROOT, "exp_libs", name + ".so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    b.build(force=True, out=out, defines=d or ("TP_VARIANT_BASE",))
    print(out)
