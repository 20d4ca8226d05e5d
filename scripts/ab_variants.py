"""Build A/B variants of libtba.so (compile-time switches; the defaults are the product) under
/tmp/tba_variants/<name>/libtba.so. Usage: python scripts/ab_variants.py name=DEF1,DEF2 ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_18929_b200 import _build  # noqa: E402

for arg in sys.argv[1:]:
    name, _, defs = arg.partition("=")
    print(name, _build.build_variant(name, [d for d in defs.split(",") if d]))
