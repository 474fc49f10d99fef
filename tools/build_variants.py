"""Build kernel variants of libhfmm (extra -D flags) next to the default library, for A/B timing:
    python tools/build_variants.py NAME=DEF1,DEF2 ...   -> paper_0911_4114_b200/libhfmm_NAME.so
Load one with HFMM_LIB=<path> (binding.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0911_4114_b200.build import build, HERE  # noqa: E402

for arg in sys.argv[1:]:
    name, _, defs = arg.partition("=")
    out = os.path.join(HERE, f"libhfmm_{name}.so")
    build(force=True, verbose=False, defines=[d for d in defs.split(",") if d], out=out)
    print(out)
