"""Build a libpa.so variant with extra -D macros into variants/<name>/libpa.so (A/B timing of compile-time
kernel parameters; load it with PA_LIB_PATH=variants/<name>/libpa.so).
Usage: python tools/build_variant.py name -DMACRO=V ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_09643_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(b.ROOT, "variants", name)
print(b.build(force=True, defs=defs, lib=os.path.join(out, "libpa.so"), objdir=os.path.join(out, "obj")))
