"""Build a measurement variant of libgcoo_cuda.so (never the product):

    python tools/build_variant.py NAME [DEFINE=VALUE ...]   -> tools/_abl/libgcoo_NAME.so

then run any script against it with GCOO_LIB=tools/_abl/libgcoo_NAME.so.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2005_14469_b200 import build  # noqa: E402

name, defines = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "tools", "_abl", f"libgcoo_{name}.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
print(build.build(out=out, defines=defines))
