"""Build a timing-experiment copy of the library (never the product .so):
    python scripts/build_experiment.py NAME DEFINE[=V] ...   ->  build/exp/libcypress_NAME.so
Probes load it with  paper_2504_07004_b200._lib.use_library(path)  before the first call."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_07004_b200 import build  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "build", "exp", f"libcypress_{name}.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
print(build.build(force=True, verbose=True, defines=defs, out=out))
